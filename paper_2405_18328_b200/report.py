"""Trace / report emission: the reference's report layer
(proj/include/warmgp/report.hpp, proj/src/report.cpp) over this package's
OptTrace and ExperimentResult.

- to_json(OptTrace)           report.cpp:31-45 (same keys per step; the
                              device-timed solver / step times are reported
                              in the reference's seconds fields)
- to_json(ExperimentResult)   report.cpp:47-84
- emit_report                 report.cpp:129-148 (JSON, or CSV with
                              17-significant-digit numerics)
- load_csv_table              report.cpp:150-172 (cells round-trip bit-exactly)
- wall_time_keys / strip_wall_time_fields   report.cpp:174-187
- parse_config_file           report.cpp:189-217 (flat `key = value`, '#')

Host-side plumbing: no device work happens here.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List

__all__ = ["IoError", "ReportFormat", "report_format_from_string", "to_json", "emit_report",
           "write_json_file", "load_json_file", "CsvTable", "load_csv_table", "wall_time_keys",
           "strip_wall_time_fields", "parse_config_file", "format_double"]


class IoError(OSError):
    """warmgp::IoError (proj/include/warmgp/common.hpp), exit code 4."""


class ReportFormat:
    Json = "json"
    Csv = "csv"


def report_format_from_string(name: str) -> str:
    """report.cpp:25-29."""
    if name in (ReportFormat.Json, ReportFormat.Csv):
        return name
    raise ValueError("unknown report format: " + name)


def format_double(v: float) -> str:
    """report.cpp:13-17: printf("%.17g") -- round-trips every double."""
    return "%.17g" % float(v)


def _vec(a) -> List[float]:
    return [float(x) for x in a]


def _trace_json(trace) -> dict:
    steps = []
    cumulative = 0.0
    for rec in trace.steps:
        cumulative += rec.step_ms / 1e3
        steps.append({
            "step": int(rec.step),
            "raw_params": _vec(rec.raw_params),
            "constrained_params": _vec(rec.constrained_params),
            "gradient": _vec(rec.gradient),
            "solver_iterations": int(rec.solver_iterations),
            "solver_seconds": rec.solver_ms / 1e3,
            "cumulative_seconds": cumulative,
            "per_column_relative_residual": _vec(rec.per_column_relative_residual),
            "warm_start_distance": float(rec.warm_start_distance),
        })
    return {"steps": steps}


def _agg(a) -> dict:
    return {"mean": a.mean, "standard_error": a.standard_error}


def _result_json(result) -> dict:
    runs = []
    for rec in result.runs:
        run = {"label": rec.label, "solver": rec.solver, "mode": rec.mode,
               "split_index": rec.split_index, "split_seed": rec.split_seed,
               "train_seed": rec.train_seed, "test_rmse": rec.test_rmse,
               "test_llh": rec.test_llh, "total_runtime_seconds": rec.total_runtime_seconds,
               "solver_runtime_seconds": rec.solver_runtime_seconds,
               "per_step_iterations": [int(v) for v in rec.per_step_iterations],
               "final_constrained": _vec(rec.final_constrained)}
        if rec.trace is not None and rec.trace.steps:
            run["trace"] = _trace_json(rec.trace)
        runs.append(run)
    summaries = {label: {"test_rmse": _agg(s.rmse), "test_llh": _agg(s.llh),
                         "total_runtime_seconds": _agg(s.total_runtime),
                         "solver_runtime_seconds": _agg(s.solver_runtime)}
                 for label, s in sorted(result.summaries.items())}
    return {"dataset": result.dataset, "splits": result.splits,
            "train_fraction": result.train_fraction, "runs": runs, "summaries": summaries,
            "speed_up": dict(sorted(result.speed_up.items()))}


def to_json(obj) -> dict:
    """report.cpp:31-84: an OptTrace (per-step records) or an ExperimentResult."""
    if hasattr(obj, "runs"):
        return _result_json(obj)
    if hasattr(obj, "steps"):
        return _trace_json(obj)
    raise TypeError("to_json: expected an OptTrace or an ExperimentResult")


def write_json_file(j: dict, path: str) -> None:
    """report.cpp:111-116 (2-space indent, trailing newline)."""
    try:
        with open(path, "w") as f:
            f.write(json.dumps(j, indent=2, allow_nan=True) + "\n")
    except OSError as e:
        raise IoError("cannot open " + path + " for writing") from e


def load_json_file(path: str) -> dict:
    """report.cpp:118-127."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise IoError("cannot open " + path) from e
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise IoError(path + ": " + str(e)) from e


_CSV_HEADER = ("dataset,label,solver,mode,split_index,split_seed,train_seed,test_rmse,test_llh,"
               "total_runtime_seconds,solver_runtime_seconds,total_iterations")


def emit_report(result, path: str, fmt: str = ReportFormat.Json) -> None:
    """report.cpp:129-148: JSON (the full nested record) or a flat CSV per
    (config, split) with 17-significant-digit numerics."""
    fmt = report_format_from_string(fmt)
    if fmt == ReportFormat.Json:
        write_json_file(to_json(result), path)
        return
    lines = [_CSV_HEADER]
    for rec in result.runs:
        total = sum(int(v) for v in rec.per_step_iterations)
        lines.append(",".join([result.dataset, rec.label, rec.solver, rec.mode, str(rec.split_index),
                               str(rec.split_seed), str(rec.train_seed), format_double(rec.test_rmse),
                               format_double(rec.test_llh), format_double(rec.total_runtime_seconds),
                               format_double(rec.solver_runtime_seconds), str(total)]))
    try:
        with open(path, "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError as e:
        raise IoError("cannot open " + path + " for writing") from e


@dataclass
class CsvTable:
    header: List[str] = field(default_factory=list)
    rows: List[List[str]] = field(default_factory=list)


def load_csv_table(path: str) -> CsvTable:
    """report.cpp:150-172: header + rows of string cells (numeric cells parse
    back bit-exactly with float())."""
    try:
        with open(path) as f:
            lines = f.read().splitlines()
    except OSError as e:
        raise IoError("cannot open " + path) from e
    table = CsvTable()
    first = True
    for line in lines:
        if not line:
            continue
        fields = line.split(",")
        if first:
            table.header = fields
            first = False
        else:
            table.rows.append(fields)
    return table


_WALL_TIME_KEYS = ("solver_seconds", "cumulative_seconds", "total_runtime_seconds",
                   "solver_runtime_seconds", "speed_up")


def wall_time_keys() -> List[str]:
    """report.cpp:174-178: keys holding wall-clock measurements (and
    quantities derived from them)."""
    return list(_WALL_TIME_KEYS)


def strip_wall_time_fields(j):
    """report.cpp:179-187: recursively removes the wall-time keys; reports are
    byte-identical across reruns once these are erased."""
    if isinstance(j, dict):
        return {k: strip_wall_time_fields(v) for k, v in j.items() if k not in _WALL_TIME_KEYS}
    if isinstance(j, list):
        return [strip_wall_time_fields(v) for v in j]
    return j


def parse_config_file(path: str) -> Dict[str, str]:
    """report.cpp:189-217: flat `key = value` lines, '#' starts a comment;
    IoError names the offending line."""
    try:
        with open(path) as f:
            lines = f.read().split("\n")
    except OSError as e:
        raise IoError("cannot open config file " + path) from e
    out: Dict[str, str] = {}
    ws = " \t\r\n"
    for number, line in enumerate(lines, start=1):
        hash_at = line.find("#")
        if hash_at >= 0:
            line = line[:hash_at]
        t = line.strip(ws)
        if not t:
            continue
        eq = t.find("=")
        if eq < 0:
            raise IoError(f"{path}: line {number} is not 'key = value'")
        key = t[:eq].strip(ws)
        value = t[eq + 1:].strip(ws)
        if not key:
            raise IoError(f"{path}: line {number} has an empty key")
        out[key] = value
    return out

