"""Paired warm/cold experiment driver: the reference's
proj/src/experiment.cpp and split_standardize (proj/src/dataset.cpp:109-166)
over the device training loop.

- split_standardize   dataset.cpp:109-166: the reference's permutation
                      (wgp_split_order, bitwise), training-split statistics
                      (population variance, zero deviation -> 1)
- paired_grid         experiment.cpp:31-44: "<solver>/cold" (resampled probes)
                      and "<solver>/warm" (warm start, fixed probes)
- run_experiment      experiment.cpp:46-131: per split the seeds
                      derive_seed(seed, 0x3711700 + split) (split) and
                      derive_seed(seed, 0x7ea1 + split) (training, shared by
                      the paired entries); test metrics at the final
                      hyperparameters; per-label mean / standard error; the
                      cold / warm total-runtime speed-up per solver
- grid_search_sgd_lr  experiment.cpp:133-168: short SGD solves at the initial
                      hyperparameters, smallest exact relative residual wins,
                      diverging candidates skipped

Deviations, by design of this build: training runs on the GPU in fp32 (the
device loop of wgp_train), and the test metrics use this package's device
predictor (iterative solves) instead of the reference's dense fp64 one.
"""
from __future__ import annotations

import dataclasses
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import (Context, Hyperparameters, KernelOperator, NumericalError, OptTrace, SolverConfig,
               TrainConfig, derive_seed, predict, solve, split_order, test_metrics, train)

__all__ = ["Dataset", "split_standardize", "GridEntry", "RunRecord", "Aggregate", "LabelSummary",
           "ExperimentResult", "ExperimentOptions", "paired_grid", "run_experiment",
           "grid_search_sgd_lr"]


@dataclass
class Dataset:
    """dataset.hpp:16-31."""
    name: str
    X: np.ndarray
    y: np.ndarray
    feature_means: Optional[np.ndarray] = None
    feature_stds: Optional[np.ndarray] = None
    target_mean: float = 0.0
    target_std: float = 1.0
    standardized: bool = False
    split_seed: int = 0
    train_fraction: float = 0.0

    @property
    def n(self) -> int:
        return int(self.X.shape[0])

    @property
    def d(self) -> int:
        return int(self.X.shape[1])


def split_standardize(ds: Dataset, train_fraction: float, split_seed: int):
    """dataset.cpp:109-166: random split (the reference's permutation) and
    standardisation of both parts with the training split's statistics."""
    if not (0.0 < train_fraction < 1.0):
        raise ValueError("split_standardize: train_fraction must lie in (0, 1)")
    X = np.asarray(ds.X, dtype=np.float64)
    y = np.asarray(ds.y, dtype=np.float64).ravel()
    n = X.shape[0]
    n_train = int(np.floor(train_fraction * n))
    if n_train < 1 or n_train >= n:
        raise ValueError("split_standardize: split leaves an empty train or test set")
    order = split_order(n, split_seed)
    tr, te = order[:n_train], order[n_train:]
    Xtr, ytr = X[tr], y[tr]
    means = Xtr.mean(axis=0)
    sd = np.sqrt(((Xtr - means) ** 2).mean(axis=0))
    stds = np.where(sd > 0.0, sd, 1.0)
    y_mean = float(ytr.mean())
    y_var = float(((ytr - y_mean) ** 2).mean())
    y_std = float(np.sqrt(y_var)) if y_var > 0.0 else 1.0
    parts = []
    for idx in (tr, te):
        parts.append(Dataset(ds.name, (X[idx] - means) / stds, (y[idx] - y_mean) / y_std, means.copy(),
                             stds.copy(), y_mean, y_std, True, split_seed, train_fraction))
    return parts[0], parts[1]


@dataclass
class GridEntry:
    """experiment.hpp:14-18: one labelled configuration, e.g. cg/warm."""
    label: str
    config: TrainConfig


@dataclass
class RunRecord:
    """experiment.hpp:20-35: the outcome of one (config, split) run."""
    label: str
    solver: str
    mode: str
    split_index: int
    split_seed: int
    train_seed: int
    test_rmse: float = 0.0
    test_llh: float = 0.0
    total_runtime_seconds: float = 0.0
    solver_runtime_seconds: float = 0.0
    per_step_iterations: List[int] = field(default_factory=list)
    final_constrained: np.ndarray = field(default_factory=lambda: np.zeros(0))
    trace: Optional[OptTrace] = None


@dataclass
class Aggregate:
    mean: float = 0.0
    standard_error: float = 0.0


@dataclass
class LabelSummary:
    rmse: Aggregate = field(default_factory=Aggregate)
    llh: Aggregate = field(default_factory=Aggregate)
    total_runtime: Aggregate = field(default_factory=Aggregate)
    solver_runtime: Aggregate = field(default_factory=Aggregate)


@dataclass
class ExperimentResult:
    """experiment.hpp:45-52."""
    dataset: str = ""
    splits: int = 0
    train_fraction: float = 0.9
    runs: List[RunRecord] = field(default_factory=list)
    summaries: Dict[str, LabelSummary] = field(default_factory=dict)
    speed_up: Dict[str, float] = field(default_factory=dict)


@dataclass
class ExperimentOptions:
    """experiment.hpp:54-59."""
    splits: int = 10
    train_fraction: float = 0.9
    seed: int = 0
    keep_traces: bool = True


def _aggregate(values: Sequence[float]) -> Aggregate:
    """experiment.cpp:14-27: mean and standard error (n - 1 denominator)."""
    a = Aggregate()
    if not values:
        return a
    v = np.asarray(values, dtype=np.float64)
    a.mean = float(v.sum() / v.size)
    if v.size > 1:
        a.standard_error = float(np.sqrt(((v - a.mean) ** 2).sum() / (v.size - 1) / v.size))
    return a


def paired_grid(solvers: Sequence[str], base: TrainConfig) -> List[GridEntry]:
    """experiment.cpp:31-44."""
    grid = []
    for kind in solvers:
        cold = dataclasses.replace(base, solver=dataclasses.replace(base.solver, kind=kind), mode="cold")
        grid.append(GridEntry(f"{kind}/cold", cold))
        grid.append(GridEntry(f"{kind}/warm", dataclasses.replace(cold, mode="warm")))
    return grid


def run_experiment(ds: Dataset, grid: Sequence[GridEntry], options: ExperimentOptions = None,
                   device: int = 0, ctx: Optional[Context] = None) -> ExperimentResult:
    """experiment.cpp:46-131 on the device: every grid entry on every split,
    test metrics at the final hyperparameters, per-label aggregates and the
    cold / warm speed-up per solver.  Runtimes are host wall clock around
    each training run (as the reference), solver runtimes the device-timed
    solver phases of the trace."""
    options = options or ExperimentOptions()
    if not grid:
        raise ValueError("run_experiment: empty config grid")
    if options.splits < 1:
        raise ValueError("run_experiment: splits must be >= 1")
    ctx = ctx or Context(device)
    result = ExperimentResult(ds.name, options.splits, options.train_fraction)
    for split in range(options.splits):
        split_seed = derive_seed(options.seed, 0x3711700 + split)
        train_ds, test_ds = split_standardize(ds, options.train_fraction, split_seed)
        train_seed = derive_seed(options.seed, 0x7ea1 + split)  # shared by paired entries
        for entry in grid:
            config = dataclasses.replace(entry.config, seed=train_seed)
            try:
                t0 = time.perf_counter()
                trace = train(train_ds.X, train_ds.y, config, ctx=ctx)
                total = time.perf_counter() - t0
                rec = RunRecord(entry.label, config.solver.kind, config.mode, split, split_seed, train_seed,
                                total_runtime_seconds=total)
                for s in trace.steps:
                    rec.solver_runtime_seconds += s.solver_ms / 1e3
                    rec.per_step_iterations.append(int(s.solver_iterations))
                if not trace.steps:
                    raise RuntimeError("OptTrace: empty trace")
                final = Hyperparameters(np.asarray(trace.back().raw_params, dtype=np.float64), config.transform)
                rec.final_constrained = final.to_constrained_vector()
                pred = predict(train_ds.X, train_ds.y, test_ds.X, final, ctx=ctx)
                m = test_metrics(pred, test_ds.y)
                rec.test_rmse, rec.test_llh = m.rmse, m.mean_loglik
                if options.keep_traces:
                    rec.trace = trace
                result.runs.append(rec)
            except NumericalError as e:
                raise NumericalError(f"split {split}, config {entry.label}: {e}") from e
    for entry in grid:
        recs = [r for r in result.runs if r.label == entry.label]
        result.summaries[entry.label] = LabelSummary(
            _aggregate([r.test_rmse for r in recs]), _aggregate([r.test_llh for r in recs]),
            _aggregate([r.total_runtime_seconds for r in recs]),
            _aggregate([r.solver_runtime_seconds for r in recs]))
    for kind in ("cg", "ap", "sgd"):
        cold, warm = result.summaries.get(f"{kind}/cold"), result.summaries.get(f"{kind}/warm")
        if cold is not None and warm is not None and warm.total_runtime.mean > 0.0:
            result.speed_up[kind] = cold.total_runtime.mean / warm.total_runtime.mean
    return result


def grid_search_sgd_lr(ds: Dataset, candidate_lrs: Sequence[float], budget_steps: int, base: TrainConfig,
                       device: int = 0, ctx: Optional[Context] = None) -> float:
    """experiment.cpp:133-168: `budget_steps` SGD steps per candidate at the
    initial hyperparameters on rhs = y; the smallest exact relative residual
    wins; diverging candidates (NumericalError) are skipped, and if all
    diverge the error lists them."""
    if len(candidate_lrs) < 2:
        raise ValueError("grid_search_sgd_lr: need at least 2 candidates")
    if budget_steps < 1:
        raise ValueError("grid_search_sgd_lr: budget must be >= 1")
    hyper = Hyperparameters.constant_constrained(ds.d, base.init_constrained, base.transform)
    op = KernelOperator(np.asarray(ds.X, dtype=np.float32), hyper, device, ctx)
    rhs = np.asarray(ds.y, dtype=np.float32).reshape(-1, 1)
    best_lr, best_res = 0.0, float("inf")
    diverged = []
    for lr in candidate_lrs:
        cfg = dataclasses.replace(base.solver, kind="sgd", learning_rate=float(lr), max_iterations=int(budget_steps),
                                  tol_mean=1e-12, tol_samples=1e-12,  # run the full budget
                                  seed=derive_seed(base.seed, 0x9f1d))
        try:
            st = solve(op, rhs, cfg)
            res = float(st.per_column_relative_residual[0])
            if res < best_res:
                best_res, best_lr = res, float(lr)
        except NumericalError:
            diverged.append("%f" % lr)
    if best_res == float("inf"):
        raise NumericalError("grid_search_sgd_lr: all candidates diverged: " + ", ".join(diverged))
    return best_lr
