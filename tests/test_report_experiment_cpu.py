"""Report layer (report.cpp) and experiment-driver host logic
(experiment.cpp, dataset.cpp:109-166) on the CPU: no device work."""
import json
import math

import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import experiment as ex
from paper_2405_18328_b200 import report as rp
from oracle import oracle as orc


def fake_trace(steps=3, p=4, s=3):
    rng = np.random.default_rng(1)
    recs = [wg.StepRecord(t + 1, rng.standard_normal(p), np.abs(rng.standard_normal(p)), rng.standard_normal(p),
                          int(rng.integers(1, 50)), float(rng.uniform(1, 9)), float(rng.uniform(10, 20)),
                          rng.uniform(0, 0.01, s), float(rng.uniform()), 0)
            for t in range(steps)]
    return wg.OptTrace(recs)


def fake_result():
    r = ex.ExperimentResult("synthetic", 2, 0.9)
    for split in range(2):
        for label, mode in (("cg/cold", "cold"), ("cg/warm", "warm")):
            rec = ex.RunRecord(label, "cg", mode, split, 11 + split, 21 + split, 0.1 * (split + 1) + 1e-17,
                               -1.0 / 3.0, 2.0 + split + (1 if mode == "cold" else 0), 1.5 + split,
                               [3, 4, 5], np.array([1.0, 2.0 / 3.0, 0.5]), fake_trace())
            r.runs.append(rec)
    for label in ("cg/cold", "cg/warm"):
        recs = [x for x in r.runs if x.label == label]
        r.summaries[label] = ex.LabelSummary(ex._aggregate([x.test_rmse for x in recs]),
                                             ex._aggregate([x.test_llh for x in recs]),
                                             ex._aggregate([x.total_runtime_seconds for x in recs]),
                                             ex._aggregate([x.solver_runtime_seconds for x in recs]))
    r.speed_up["cg"] = r.summaries["cg/cold"].total_runtime.mean / r.summaries["cg/warm"].total_runtime.mean
    return r


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 5), (17, 0), (1000, 123456789), (4097, 2 ** 63 + 7)])
def test_split_order_matches_oracle_bitwise(n, seed):
    """dataset.cpp:118-124 through the C-ABI (host-only) against the oracle."""
    a = wg.split_order(n, seed)
    b = orc.split_order(n, seed)
    assert np.array_equal(a, b)
    assert np.array_equal(np.sort(a), np.arange(n))


def test_split_standardize_statistics_and_errors():
    rng = np.random.default_rng(3)
    X = rng.normal(5.0, 3.0, size=(101, 3))
    X[:, 2] = 7.0  # constant column: deviation 1 (dataset.cpp:148)
    y = rng.normal(2.0, 4.0, size=101)
    ds = ex.Dataset("toy", X, y)
    tr, te = ex.split_standardize(ds, 0.9, 99)
    assert tr.n == 90 and te.n == 11
    order = wg.split_order(101, 99)
    assert np.allclose(tr.X * tr.feature_stds + tr.feature_means, X[order[:90]])
    assert np.allclose(te.y * te.target_std + te.target_mean, y[order[90:]])
    assert np.allclose(tr.X[:, :2].mean(0), 0.0, atol=1e-12)
    assert np.allclose(tr.X[:, :2].std(0), 1.0)  # population deviation
    assert tr.feature_stds[2] == 1.0 and np.all(tr.X[:, 2] == 0.0)
    assert abs(tr.y.mean()) < 1e-12 and abs(tr.y.std() - 1.0) < 1e-12
    with pytest.raises(ValueError, match="train_fraction must lie in"):
        ex.split_standardize(ds, 1.0, 0)
    with pytest.raises(ValueError, match="empty train or test set"):
        ex.split_standardize(ex.Dataset("t", X[:1], y[:1]), 0.5, 0)


def test_paired_grid_and_aggregate():
    base = wg.TrainConfig(steps=3)
    g = ex.paired_grid(["cg", "ap"], base)
    assert [e.label for e in g] == ["cg/cold", "cg/warm", "ap/cold", "ap/warm"]
    assert [e.config.mode for e in g] == ["cold", "warm", "cold", "warm"]
    assert [e.config.solver.kind for e in g] == ["cg", "cg", "ap", "ap"]
    assert base.solver.kind == "cg" and base.mode == "warm"  # base untouched
    a = ex._aggregate([1.0, 2.0, 4.0])
    assert a.mean == pytest.approx(7 / 3)
    assert a.standard_error == pytest.approx(np.std([1.0, 2.0, 4.0], ddof=1) / math.sqrt(3))
    assert ex._aggregate([5.0]).standard_error == 0.0
    with pytest.raises(ValueError, match="empty config grid"):
        ex.run_experiment(ex.Dataset("t", np.zeros((4, 1)), np.zeros(4)), [])


def test_trace_json_keys_and_wall_time_strip():
    t = fake_trace()
    j = rp.to_json(t)
    keys = {"step", "raw_params", "constrained_params", "gradient", "solver_iterations", "solver_seconds",
            "cumulative_seconds", "per_column_relative_residual", "warm_start_distance"}
    assert [set(s) for s in j["steps"]] == [keys] * 3
    cum = np.cumsum([r.step_ms / 1e3 for r in t.steps])
    assert np.allclose([s["cumulative_seconds"] for s in j["steps"]], cum)
    stripped = rp.strip_wall_time_fields(j)
    assert all("solver_seconds" not in s and "cumulative_seconds" not in s for s in stripped["steps"])
    assert set(rp.wall_time_keys()) == {"solver_seconds", "cumulative_seconds", "total_runtime_seconds",
                                        "solver_runtime_seconds", "speed_up"}


def test_emit_report_json_and_csv_round_trip(tmp_path):
    r = fake_result()
    pj, pc = str(tmp_path / "r.json"), str(tmp_path / "r.csv")
    rp.emit_report(r, pj, "json")
    j = rp.load_json_file(pj)
    assert j == json.loads(json.dumps(rp.to_json(r)))
    assert j["runs"][0]["trace"]["steps"][0]["step"] == 1 and j["speed_up"]["cg"] > 1
    assert open(pj).read().endswith("\n")
    s = rp.strip_wall_time_fields(j)
    assert "speed_up" not in s and "total_runtime_seconds" not in s["runs"][0]
    assert "total_runtime_seconds" not in s["summaries"]["cg/warm"]
    rp.emit_report(r, pc, "csv")
    tab = rp.load_csv_table(pc)
    assert tab.header == rp._CSV_HEADER.split(",")
    assert len(tab.rows) == 4
    for rec, row in zip(r.runs, tab.rows):
        cell = dict(zip(tab.header, row))
        assert float(cell["test_rmse"]) == rec.test_rmse  # 17 digits: bit-exact
        assert float(cell["test_llh"]) == rec.test_llh
        assert int(cell["total_iterations"]) == 12 and cell["mode"] == rec.mode
    with pytest.raises(ValueError, match="unknown report format"):
        rp.emit_report(r, pc, "xml")
    with pytest.raises(rp.IoError):
        rp.emit_report(r, str(tmp_path / "missing" / "x.json"), "json")
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(rp.IoError):
        rp.load_json_file(str(tmp_path / "bad.json"))


def test_parse_config_file(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text("# comment\n  solver = cg  # trailing\n\nsteps=20\r\nname = a b\n")
    assert rp.parse_config_file(str(p)) == {"solver": "cg", "steps": "20", "name": "a b"}
    p.write_text("ok = 1\nbroken line\n")
    with pytest.raises(rp.IoError, match="line 2 is not 'key = value'"):
        rp.parse_config_file(str(p))
    p.write_text(" = 3\n")
    with pytest.raises(rp.IoError, match="line 1 has an empty key"):
        rp.parse_config_file(str(p))
    with pytest.raises(rp.IoError, match="cannot open config file"):
        rp.parse_config_file(str(tmp_path / "nope.cfg"))
