"""Paired warm/cold experiment driver (experiment.cpp) and the report layer
on the device path: seeds shared by paired entries, reruns identical once
wall-time fields are stripped (report.cpp:179-187), the warm run's final
hyperparameters equal to the oracle's training run on the same split."""
import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import experiment as ex
from paper_2405_18328_b200 import report as rp
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def toy(n=700, d=3, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    y = np.sin(2 * X).sum(1) / np.sqrt(d) + 0.1 * rng.standard_normal(n)
    return ex.Dataset("toy", X, y)


def base_config(mod, steps=4):
    return mod.TrainConfig(steps=steps, learning_rate=0.1, num_probes=8, mode="warm", transform="log",
                           estimator="pathwise", rff_features=300, init_noise=0.5, init_constrained=1.0,
                           solver=mod.SolverConfig(kind="cg", tol_mean=1e-4, tol_samples=1e-4,
                                                   max_iterations=3000))


def test_run_experiment_paired_and_deterministic(tmp_path):
    ds = toy()
    grid = ex.paired_grid(["cg"], base_config(wg))
    opts = ex.ExperimentOptions(splits=2, train_fraction=0.9, seed=5)
    ctx = wg.Context(0)
    r1 = ex.run_experiment(ds, grid, opts, ctx=ctx)
    r2 = ex.run_experiment(ds, grid, opts, ctx=ctx)
    assert [(r.label, r.split_index) for r in r1.runs] == [("cg/cold", 0), ("cg/warm", 0), ("cg/cold", 1),
                                                           ("cg/warm", 1)]
    for split in range(2):
        cold, warm = r1.runs[2 * split], r1.runs[2 * split + 1]
        assert cold.split_seed == warm.split_seed == wg.derive_seed(5, 0x3711700 + split)
        assert cold.train_seed == warm.train_seed == wg.derive_seed(5, 0x7ea1 + split)
        assert cold.mode == "cold" and warm.mode == "warm"
        assert np.isfinite(warm.test_rmse) and np.isfinite(warm.test_llh) and warm.test_rmse < 1.0
        assert len(warm.per_step_iterations) == 4 and warm.trace is not None
    assert r1.speed_up["cg"] > 0
    assert set(r1.summaries) == {"cg/cold", "cg/warm"}
    j1, j2 = rp.to_json(r1), rp.to_json(r2)
    assert rp.strip_wall_time_fields(j1) == rp.strip_wall_time_fields(j2)
    rp.emit_report(r1, str(tmp_path / "r.json"), "json")
    rp.emit_report(r1, str(tmp_path / "r.csv"), "csv")
    assert rp.strip_wall_time_fields(rp.load_json_file(str(tmp_path / "r.json"))) == \
        rp.strip_wall_time_fields(j1)
    assert len(rp.load_csv_table(str(tmp_path / "r.csv")).rows) == 4
    # the warm run of split 0 against the oracle's training run on the same split
    tr, _ = ex.split_standardize(ds, 0.9, r1.runs[1].split_seed)
    ocfg = base_config(orc)
    ocfg.seed = r1.runs[1].train_seed
    o = orc.train(tr.X.astype(np.float32).astype(np.float64), tr.y.astype(np.float32).astype(np.float64), ocfg)
    oc = o["constrained_params"][-1]
    assert np.max(np.abs(r1.runs[1].final_constrained - oc) / np.abs(oc)) <= 1e-3


def test_grid_search_sgd_lr():
    tr, _ = ex.split_standardize(toy(500), 0.9, 3)
    base = base_config(wg)
    base.solver = wg.SolverConfig(kind="sgd", minibatch_size=100, momentum=0.9)
    lrs = [0.3, 1.0, 3.0, 1e9]
    best = ex.grid_search_sgd_lr(tr, lrs, 40, base)
    assert best in lrs[:3]
    # the winner has the smallest exact relative residual among the finite candidates
    hyper = wg.Hyperparameters.constant_constrained(tr.d, 1.0, "log")
    op = wg.KernelOperator(tr.X.astype(np.float32), hyper)
    res = {}
    for lr in lrs[:3]:
        cfg = wg.SolverConfig(kind="sgd", learning_rate=lr, max_iterations=40, tol_mean=1e-12, tol_samples=1e-12,
                              minibatch_size=100, momentum=0.9, seed=wg.derive_seed(base.seed, 0x9f1d))
        res[lr] = wg.solve(op, tr.y.astype(np.float32).reshape(-1, 1), cfg).per_column_relative_residual[0]
    assert best == min(res, key=res.get)
    with pytest.raises(wg.NumericalError, match="all candidates diverged"):
        ex.grid_search_sgd_lr(tr, [1e9, 1e10], 40, base)
