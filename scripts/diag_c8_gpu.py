"""Acceptance C7/C8 benchmark on the device: the full warm/cold gap table."""
import dataclasses
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import experiment as ex  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from test_gpu_acceptance import dense_metrics, tail_iterations, KINDS  # noqa: E402

ctx = wg.Context(0)
X, y = orc.synthesize(2223, 26, 1.0, 1.0, 0.5, 4242)
full = ex.Dataset("c", X, y)
base = wg.TrainConfig(steps=50, num_probes=16, solver=wg.SolverConfig(tol_mean=0.01, tol_samples=0.1, block_size=250,
                                                                       minibatch_size=1000, max_iterations=100000))
first_train, _ = ex.split_standardize(full, 0.9, wg.derive_seed(0, 0x3711700))
sgd_probe = dataclasses.replace(base, solver=dataclasses.replace(base.solver, kind="sgd"))
lr = ex.grid_search_sgd_lr(first_train, [2, 4, 8, 16], 60, sgd_probe, ctx=ctx)
base = dataclasses.replace(base, solver=dataclasses.replace(base.solver, learning_rate=lr))
res = ex.run_experiment(full, ex.paired_grid(list(KINDS), base), ex.ExperimentOptions(splits=5, seed=0,
                                                                                    keep_traces=False), ctx=ctx)
print("sgd lr", lr, "speed_up", res.speed_up)
for kind in KINDS:
    for split in range(5):
        recs = {r.mode: r for r in res.runs if r.split_index == split and r.solver == kind}
        w, c = recs["warm"], recs["cold"]
        mw = dense_metrics(full, w.split_seed, w.final_constrained)
        mc = dense_metrics(full, c.split_seed, c.final_constrained)
        print("%s %d ratio %.2f | rmse w %.6f c %.6f gap %.5f | llh gap %.4f | final w %s c %s" % (
            kind, split, tail_iterations(w) / tail_iterations(c), mw.rmse, mc.rmse, abs(mw.rmse - mc.rmse),
            abs(mw.mean_loglik - mc.mean_loglik), np.round(w.final_constrained[-3:], 5),
            np.round(c.final_constrained[-3:], 5)), flush=True)
