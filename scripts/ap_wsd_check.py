"""Writes (AP solutions, residuals, iterations; warm-start distances of a short
training run) to argv[1] -- run under different WGP_AP_EXACT_EVERY /
WGP_WSD_PRODUCT settings by tests/test_gpu_parity.py."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

rng = np.random.default_rng(4)
X = rng.standard_normal((3000, 4)).astype(np.float32)
rhs = rng.standard_normal((3000, 9)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.1, 0.9, 1.3, 1.2, 1.0, 0.2])
st = ctx.solve(rhs, wg.SolverConfig(kind="ap", block_size=250, tol_mean=1e-4, tol_samples=1e-4, max_iterations=60))
p = datasets.config0(n=1500, d=5)
ctx.set_data(p.X)
w = []
for kind in ("cg", "ap"):
    tr = ctx.train(p.y, wg.TrainConfig(steps=4, num_probes=6, solver=wg.SolverConfig(kind=kind, block_size=300,
                                                                                      tol_mean=1e-3, tol_samples=1e-3)))
    w.append([r.warm_start_distance for r in tr.steps])
np.savez(sys.argv[1], x=st.solutions, rel=st.per_column_relative_residual, it=st.iterations_used, wsd=np.array(w))
