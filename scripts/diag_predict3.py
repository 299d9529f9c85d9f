"""Does predict's setup disturb the context's solves?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(11)
X = rng.standard_normal((1500, 4)).astype(np.float32)
Xt = rng.standard_normal((300, 4)).astype(np.float32)
y = (np.sin(X[:, 0]) + 0.5 * X[:, 1] + 0.1 * rng.standard_normal(1500)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.2, 0.9, 1.5, 2.0, 1.1, 0.3])
cfg = wg.SolverConfig(kind="cg", tol_mean=1e-8, tol_samples=1e-8, max_iterations=2000)
st = ctx.solve(y.reshape(-1, 1), cfg)
print("public before", st.per_column_relative_residual[0], flush=True)
pred = ctx.predict(Xt, y, cfg)
print("means", pred.means[:3], flush=True)
st = ctx.solve(y.reshape(-1, 1), cfg)
print("public after", st.per_column_relative_residual[0], flush=True)
pred = ctx.predict(Xt[:5], y, cfg)
print("means (5 test points)", pred.means[:3], flush=True)
