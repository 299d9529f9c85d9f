"""Diagnostics of the alpha solve in predict: CG at several tolerances."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(11)
X = rng.standard_normal((1500, 4)).astype(np.float32)
y = (np.sin(X[:, 0]) + 0.5 * X[:, 1] + 0.1 * rng.standard_normal(1500)).astype(np.float32)
ls, sf, sig = np.array([1.2, 0.9, 1.5, 2.0]), 1.1, 0.3
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([*ls, sf, sig])
for tol in (1e-3, 1e-4, 1e-5, 1e-6):
    st = ctx.solve(y.reshape(-1, 1), wg.SolverConfig(kind="cg", tol_mean=tol, tol_samples=tol, max_iterations=5000))
    print(f"tol {tol:g}: its {st.iterations_used}, rel {st.per_column_relative_residual}, |x| {np.abs(st.solutions).max():.3e}")

from oracle import dense_ref  # noqa: E402
Xt = rng.standard_normal((300, 4)).astype(np.float32)
cfg = wg.SolverConfig(kind="cg", tol_mean=1e-5, tol_samples=1e-5, max_iterations=5000)
pred = ctx.predict(Xt, y, cfg)
means, var, nv = dense_ref.predict(X, y, Xt, ls, sf, sig)
print("means gpu", pred.means[:4], "oracle", means[:4])
print("var gpu", pred.variances[:4], "oracle", var[:4])
alpha = ctx.solve(y.reshape(-1, 1), cfg).solutions[:, 0].astype(np.float64)
r = np.sqrt((((X[:, None, :].astype(np.float64) - Xt[None, :, :]) / ls) ** 2).sum(-1))
Ks = sf * sf * (1 + np.sqrt(3) * r) * np.exp(-np.sqrt(3) * r)
print("K*^T alpha (numpy, gpu alpha)", (Ks.T @ alpha)[:4])
