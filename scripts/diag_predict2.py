"""predict on a fresh context at tol 1e-6 (the failing test's setup)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import dense_ref  # noqa: E402

rng = np.random.default_rng(11)
X = rng.standard_normal((1500, 4)).astype(np.float32)
Xt = rng.standard_normal((300, 4)).astype(np.float32)
y = (np.sin(X[:, 0]) + 0.5 * X[:, 1] + 0.1 * rng.standard_normal(1500)).astype(np.float32)
ls, sf, sig = np.array([1.2, 0.9, 1.5, 2.0]), 1.1, 0.3
means, var, nv = dense_ref.predict(X, y, Xt, ls, sf, sig)
for tol in (1e-6, 1e-5):
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    cfg = wg.SolverConfig(kind="cg", tol_mean=tol, tol_samples=tol, max_iterations=5000)
    pred = ctx.predict(Xt, y, cfg)
    print(tol, "means err", np.max(np.abs(pred.means - means)), "var err", np.max(np.abs(pred.variances - var)))
    ctx.close()
