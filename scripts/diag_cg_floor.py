"""CG at a tolerance below the fp32 floor: exact residual vs iteration cap."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(11)
X = rng.standard_normal((1500, 4)).astype(np.float32)
y = (np.sin(X[:, 0]) + 0.5 * X[:, 1] + 0.1 * rng.standard_normal(1500)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.2, 0.9, 1.5, 2.0, 1.1, 0.3])
for cap in (100, 200, 250, 300, 350, 400, 500, 700, 1000, 2000):
    st = ctx.solve(y.reshape(-1, 1), wg.SolverConfig(kind="cg", tol_mean=1e-8, tol_samples=1e-8, max_iterations=cap))
    print(f"cap {cap}: rel {st.per_column_relative_residual[0]:.3e} |x| {np.abs(st.solutions).max():.3e}", flush=True)
