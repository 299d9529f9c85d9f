"""One CG solve per fresh context (tol below the fp32 floor) at several caps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(11)
X = rng.standard_normal((1500, 4)).astype(np.float32)
y = (np.sin(X[:, 0]) + 0.5 * X[:, 1] + 0.1 * rng.standard_normal(1500)).astype(np.float32)
for cap in (60, 100, 150, 200, 300, 2000):
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([1.2, 0.9, 1.5, 2.0, 1.1, 0.3])
    st = ctx.solve(y.reshape(-1, 1), wg.SolverConfig(kind="cg", tol_mean=1e-8, tol_samples=1e-8, max_iterations=cap))
    print(f"fresh cap {cap}: rel {st.per_column_relative_residual[0]:.3e}", flush=True)
    ctx.close()
