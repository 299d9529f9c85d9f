"""AP solve on a config-3-like problem (d=3 uniform inputs), for profiling."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(0)
X = rng.uniform(size=(n, 3)).astype(np.float32)
B = rng.standard_normal((n, 65)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.0, 1.0, 1.0, 1.0, 0.5])
cfg = wg.SolverConfig(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=epochs, block_size=1000)
ctx.solve(B, wg.SolverConfig(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=1, block_size=1000))
t = time.time()
st = ctx.solve(B, cfg)
print(f"n={n} AP {st.iterations_used} epochs: {time.time() - t:.3f} s wall, residual {st.per_column_relative_residual[0]:.3e}")
