"""A few AP epochs at config 3 (n = 391,386, b = 1000) for a launch list (dev profiling)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = datasets.config3()
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([1.0] * 3 + [1.0, 0.5])
B = np.random.default_rng(0).standard_normal((p.X.shape[0], 65)).astype(np.float32)
st = ctx.solve(B, wg.SolverConfig(kind="ap", tol_mean=1e-6, tol_samples=1e-6, max_iterations=epochs, block_size=1000))
print("epochs", st.iterations_used)
