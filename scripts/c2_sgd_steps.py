"""64 config-2 SGD steps (minibatch 1000, s = 65) for a launch-list profile,
and their wall time per step without a profiler."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config2()
n = p.X.shape[0]
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([1.0] * p.X.shape[1] + [1.0, 0.5])
B = np.random.default_rng(0).standard_normal((n, 65)).astype(np.float32)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for rep in range(2):
    cfg = wg.SolverConfig(kind="sgd", tol_mean=1e-12, tol_samples=1e-12, max_iterations=steps, minibatch_size=1000,
                          momentum=0.9, learning_rate=10.0)
    t0 = time.perf_counter()
    ctx.solve(B, cfg)
    print(f"{steps} SGD steps: {(time.perf_counter() - t0) * 1e3 / steps:.3f} ms per step (wall, incl. solve setup)")
