"""SGD (or CG) solution after a fixed number of steps (no convergence), saved for a
bitwise comparison between library builds.  usage: sgd_bitwise.py out.npy [sgd|cg]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(6)
n, d, s = 6000, 6, 9
X = rng.standard_normal((n, d)).astype(np.float32)
B = rng.standard_normal((n, s)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.0] * d + [1.0, 0.4])
kind = sys.argv[2] if len(sys.argv) > 2 else "sgd"
cfg = wg.SolverConfig(kind=kind, tol_mean=1e-12, tol_samples=1e-12, max_iterations=203 if kind == "sgd" else 37,
                      minibatch_size=500, momentum=0.9, learning_rate=3.0, seed=11)
st = ctx.solve(B, cfg)
np.save(sys.argv[1], st.solutions)
print("steps", st.iterations_used)
