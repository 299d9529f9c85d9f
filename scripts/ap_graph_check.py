"""AP with the epoch graph vs eager (WGP_NO_GRAPHS=1, read once per process):
solutions must agree bitwise.  usage: ap_graph_check.py [out.npy]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(4)
n, d, s = 5000, 5, 9
X = rng.standard_normal((n, d)).astype(np.float32)
B = rng.standard_normal((n, s)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.0] * d + [1.0, 0.3])
cfg = wg.SolverConfig(kind="ap", tol_mean=1e-4, tol_samples=1e-4, max_iterations=12, block_size=700)
st = ctx.solve(B, cfg)
st2 = ctx.solve(B, cfg)  # second solve: cached graph
assert np.array_equal(st.solutions, st2.solutions)
np.save(sys.argv[1], st.solutions)
print("epochs", st.iterations_used, "res", st.per_column_relative_residual[0])
