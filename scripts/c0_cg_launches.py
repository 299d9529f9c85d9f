"""One config-0 CG solve (n=2048, s=17) for a launch list: which kernels make up an iteration."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config0()
ctx = wg.Context(0, hv_impl=os.environ.get("HV_IMPL", "tc"))
ctx.set_data(p.X)
ctx.set_hyper([1.0] * 8 + [1.0, 0.5])
rhs = np.random.default_rng(0).standard_normal((p.X.shape[0], 17)).astype(np.float32)
cfg = wg.SolverConfig(kind="cg", tol_mean=1e-6, tol_samples=1e-6, max_iterations=40)
ctx.solve(rhs, cfg)
st = ctx.solve(rhs, cfg)
print("iterations", st.iterations_used)
