"""CG solutions at config-0 size (fp64 and fp32 CG, 2 solves, the second warm)
for the bitwise comparison of the CG iteration paths (cg_fused with
the H.V reduction folded in / after it / three kernels), selected by WGP_CG_NO_FOLD /
WGP_CG_NO_FUSED (read once per process).  usage: cg_path_check.py OUT.npy"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config0()
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([2.6] * 8 + [1.14, 0.1])  # late, ill-conditioned hyperparameters
rhs = np.random.default_rng(3).standard_normal((p.X.shape[0], 17)).astype(np.float32)
res = []
for prec in ("f64", "f32"):
    ctx.set_cg_precision(prec)
    cfg = wg.SolverConfig(kind="cg", tol_mean=1e-3, tol_samples=1e-3, max_iterations=400)
    st = ctx.solve(rhs, cfg)
    st2 = ctx.solve(rhs * 1.01, cfg, init=st.solutions)
    res += [st.solutions.ravel(), st2.solutions.ravel(), np.array([st.iterations_used, st2.iterations_used], float)]
np.save(sys.argv[1], np.concatenate(res))
