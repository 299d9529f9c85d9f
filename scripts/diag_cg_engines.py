"""fp64 CG iteration counts on fixed systems (config 2's points, several
noise levels) for the operator engine selected by WGP_HV64_ENGINE: does the
int8-slice engine's ~1e-12 nonlinearity cost iterations?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

q = datasets.config2()
ctx = wg.Context(0)
ctx.set_data(q.X)
rhs = np.random.default_rng(0).standard_normal((q.X.shape[0], 65)).astype(np.float32)
out = []
for sig in (0.5, 0.2, 0.1, 0.05):
    ctx.set_hyper([*q.lengthscales, q.signal, sig])
    for tol in (1e-2, 1e-4):
        st = ctx.solve(rhs, wg.SolverConfig(kind="cg", tol_mean=tol, tol_samples=tol, max_iterations=5000))
        out.append((sig, tol, st.iterations_used))
print(os.environ.get("WGP_HV64_ENGINE", "i8"), out)
