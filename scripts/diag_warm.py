"""Warm-start diagnostics for the exact-warm-start solver test."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2405_18328_b200 as wg  # noqa: E402
from test_gpu_parity import kernel_problem  # noqa: E402
from oracle import oracle as orc  # noqa: E402

X, ls, sf, sig, rhs = kernel_problem(700, 3, 4, seed=12)
for impl in ("tc", "simt"):
    ctx = wg.Context(0, hv_impl=impl)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    cfg = wg.SolverConfig(kind="cg", tol_mean=1e-3, tol_samples=1e-3, max_iterations=50000)
    a = ctx.solve(rhs, cfg)
    tight = wg.SolverConfig(kind="cg", tol_mean=1e-6, tol_samples=1e-6, max_iterations=5000)
    e = ctx.solve(rhs, tight)
    for name, st in (("a", a), ("tight", e)):
        hx = orc.hv(X, ls, sf, sig, st.solutions)
        r = np.linalg.norm(rhs - hx, axis=0) / np.linalg.norm(rhs, axis=0)
        print(impl, name, "its", st.iterations_used, "reported", st.per_column_relative_residual,
              "oracle-exact", r)
    w = ctx.solve(rhs, cfg, init=e.solutions)
    print(impl, "warm from tight: its", w.iterations_used, w.per_column_relative_residual)
    w = ctx.solve(rhs, cfg, init=a.solutions)
    print(impl, "warm from a: its", w.iterations_used, w.per_column_relative_residual)
    ctx.close()
