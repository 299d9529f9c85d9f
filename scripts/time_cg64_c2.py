"""Device time per fp64 CG iteration at config 2 (n = 41,157, s = 65): ~ the
hv_f64 operator + the fused vector kernel (dev timing, CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

q = datasets.config2()
ctx = wg.Context(0)
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
rhs = np.random.default_rng(0).standard_normal((q.X.shape[0], 65)).astype(np.float32)
st = torch.cuda.ExternalStream(ctx.stream)
for its in (10, 40):
    cfg = wg.SolverConfig(kind="cg", tol_mean=1e-14, tol_samples=1e-14, max_iterations=its)
    ctx.solve(rhs, cfg)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    r = ctx.solve(rhs, cfg)
    b.record(st)
    b.synchronize()
    print(f"its={r.iterations_used} ms={a.elapsed_time(b):.2f}")
