"""Device time per fp64 CG iteration (default config 2, n = 41,157, s = 65): ~ the
fp64 operator + the fused vector kernel (dev timing, CUDA events).
usage: time_cg64_c2.py [config] [s]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = int(sys.argv[2]) if len(sys.argv) > 2 else 65
its_pair = (2, 4) if name == "c4" else (10, 40)
q = datasets.CONFIGS[name]()
ctx = wg.Context(0)
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
rhs = np.random.default_rng(0).standard_normal((q.X.shape[0], s)).astype(np.float32)
st = torch.cuda.ExternalStream(ctx.stream)
for its in its_pair:
    cfg = wg.SolverConfig(kind="cg", tol_mean=1e-14, tol_samples=1e-14, max_iterations=its)
    ctx.solve(rhs, cfg)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    r = ctx.solve(rhs, cfg)
    b.record(st)
    b.synchronize()
    print(f"its={r.iterations_used} ms={a.elapsed_time(b):.2f}")
