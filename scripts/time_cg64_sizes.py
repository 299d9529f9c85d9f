"""fp64 CG iteration time vs n (config-2-shaped data, s = 65) for the operator
engine from WGP_HV64_ENGINE (the crossover that sets hv_f64's engine choice)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

ctx = wg.Context(0)
st = torch.cuda.ExternalStream(ctx.stream)
res = []
for n in (4096, 8192, 16384, 24576):
    q = datasets.config2(n=n)
    ctx.set_data(q.X)
    ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
    rhs = np.random.default_rng(0).standard_normal((n, 65)).astype(np.float32)
    t = []
    for its in (10, 40):
        cfg = wg.SolverConfig(kind="cg", tol_mean=1e-14, tol_samples=1e-14, max_iterations=its)
        ctx.solve(rhs, cfg)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.solve(rhs, cfg)
        b.record(st)
        b.synchronize()
        t.append(a.elapsed_time(b))
    res.append((n, round(1e3 * (t[1] - t[0]) / 30, 1)))
print(os.environ.get("WGP_HV64_ENGINE", "default"), "us per iteration:", res)
