"""Kernel + step time of one H.V engine at config 1 (CUDA events on the context
stream; kernel time from the library's own events).  usage: diag_f16_time.py impl"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = sys.argv[1]
n, d, s = (int(a) for a in (sys.argv[2:5] if len(sys.argv) > 4 else (13500, 26, 65)))
p = datasets.config1(n=n, d=d, s=s)
ctx = wg.Context(0, hv_impl=impl)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
st = torch.cuda.ExternalStream(ctx.stream)
Vt = torch.from_numpy(np.ascontiguousarray(p.V.T)).cuda()
o = torch.empty_like(Vt)
with torch.cuda.stream(st):
    for _ in range(3):
        ctx.hv_device(Vt.data_ptr(), n, s, o.data_ptr(), n)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    a.record(st)
    for _ in range(20):
        ctx.hv_device(Vt.data_ptr(), n, s, o.data_ptr(), n)
    b.record(st)
    b.synchronize()
ms = a.elapsed_time(b) / 20
kms, kl = ctx.profile_read()
print(f"{impl} n={n} d={d} s={s} step {ms:.4f} ms, kernel {kms / max(kl, 1):.4f} ms, {n * n / ms * 1e3:.3e} entries/s")
