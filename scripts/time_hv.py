"""Time the fused H.V (device pointers, CUDA events on the context stream).
usage: time_hv.py [impl] [n] [d] [s] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = sys.argv[1] if len(sys.argv) > 1 else "tc"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 13500
d = int(sys.argv[3]) if len(sys.argv) > 3 else 26
s = int(sys.argv[4]) if len(sys.argv) > 4 else 65
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
p = datasets.config1(n=n, d=d, s=s)
ctx = wg.Context(0, hv_impl=impl)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
st = torch.cuda.ExternalStream(ctx.stream)
Vt = torch.from_numpy(np.ascontiguousarray(p.V.T)).cuda()
out = torch.empty_like(Vt)
with torch.cuda.stream(st):
    for _ in range(3):
        ctx.hv_device(Vt.data_ptr(), n, s, out.data_ptr(), n)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = impl in ("tc", "tc_f16") and not os.environ.get("TIME_HV_NOPROF")
    if prof:
        ctx.profile(True)
    a.record(st)
    for _ in range(reps):
        ctx.hv_device(Vt.data_ptr(), n, s, out.data_ptr(), n)
    b.record(st)
    b.synchronize()
ms = a.elapsed_time(b) / reps
kms, kl = ctx.profile_read() if prof else (ms * reps, reps)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("WGP_TC"))
print(f"impl={impl} n={n} d={d} s={s} [{env}] ms={ms:.4f} kernel_ms={kms / max(kl, 1):.4f} "
      f"entries/s={n * n / ms * 1e3:.3e}")
