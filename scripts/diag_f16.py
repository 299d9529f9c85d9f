"""fp16x3 K.V engine (tc_f16) vs 3xTF32 (tc) vs SIMT: accuracy against the fp64
oracle (relative Frobenius + worst column) on config 1 and on columns with
extreme scales, plus kernel timing.  usage: diag_f16.py [n] [d] [s]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 13500
d = int(sys.argv[2]) if len(sys.argv) > 2 else 26
s = int(sys.argv[3]) if len(sys.argv) > 3 else 65
p = datasets.config1(n=n, d=d, s=s)
V = p.V.copy()
# extreme column scales: the fp16 planes must follow any column magnitude
scales = np.ones(s)
scales[1], scales[2], scales[3], scales[4] = 1e-30, 1e-8, 1e8, 1e30
V[:, 5] = 0.0
V[:, 6] = 0.0
V[7, 6] = 3.0
V[:, 7] = np.linspace(-1e-20, 1e3, n)  # wide dynamic range inside one column
V = (V * scales[None, :]).astype(np.float32)
ref = orc.hv(p.X, p.lengthscales, p.signal, p.noise, V.astype(np.float64))
for impl in ("tc", "tc_f16", "simt"):
    ctx = wg.Context(0, hv_impl=impl)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    out = ctx.hv(V)
    colerr = np.linalg.norm(out - ref, axis=0) / np.maximum(np.linalg.norm(ref, axis=0), 1e-300)
    base = [c for c in range(s) if c not in (1, 2, 3, 4, 5, 6, 7)]
    fro = np.linalg.norm(out[:, base] - ref[:, base]) / np.linalg.norm(ref[:, base])
    entry = np.max(np.abs(out[:, base] - ref[:, base])) / np.max(np.abs(ref[:, base]))
    print(f"{impl:7s} fro(regular cols)={fro:.3e} max-abs/max={entry:.3e} worst col={colerr.max():.3e} "
          f"scaled cols 1e-30,1e-8,1e8,1e30: {colerr[1]:.2e} {colerr[2]:.2e} {colerr[3]:.2e} {colerr[4]:.2e} "
          f"zero col max|out|={np.abs(out[:, 5]).max():.1e} single={colerr[6]:.2e} ramp={colerr[7]:.2e}",
          flush=True)
    # timing on device buffers
    st = torch.cuda.ExternalStream(ctx.stream)
    Vt = torch.from_numpy(np.ascontiguousarray(p.V.T)).cuda()
    o = torch.empty_like(Vt)
    with torch.cuda.stream(st):
        for _ in range(3):
            ctx.hv_device(Vt.data_ptr(), n, s, o.data_ptr(), n)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if impl != "simt":
            ctx.profile(True)
        a.record(st)
        for _ in range(20):
            ctx.hv_device(Vt.data_ptr(), n, s, o.data_ptr(), n)
        b.record(st)
        b.synchronize()
    ms = a.elapsed_time(b) / 20
    kms, kl = ctx.profile_read() if impl != "simt" else (ms * 20, 20)
    print(f"{impl:7s} step {ms:.4f} ms, kernel {kms / max(kl, 1):.4f} ms, {n * n / ms * 1e3:.3e} entries/s", flush=True)
    ctx.close()
