"""wgp_hv end to end at config 1 (pinned host buffers), upload modes interleaved in one
process (WGP_HV_UPLOAD is read per call): copy engine, zero-copy split, auto.  Prints
per-round medians so the host link's slow / fast states show."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = sys.argv[1] if len(sys.argv) > 1 else "tc_f16"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = datasets.config1()
n, s = p.X.shape[0], 65
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
ctx.set_hv_impl(impl)
st = torch.cuda.ExternalStream(ctx.stream)
Vh = torch.from_numpy(np.asfortranarray(p.V).T.copy()).pin_memory()
outh = torch.empty((s, n), pin_memory=True)
outs = {}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = wg.load()
var = sys.argv[3] if len(sys.argv) > 3 else "WGP_HV_UPLOAD"  # or WGP_HV_DOWNLOAD (modes ce, zc)
modes = ["ce", "zc", "auto"] if var == "WGP_HV_UPLOAD" else ["ce", "zc"]
ts = {m: [] for m in modes}
for rnd in range(rounds):
    line = []
    for mode in modes:
        os.environ[var] = mode
        t = []
        for i in range(22):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            rc = lib.wgp_hv(ctx._h, C.c_void_p(Vh.data_ptr()), s, C.c_void_p(outh.data_ptr()))
            b.record(st)
            b.synchronize()
            assert rc == 0
            if i >= 2:
                t.append(a.elapsed_time(b))
        ts[mode] += t
        outs[mode] = outh.numpy().copy()
        line.append(f"{mode} {np.median(t):.3f}")
    print(f"round {rnd}: " + "  ".join(line) + " ms")
print("results bitwise equal across modes:", all(np.array_equal(outs[modes[0]], outs[m]) for m in modes))
for mode in modes:
    t = np.array(ts[mode])
    print(f"impl={impl} {var}={mode:5s} e2e median {np.median(t):.4f} mean {t.mean():.4f} p10 {np.percentile(t, 10):.4f} "
          f"p90 {np.percentile(t, 90):.4f} ms  entries/s (mean) {n * n / (t.mean() / 1e3):.3e}")
os._exit(0)
