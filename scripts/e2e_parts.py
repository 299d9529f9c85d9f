"""Where the e2e H.V step goes (config 1): pinned H2D of V, device H.V, D2H of the result (dev timing)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config1()
n, s = p.X.shape[0], 65
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
st = torch.cuda.ExternalStream(ctx.stream)
Vh = torch.from_numpy(np.asfortranarray(p.V).T.copy()).pin_memory()
outh = torch.empty((s, n), pin_memory=True)
Vd = torch.empty((s, n), device="cuda")
od = torch.empty((s, n), device="cuda")
lib = wg.load()


def t(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


with torch.cuda.stream(st):
    print("h2d  %.3f ms" % t(lambda: Vd.copy_(Vh, non_blocking=True)))
    print("d2h  %.3f ms" % t(lambda: outh.copy_(od, non_blocking=True)))
    print("hv   %.3f ms" % t(lambda: ctx.hv_device(Vd.data_ptr(), n, s, od.data_ptr(), n)))
    print("e2e  %.3f ms" % t(lambda: lib.wgp_hv(ctx._h, C.c_void_p(Vh.data_ptr()), s, C.c_void_p(outh.data_ptr()))))
os._exit(0)  # skip teardown: torch would record events on the (destroyed) context stream
