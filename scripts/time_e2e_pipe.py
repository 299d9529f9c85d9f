"""wgp_hv end to end at config 1 (pinned host V in, host result out), the
pipeline modes interleaved in one process (WGP_HV_PIPE is read per call):
median ms per mode over rounds of 20 calls each."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = sys.argv[1] if len(sys.argv) > 1 else "tc_f16"
modes = sys.argv[2].split(";") if len(sys.argv) > 2 else ["", "1"]
p = datasets.config1()
n, s = p.X.shape[0], 65
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
ctx.set_hv_impl(impl)
st = torch.cuda.ExternalStream(ctx.stream)
Vh = torch.from_numpy(np.asfortranarray(p.V).T.copy()).pin_memory()
outh = torch.empty((s, n), pin_memory=True)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = wg.load()
if os.environ.get("E2E_NVML"):  # the bench's clock sampler beside the calls (every E2E_NVML ms)
    import threading

    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    period = float(os.environ["E2E_NVML"]) / 1e3

    def sample():
        while True:
            pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)
            time.sleep(period)

    threading.Thread(target=sample, daemon=True).start()
ts = {m: [] for m in modes}
res = {}
for rnd in range(6):
    for mode in modes:
        os.environ["WGP_HV_PIPE"] = mode
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
                ts[mode].append(a.elapsed_time(b))
        res[mode] = outh.numpy().T.astype(np.float64)
one = res.get("1", next(iter(res.values())))
for mode in modes:
    t = np.array(ts[mode])
    err = np.linalg.norm(res[mode] - one) / np.linalg.norm(one)
    print(f"impl={impl} pipe={mode or 'model'!s:8} e2e median {np.median(t):.4f} mean {t.mean():.4f} p10 {np.percentile(t, 10):.4f}"
          f" ms  entries/s {n * n / (np.median(t) / 1e3):.3e}  rel vs one launch {err:.1e}")
os._exit(0)
