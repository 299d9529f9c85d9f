"""Host cost per fused H.V call: many tiny device-pointer calls (GPU time
negligible) timed on the host, for the tc and simt engines."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

n, s, reps = 512, 8, 2000
X = np.random.default_rng(0).standard_normal((n, 4)).astype(np.float32)
for impl in ("tc", "simt"):
    ctx = wg.Context(0, hv_impl=impl)
    ctx.set_data(X)
    ctx.set_hyper([1.0] * 4 + [1.0, 0.5])
    V = torch.randn(s, n, device="cuda")
    out = torch.empty_like(V)
    for _ in range(20):
        ctx.hv_device(V.data_ptr(), n, s, out.data_ptr(), n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.hv_device(V.data_ptr(), n, s, out.data_ptr(), n)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{impl}: enqueue {1e6 * (t1 - t0) / reps:.1f} us/call, total {1e6 * (t2 - t0) / reps:.1f} us/call")
    ctx.close()
