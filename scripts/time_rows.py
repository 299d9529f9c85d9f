"""Time an H.V restricted to a row block (AP's left-looking residual shape)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 391386
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
rng = np.random.default_rng(0)
X = rng.uniform(size=(n, 3)).astype(np.float32)
ctx = wg.Context(0)
ctx.set_data(X)
ctx.set_hyper([1.0, 1.0, 1.0, 1.0, 0.5])
ctx.set_rows(5000, 5000 + rows)
st = torch.cuda.ExternalStream(ctx.stream)
V = torch.randn(65, n, device="cuda")
out = torch.empty(65, rows, device="cuda")
with torch.cuda.stream(st):
    for _ in range(3):
        ctx.hv_device(V.data_ptr(), n, 65, out.data_ptr(), rows)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    a.record(st)
    for _ in range(20):
        ctx.hv_device(V.data_ptr(), n, 65, out.data_ptr(), rows)
    b.record(st)
    b.synchronize()
kms, kl = ctx.profile_read()
ms = a.elapsed_time(b) / 20
print(f"n={n} rows={rows}: {ms:.3f} ms per call, kernel {kms / max(kl, 1):.3f} ms, {rows * n / ms * 1e3:.3e} entries/s")
