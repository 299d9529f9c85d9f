"""Wall time of one gradient contraction (wgp_grad: prep + kernel + finalize
+ the O(n s) dots) at a BASELINE config, tensor-core vs CUDA-core engine.
Usage: python scripts/time_grad.py [c3|c2|c0] [reps]"""
import sys
import time

import numpy as np

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import datasets

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = datasets.CONFIGS[cfg]()
n, d = p.X.shape
s = 64 if cfg != "c0" else 16
rng = np.random.default_rng(1)
vy = rng.standard_normal(n).astype(np.float32)
L = np.asfortranarray(rng.standard_normal((n, s)).astype(np.float32))
R = np.asfortranarray(rng.standard_normal((n, s)).astype(np.float32))
ctx = wg.Context(0)
ctx.set_data(p.X)
raw = np.log(np.expm1(np.array([*p.lengthscales, p.signal, p.noise])))
for impl in ("tc", "simt"):
    ctx.set_hv_impl(impl)
    ga, gb = ctx.grad("softplus", raw, vy, L, R, 0.5 / s)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ga, gb = ctx.grad("softplus", raw, vy, L, R, 0.5 / s)
        ts.append(time.perf_counter() - t0)
    print(f"{cfg} n={n} d={d} s={s} {impl}: {min(ts)*1e3:.1f} ms  (n^2/t = {n*n/min(ts):.3e} entries/s)"
          f"  a[0]={ga[0]:.9e} b[0]={gb[0]:.9e}", flush=True)
