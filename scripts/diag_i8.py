"""The fp64 CG operator's engines (hv_f64.cu DMMA vs hv_i8.cu int8 slices):
accuracy against the fp64 oracle, symmetry / linearity, timing.
usage: diag_i8.py OUT.npz   (engine from WGP_HV64_ENGINE: dmma | default i8)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

out = {}
ctx = wg.Context(0)
for (n, d, s, seed) in [(300, 3, 5, 1), (1000, 9, 17, 2), (2048, 8, 17, 3), (777, 11, 65, 4), (1500, 16, 80, 5),
                        (129, 1, 1, 6), (64, 2, 2, 7)]:
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    ls = rng.uniform(0.6, 1.8, d)
    V = rng.standard_normal((n, s))
    V[:, 0] *= 1e-20
    ctx.set_data(X)
    ctx.set_hyper([*ls, 1.3, 0.4])
    g = ctx.hv_f64(V)
    ref = orc.hv(X, ls, 1.3, 0.4, V)
    rel = np.linalg.norm(g - ref, axis=0) / np.linalg.norm(ref, axis=0)
    out[f"hv_{n}_{d}_{s}"] = g
    print(f"n={n} d={d} s={s}: max col rel vs oracle {rel.max():.2e}", flush=True)
# symmetry (H e_j columns) and linearity
n = 300
rng = np.random.default_rng(9)
X = rng.standard_normal((n, 4)).astype(np.float32)
ctx.set_data(X)
ctx.set_hyper([1.0, 0.8, 1.2, 0.9, 1.1, 0.3])
E = np.eye(n)
H = np.concatenate([ctx.hv_f64(E[:, c:c + 60]) for c in range(0, n, 60)], axis=1)
print("symmetric bitwise:", np.array_equal(H, H.T), "max asym", np.abs(H - H.T).max(), flush=True)
a, b = rng.standard_normal((n, 7)), rng.standard_normal((n, 7))
lin = np.abs(ctx.hv_f64(a + b) - ctx.hv_f64(a) - ctx.hv_f64(b)).max() / np.abs(ctx.hv_f64(a)).max()
print(f"linearity {lin:.2e}", flush=True)
out["H"] = H
# timing at config 2 (device timing through a short fp64 CG: ~1 operator / iteration)
q = datasets.config2()
ctx.set_data(q.X)
ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
V = np.random.default_rng(0).standard_normal((q.X.shape[0], 65))
t0 = time.perf_counter()
for _ in range(3):
    ctx.hv_f64(V)
print(f"config 2 hv_f64 host call {1e3 * (time.perf_counter() - t0) / 3:.2f} ms (incl. 2 x 21 MB PCIe)", flush=True)
out["c2"] = ctx.hv_f64(V)
np.savez(sys.argv[1], **out)
