"""Config-3 AP epoch cost: device solve time at 1 and 3 epochs (fixed
hyperparameters) against the hv_tc kernel time inside (wgp_profile)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config3()
n = p.X.shape[0]
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([1.0] * 3 + [1.0, 0.5])
B = np.random.default_rng(0).standard_normal((n, 65)).astype(np.float32)
for ep in (1, 3, 1, 3):
    cfg = wg.SolverConfig(kind="ap", tol_mean=1e-9, tol_samples=1e-9, max_iterations=ep, block_size=1000)
    ctx.profile(True)
    t0 = time.perf_counter()
    st = ctx.solve(B, cfg)
    dt = time.perf_counter() - t0
    kms, kl = ctx.profile_read()
    print(f"epochs={st.iterations_used} wall {dt * 1e3:.1f} ms  hv_tc kernels {kms:.1f} ms in {kl} launches", flush=True)
