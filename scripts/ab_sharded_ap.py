"""Same-box A/B of sharded_ap (world 1, config-2 shape, fixed 5 epochs):
this tree's module vs ab/sharded_head.py (a previous version), and the
device-resident ctx.solve AP for the host-overhead floor."""
import importlib.util
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets, sharded  # noqa: E402

p = datasets.config2()
n = p.X.shape[0]
ctx = wg.Context(0)
ctx.set_data(p.X)
ctx.set_hyper([1.0] * p.X.shape[1] + [1.0, 0.5])
rng = np.random.default_rng(0)
B = rng.standard_normal((n, 65)).astype(np.float32)
mods = {"new": sharded}
head = os.path.join(ROOT, "ab", "sharded_head.py")
if os.path.exists(head):
    spec = importlib.util.spec_from_file_location("sharded_head", head)
    m = importlib.util.module_from_spec(spec)
    sys.modules["sharded_head"] = m  # dataclasses resolve their module
    spec.loader.exec_module(m)
    mods["head"] = m
Bd = torch.from_numpy(B).cuda()
for rep in range(2):
    for name, mod in mods.items():
        ops = mod.device_ap_ops(ctx, 0, n)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = mod.sharded_ap(ops, Bd, n, 0, n, block_size=1000, tol_mean=1e-9, tol_samples=1e-9, max_iterations=5)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{name}: {dt * 1e3:.1f} ms for {st.iterations_used} epochs, res {st.per_column_relative_residual[0]:.3e}",
              flush=True)
    cfg = wg.SolverConfig(kind="ap", tol_mean=1e-9, tol_samples=1e-9, max_iterations=5, block_size=1000)
    t0 = time.perf_counter()
    st = ctx.solve(B, cfg)
    print(f"device ctx.solve: {(time.perf_counter() - t0) * 1e3:.1f} ms (incl. host copies), "
          f"res {st.per_column_relative_residual[0]:.3e}", flush=True)
