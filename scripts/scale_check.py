"""Full-size BASELINE configs on one GPU: config 3 outer steps with AP
(blocks of 1000, epoch cap as given) and single H.V timings at configs 3, 4."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for name in ("c3", "c4"):
    p = datasets.CONFIGS[name]()
    n, d = p.X.shape
    ctx = wg.Context(0)
    ctx.set_data(p.X)
    ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
    st = torch.cuda.ExternalStream(ctx.stream)
    V = torch.randn(65, n, device="cuda")
    out = torch.empty_like(V)
    with torch.cuda.stream(st):
        ctx.hv_device(V.data_ptr(), n, 65, out.data_ptr(), n)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.hv_device(V.data_ptr(), n, 65, out.data_ptr(), n)
        b.record(st)
        b.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name}: n={n} H.V s=65 {ms:.1f} ms, {n * n / ms * 1e3:.3e} entries/s", flush=True)
    if name == "c3":
        cfg = wg.TrainConfig(steps=steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0,
                             transform="log", estimator="pathwise", rff_features=1000, init_noise=0.5,
                             init_constrained=1.0, warm_start_distance=False,
                             solver=wg.SolverConfig(kind="ap", tol_mean=0.01, tol_samples=0.01,
                                                    max_iterations=epochs, block_size=1000))
        t0 = time.time()
        tr = ctx.train(p.y, cfg)
        for r in tr.steps:
            print(f"c3 AP step {r.step}: {r.step_ms:.0f} ms (solve {r.solver_ms:.0f} ms, {r.solver_iterations} epochs), "
                  f"residual[0] {r.per_column_relative_residual[0]:.3e}, theta {np.round(r.constrained_params, 4)}",
                  flush=True)
        print(f"wall {time.time() - t0:.1f} s", flush=True)
    ctx.close()
