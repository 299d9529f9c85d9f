"""Device time per CG iteration (config 0, fp64 and fp32 CG) and per SGD step
(config 2) through the library, CUDA events around solves (dev timing)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402


def timed(ctx, fn, reps=3):
    st = torch.cuda.ExternalStream(ctx.stream)
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        out = fn()
        b.record(st)
        b.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best, out


p = datasets.config0()
ctx = wg.Context(0, hv_impl=os.environ.get("HV_IMPL", "tc"))
ctx.set_data(p.X)
ctx.set_hyper([2.6] * 8 + [1.14, 0.1])  # config 0's late hyperparameters (ill-conditioned)
rhs = np.random.default_rng(0).standard_normal((p.X.shape[0], 17)).astype(np.float32)
for prec in ("f64", "f32"):
    ctx.set_cg_precision(prec)
    cfg = wg.SolverConfig(kind="cg", tol_mean=1e-12, tol_samples=1e-12, max_iterations=200)
    ms, st = timed(ctx, lambda: ctx.solve(rhs, cfg))
    print(f"config 0 CG {prec}: {1e3 * ms / st.iterations_used:.1f} us per iteration ({st.iterations_used} it, incl. setup)")
q = datasets.config2()
ctx.set_data(q.X)
ctx.set_hyper([1.0] * 9 + [1.0, 0.5])
B = np.random.default_rng(0).standard_normal((q.X.shape[0], 65)).astype(np.float32)
for steps in (64, 512):
    cfg = wg.SolverConfig(kind="sgd", tol_mean=1e-12, tol_samples=1e-12, max_iterations=steps, minibatch_size=1000,
                          momentum=0.9, learning_rate=10.0)
    ms, st = timed(ctx, lambda: ctx.solve(B, cfg))
    print(f"config 2 SGD: {ms / steps:.4f} ms per step ({steps} steps, incl. setup)")
