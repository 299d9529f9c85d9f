"""Outer steps with AP at configs 2 and 3 (device time per step, epochs) -- dev timing."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

impl = os.environ.get("HV_IMPL", "tc")
which = sys.argv[1:] or ["c3", "c2"]
for name, gen, cap, steps in (("c3", datasets.config3, 10, 3), ("c2", datasets.config2, 100, 3)):
    if name not in which:
        continue
    p = gen()
    ctx = wg.Context(0, hv_impl=impl)
    ctx.set_data(p.X)
    cfg = wg.TrainConfig(steps=steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0, transform="log",
                         estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                         warm_start_distance=False,
                         solver=wg.SolverConfig(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=cap,
                                                block_size=1000))
    tr = ctx.train(p.y, cfg)
    print(name, impl, [round(r.step_ms, 1) for r in tr.steps], [r.solver_iterations for r in tr.steps],
          [round(float(r.per_column_relative_residual.max()), 5) for r in tr.steps], flush=True)
    ctx.close()
