"""Config 0 outer loop on the device: per-step time and CG iterations."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config0()
ctx = wg.Context(0)
ctx.set_data(p.X)
cfg = wg.TrainConfig(steps=20, learning_rate=0.1, num_probes=16, mode="warm", seed=0, transform="log",
                     estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                     warm_start_distance=False,
                     solver=wg.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=1000))
tr = ctx.train(p.y, cfg)
its = np.array([r.solver_iterations for r in tr.steps])
sms = np.array([r.solver_ms for r in tr.steps])
tms = np.array([r.step_ms for r in tr.steps])
print("iterations", its.tolist())
print(f"step ms mean {tms.mean():.2f}, solve ms mean {sms.mean():.2f}, solve us/iteration {1e3 * sms.sum() / its.sum():.1f}")
