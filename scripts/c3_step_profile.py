"""One config-3 outer step (AP, 1 epoch) for a launch-list profile."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config3()
ctx = wg.Context(0, hv_impl=os.environ.get("HV_IMPL", "tc"))
ctx.set_data(p.X)
cfg = wg.TrainConfig(steps=1, learning_rate=0.1, num_probes=64, mode="warm", seed=0, transform="log",
                     estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                     warm_start_distance=False,
                     solver=wg.SolverConfig(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=1,
                                            block_size=1000))
tr = ctx.train(p.y, cfg)
print(tr.steps[0].step_ms, tr.steps[0].solver_ms)
