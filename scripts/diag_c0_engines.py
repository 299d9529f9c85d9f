"""Config 0 (CG tol 0.01, 20 warm steps): per-step CG iterations and
warm-start distances of the device run vs the fp64 oracle (fp64 CG operator
engine from WGP_HV64_ENGINE)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402


def cfg(mod):
    c = mod.TrainConfig(steps=20, learning_rate=0.1, num_probes=16, mode="warm", seed=0, transform="log",
                        estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                        solver=mod.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=1000))
    if mod is wg:
        c.warm_start_distance = True
    return c


p = datasets.config0()
ctx = wg.Context(0)
ctx.set_data(p.X)
g = ctx.train(p.y, cfg(wg))
o = orc.train(p.X, p.y, cfg(orc))
gi = np.array([r.solver_iterations for r in g.steps])
gw = np.array([r.warm_start_distance for r in g.steps])
gc = np.array([r.constrained_params for r in g.steps])
print("engine", os.environ.get("WGP_HV64_ENGINE", "i8"))
print("iters dev ", gi.tolist())
print("iters orc ", o["solver_iterations"].tolist())
print("wsd rel   ", np.round(np.abs(gw[1:] - o["warm_start_distance"][1:]) / o["warm_start_distance"][1:], 5).tolist())
print("theta rel ", float(np.max(np.abs(gc - o["constrained_params"]) / np.abs(o["constrained_params"]))))
