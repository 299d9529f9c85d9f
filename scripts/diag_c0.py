"""Config-0 trajectory diagnostics: GPU vs fp64 oracle vs fp32-vector oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402


def cfg(mod, tol, f32=False, steps=20):
    s = mod.SolverConfig(kind="cg", tol_mean=tol, tol_samples=tol, max_iterations=1000)
    if f32:
        s.f32_vectors = True
    return mod.TrainConfig(steps=steps, learning_rate=0.1, num_probes=16, mode="warm", seed=0,
                           transform="log", estimator="pathwise", rff_features=1000,
                           init_noise=0.5, solver=s)


p = datasets.config0()
ctx = wg.Context(0)
ctx.set_data(p.X)
for tol in (0.01, 1e-4):
    g = ctx.train(p.y, cfg(wg, tol))
    o = orc.train(p.X, p.y, cfg(orc, tol))
    o32 = orc.train(p.X, p.y, cfg(orc, tol, True))
    gc = np.array([r.constrained_params for r in g.steps])
    relerr = np.max(np.abs(gc - o["constrained_params"]) / np.abs(o["constrained_params"]), axis=1)
    print(f"tol={tol}")
    print(" gpu it ", [r.solver_iterations for r in g.steps])
    print(" o64 it ", o["solver_iterations"].tolist())
    print(" o32 it ", o32["solver_iterations"].tolist())
    print(" max rel param diff per step", np.array2string(relerr, precision=2))
    print(" o32 vs o64 param diff", np.max(np.abs(o32["constrained_params"] - o["constrained_params"]) / o["constrained_params"]))
    print(" step ms", [round(r.step_ms, 2) for r in g.steps][:5], "solver ms", [round(r.solver_ms, 2) for r in g.steps][:5])
