"""BASELINE config 4 end to end on one GPU (dev check): n = 1,844,352, d = 11,
64 pathwise probes + y (s = 65), 2000 RFF features, CG tol 0.01 (cap 1000),
warm start, log-space Adam lr 0.1 -- `steps` outer steps with the given CG
precision, per-step device times, iterations and residuals."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
t0 = time.time()
p = datasets.config4()
print(f"data {time.time() - t0:.1f}s", flush=True)
ctx = wg.Context(0, cg_precision=prec)
ctx.set_data(p.X)
cfg = wg.TrainConfig(steps=steps, learning_rate=0.1, num_probes=64, mode="warm", seed=0, transform="log",
                     estimator="pathwise", rff_features=2000, init_noise=0.5, init_constrained=1.0,
                     warm_start_distance=True,
                     solver=wg.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=cap))
t0 = time.time()
tr = ctx.train(p.y, cfg)
wall = time.time() - t0
rec = [{"step": r.step, "ms": r.step_ms, "solver_ms": r.solver_ms, "wsd_ms": r.warm_distance_ms,
        "iterations": r.solver_iterations, "max_residual": float(r.per_column_relative_residual.max()),
        "theta": [float(v) for v in r.constrained_params]} for r in tr.steps]
out = {"config": f"c4 n=1844352 d=11 s=65 RFF 2000 CG tol 0.01 cap {cap}", "cg_precision": prec, "wall_s": wall,
       "steps": rec}
print(json.dumps(out), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/c4_outer_{prec}_cap{cap}.json", "w") as f:
    json.dump(out, f, indent=1)
