"""Golden fixtures for tests/test_gpu_outer_parity.py: the fp64 oracle's
outer loop (the reference's algorithm, proj/src/optimizer.cpp:81-171, with
BASELINE's pathwise RFF probes and log-space hyperparameters) at

  * BASELINE config 2 (n=41,157, d=9, 64 probes + y, RFF 1000, Adam lr 0.1,
    warm start, seed 0) -- exactly bench.py's settings:
      - CG, tol 0.01, reference cap (10 n), 3 steps;
      - SGD, minibatch 1000, momentum 0.9, lr 30 (bench.py's grid-search
        result, proj/src/experiment.cpp:133-168), tol 0.01, reference cap
        (100 n / m), 2 steps;
      - AP, blocks of 1000, tol 0.01, with a 10-epoch budget per step (the
        reference cap of 1000 epochs costs the CPU oracle hours), 3 steps;
  * config 3's generator at n = 20,000 (the full 391,386 points are out of
    the CPU oracle's reach): AP, blocks of 1000, 10-epoch budget, 3 steps;
  * config 4's generator (d = 11, 2000 RFF features) at n = 20,000: CG, tol 0.01,
    cap 1000 (config 4's settings), 3 steps.

Stored per step: constrained theta, the gradient, solver iterations, the
per-column relative residuals, the warm-start distance.  The inputs are
regenerated from paper_2405_18328_b200.datasets (seeded), not stored.
Run: python tests/golden/make_outer_c2_c3.py [name ...]   (CPU, ~1 h on 8 cores)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "c2_cg": dict(config="c2", steps=3, solver=dict(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=0)),
    "c2_sgd": dict(config="c2", steps=2, solver=dict(kind="sgd", tol_mean=0.01, tol_samples=0.01, max_iterations=0,
                                                      minibatch_size=1000, momentum=0.9, learning_rate=30.0, seed=0)),
    "c2_ap": dict(config="c2", steps=3, solver=dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=10,
                                                     block_size=1000)),
    "c3_ap_n20000": dict(config="c3", n=20000, steps=3,
                         solver=dict(kind="ap", tol_mean=0.01, tol_samples=0.01, max_iterations=10, block_size=1000)),
    "c4_cg_n20000": dict(config="c4", n=20000, steps=3, rff_features=2000,
                         solver=dict(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=1000)),
}


def problem(case):
    gen = datasets.CONFIGS[case["config"]]
    return gen(n=case["n"]) if "n" in case else gen()


def train_config(mod, case):
    return mod.TrainConfig(steps=case["steps"], learning_rate=0.1, num_probes=64, mode="warm", seed=0,
                           transform="log", estimator="pathwise", rff_features=case.get("rff_features", 1000),
                           init_noise=0.5, init_constrained=1.0, solver=mod.SolverConfig(**case["solver"]))


def main(names):
    for name in names:
        case = CASES[name]
        p = problem(case)
        t0 = time.time()
        o = orc.train(p.X, p.y, train_config(orc, case))
        out = {"case": name, "config": case, "n": int(p.X.shape[0]), "d": int(p.X.shape[1]),
               "oracle_seconds": time.time() - t0,
               "constrained_params": o["constrained_params"].tolist(), "gradient": o["gradient"].tolist(),
               "solver_iterations": o["solver_iterations"].tolist(),
               "per_column_relative_residual": o["per_column_relative_residual"].tolist(),
               "warm_start_distance": o["warm_start_distance"].tolist()}
        with open(os.path.join(HERE, f"outer_{name}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(name, f"{out['oracle_seconds']:.0f}s", out["solver_iterations"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
