"""Golden fixture for tests/test_gpu_acceptance.py::test_c8_warm_cold_metric_parity:
acceptance criterion 8 (proj/tests/acceptance/acceptance_main.cpp:437-463) on
split 0 with CG, run by the fp64 oracle (the reference's algorithm and RNG
streams on the reference's synthetic data).  The reference algorithm itself
puts this pair's RMSE gap at 0.00511, just above the criterion's 0.005.
Run: python tests/golden/make_acceptance_c8.py  (CPU, a few minutes)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import dense_ref  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import experiment as ex  # noqa: E402
import paper_2405_18328_b200 as wg  # noqa: E402

X, y = orc.synthesize(2223, 26, 1.0, 1.0, 0.5, 4242)
full = ex.Dataset("c8", X, y)
split = 0
split_seed = wg.derive_seed(0, 0x3711700 + split)
train_seed = wg.derive_seed(0, 0x7ea1 + split)
tr, te = ex.split_standardize(full, 0.9, split_seed)
Xtr = tr.X.astype(np.float32).astype(np.float64)
ytr = tr.y.astype(np.float32).astype(np.float64)
out = {"criterion": 8, "solver": "cg", "split": split, "split_seed": split_seed, "train_seed": train_seed}
for mode in ("warm", "cold"):
    cfg = orc.TrainConfig(steps=50, num_probes=16, mode=mode, seed=train_seed,
                          solver=orc.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.1, block_size=250,
                                                  minibatch_size=1000, max_iterations=100000))
    c = orc.train(Xtr, ytr, cfg)["constrained_params"][-1]
    d = tr.d
    m, v, nz = dense_ref.predict(Xtr, ytr, te.X.astype(np.float32).astype(np.float64), c[:d], c[d], c[d + 1])
    met = wg.test_metrics(wg.PredictiveDistribution(m, v, nz), te.y)
    out[mode] = {"final_constrained": [float(t) for t in c], "test_rmse": met.rmse, "test_llh": met.mean_loglik}
out["rmse_gap"] = abs(out["warm"]["test_rmse"] - out["cold"]["test_rmse"])
out["llh_gap"] = abs(out["warm"]["test_llh"] - out["cold"]["test_llh"])
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "acceptance_c8_cg_split0.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out["rmse_gap"], out["llh_gap"])
