"""Acceptance C8 on split 0 with the fp64 oracle (the reference's algorithm):
warm / cold CG training on the reference's synthetic data, dense-predictor
test metrics and their gap (compare with tests/test_gpu_acceptance.py)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import dense_ref  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import experiment as ex  # noqa: E402
import paper_2405_18328_b200 as wg  # noqa: E402

split = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kind = sys.argv[2] if len(sys.argv) > 2 else "cg"
X, y = orc.synthesize(2223, 26, 1.0, 1.0, 0.5, 4242)
full = ex.Dataset("c8", X, y)
split_seed = wg.derive_seed(0, 0x3711700 + split)
train_seed = wg.derive_seed(0, 0x7ea1 + split)
tr, te = ex.split_standardize(full, 0.9, split_seed)
Xtr = tr.X.astype(np.float32).astype(np.float64)
ytr = tr.y.astype(np.float32).astype(np.float64)
out = {}
for mode in ("warm", "cold"):
    cfg = orc.TrainConfig(steps=50, num_probes=16, mode=mode, seed=train_seed,
                          solver=orc.SolverConfig(kind=kind, tol_mean=0.01, tol_samples=0.1, block_size=250,
                                                  minibatch_size=1000, max_iterations=100000, learning_rate=4.0))
    o = orc.train(Xtr, ytr, cfg)
    c = o["constrained_params"][-1]
    d = tr.d
    m, v, nz = dense_ref.predict(Xtr, ytr, te.X.astype(np.float32).astype(np.float64), c[:d], c[d], c[d + 1])
    met = wg.test_metrics(wg.PredictiveDistribution(m, v, nz), te.y)
    out[mode] = (c, met)
    print(mode, "rmse %.6f llh %.6f" % (met.rmse, met.mean_loglik), "final", np.round(c[-3:], 5), flush=True)
print("oracle %s split %d: rmse gap %.5f llh gap %.4f" % (kind, split, abs(out["warm"][1].rmse - out["cold"][1].rmse),
      abs(out["warm"][1].mean_loglik - out["cold"][1].mean_loglik)))
