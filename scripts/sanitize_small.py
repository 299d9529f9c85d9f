"""Small shapes through every device path, for compute-sanitizer runs (not run in this
round: the pool disallows compute-sanitizer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

rng = np.random.default_rng(0)
ctx = wg.Context(0)
for n, d, s in ((1, 2, 1), (129, 3, 17), (300, 9, 65), (257, 26, 5)):
    X = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, s)).astype(np.float32)
    ctx.set_data(X)
    ctx.set_hyper([1.0] * d + [1.1, 0.4])
    for impl in ("tc", "simt", "tc_bf16"):
        ctx.set_hv_impl(impl)
        ctx.hv(V)
    ctx.set_hv_impl("tc")
    raw = np.zeros(d + 2)
    ctx.grad("log", raw, V[:, 0].copy(), V[:, :min(s, 8)], V[:, :min(s, 8)], 0.5)
    for kind in ("cg", "ap", "sgd"):
        ctx.solve(V[:, :3], wg.SolverConfig(kind=kind, max_iterations=20, block_size=64, minibatch_size=min(n, 50),
                                            learning_rate=1.0))
print("sanitize run ok")
