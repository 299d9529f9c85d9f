"""fp64 CG path: operator symmetry / parity, config-0 trajectory and iteration
counts against the fp64 oracle, and hv_f64 timings (dev diagnostic)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

ctx = wg.Context(0)
rng = np.random.default_rng(0)
# 1. symmetry and parity of the fp64 operator
n, d = 300, 8
X = rng.standard_normal((n, d)).astype(np.float32)
ls = rng.uniform(0.6, 1.6, d)
ctx.set_data(X)
ctx.set_hyper([*ls, 1.2, 0.3])
H = np.concatenate([ctx.hv_f64(np.eye(n)[:, c:c + 100]) for c in range(0, n, 100)], axis=1)
print("H symmetric bitwise:", np.array_equal(H, H.T), "max asym", np.abs(H - H.T).max())
Ht = np.concatenate([ctx.hv(np.eye(n, dtype=np.float32)[:, c:c + 64]) for c in range(0, n, 64)], axis=1)
print("tc H max asym", np.abs(Ht - Ht.T).max())
V = rng.standard_normal((n, 17))
ref = orc.hv(X, ls, 1.2, 0.3, V)
print("hv_f64 rel err vs oracle", np.linalg.norm(ctx.hv_f64(V) - ref) / np.linalg.norm(ref))
# linearity: H(a+b) == Ha + Hb to fp64 rounding
a, b = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
print("linearity", np.abs(ctx.hv_f64(a + b) - ctx.hv_f64(a) - ctx.hv_f64(b)).max())

# 2. config 0 trajectory
p = datasets.config0()


def c0(mod, prec=None, tol=0.01):
    return mod.TrainConfig(steps=20, learning_rate=0.1, num_probes=16, mode="warm", seed=0,
                           transform="log", estimator="pathwise", rff_features=1000,
                           init_noise=0.5, init_constrained=1.0,
                           solver=mod.SolverConfig(kind="cg", tol_mean=tol, tol_samples=tol, max_iterations=1000))


t = time.time()
o = orc.train(p.X, p.y, c0(orc))
print(f"oracle {time.time() - t:.1f}s it", list(o["solver_iterations"]), o["solver_iterations"].sum())
ctx.set_data(p.X)
for prec in ("f64", "f32"):
    ctx.set_cg_precision(prec)
    g = ctx.train(p.y, c0(wg))
    g = ctx.train(p.y, c0(wg))
    gc = np.array([r.constrained_params for r in g.steps])
    gi = np.array([r.solver_iterations for r in g.steps])
    rel = np.abs(gc - o["constrained_params"]) / np.abs(o["constrained_params"])
    print(prec, "max rel", rel.max(), "per step", np.round(rel.max(axis=1), 6))
    print(prec, "it", list(gi), gi.sum(), "solver ms", round(sum(r.solver_ms for r in g.steps), 2),
          "step ms", round(sum(r.step_ms for r in g.steps), 2))
    print(prec, "wsd", [round(r.warm_start_distance, 6) for r in g.steps[:4]], "oracle", np.round(o["warm_start_distance"][:4], 6))
ctx.set_cg_precision("f64")

# 3. hv_f64 timing
import ctypes as C  # noqa: E402
for name, gen, s in (("c0", datasets.config0, 17), ("c1", datasets.config1, 65), ("c2", datasets.config2, 65)):
    q = gen()
    ctx.set_data(q.X)
    ctx.set_hyper([*q.lengthscales, q.signal, q.noise])
    V = rng.standard_normal((q.X.shape[0], s))
    ctx.hv_f64(V)
    t = time.time()
    k = 5 if name != "c2" else 3
    for _ in range(k):
        ctx.hv_f64(V)
    dt = (time.time() - t) / k
    n = q.X.shape[0]
    print(f"hv_f64 {name} n={n} s={s}: {dt * 1e3:.2f} ms (host incl. copies) {n * n / dt:.3e} entries/s")
