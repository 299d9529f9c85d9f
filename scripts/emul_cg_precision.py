"""Numpy emulation of CG's sensitivity to the operator's arithmetic (the study
behind the fp64 CG path, DESIGN.md §4.1b / §5).

CG (the reference's per-column CG with the refresh every 50 iterations,
proj/src/solvers.cpp:81-139, without the best-iterate safeguard) on config 0's
H at the hyperparameters of its last outer step (from the fp64 oracle run),
rhs = [y, 16 N(0,1) columns], tol 0.01, with the matvec / vector arithmetic
replaced by models of the device engines:
  * fp64 exact; fp32 vectors; fp32-rounded (fixed, symmetric) entries;
  * P rounded to 22 bits (tf32 hi + lo) before an exact product;
  * asymmetric entry perturbations; matvec noise eps |H||P| and eps rms;
Prints CG iterations and the true final residual of each.  CPU, ~1 minute."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dense_ref as dr  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2405_18328_b200 import datasets  # noqa: E402

p = datasets.config0()
cfg = orc.TrainConfig(steps=20, learning_rate=0.1, num_probes=16, mode="warm", seed=0, transform="log",
                      estimator="pathwise", rff_features=1000, init_noise=0.5, init_constrained=1.0,
                      solver=orc.SolverConfig(kind="cg", tol_mean=0.01, tol_samples=0.01, max_iterations=1000))
th = orc.train(p.X, p.y, cfg)["constrained_params"][-1]
X = p.X.astype(np.float64)
d = X.shape[1]
H, _, _ = dr.kernel_matrices(X, th[:d], th[d], th[d + 1])
n = H.shape[0]
rng = np.random.default_rng(1)
B = np.concatenate([p.y.astype(np.float64)[:, None], rng.standard_normal((n, 16))], axis=1)
s = B.shape[1]


def tf32(a):
    b = np.asarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32).astype(np.float64)


def cg(mv, tol=0.01, f32vec=False, maxit=1000):
    rnd = (lambda a: a.astype(np.float32).astype(np.float64)) if f32vec else (lambda a: a)
    x = np.zeros_like(B)
    r = B.copy()
    pp = r.copy()
    bn = np.linalg.norm(B, axis=0)
    rs = (r * r).sum(0)
    it = 0
    while it < maxit:
        conv = np.sqrt(rs) / bn <= tol
        if conv.all():
            break
        it += 1
        hp = rnd(mv(pp))
        pap = (pp * hp).sum(0)
        a = np.where(conv, 0, rs / np.where(pap == 0, 1, pap))
        x = rnd(x + a * pp)
        r = rnd(r - a * hp)
        if it % 50 == 0:
            r = rnd(B - mv(x))
        rn = (r * r).sum(0)
        be = rn / rs
        rs = rn
        pp = rnd(np.where(conv, 0, r + be * pp))
    return it, float((np.linalg.norm(B - H @ x, axis=0) / bn).max())


H32 = H.astype(np.float32).astype(np.float64)
Ha = (H * (1 + 4e-7 * rng.standard_normal(H.shape))).astype(np.float32).astype(np.float64)
absH = np.abs(H)
cases = [
    ("fp64 exact", lambda P: H @ P, False),
    ("fp32 vectors, exact product", lambda P: H @ P, True),
    ("fp32-rounded symmetric entries, fp64 P", lambda P: H32 @ P, False),
    ("P rounded to 22 bits (tf32 hi+lo)", lambda P: H @ (tf32(P) + tf32(P - tf32(P))), False),
    ("asymmetric 4e-7 entry noise", lambda P: Ha @ P, False),
]
for eps in (1e-7, 1e-8, 1e-9):
    cases.append((f"matvec noise {eps:g} |H||P|",
                  lambda P, e=eps: H @ P + e * (absH @ np.abs(P)) * rng.standard_normal(P.shape), False))
for name, mv, f32 in cases:
    it, res = cg(mv, f32vec=f32)
    print(f"{name:42s} {it:4d} iterations, true residual {res:.4f}")
