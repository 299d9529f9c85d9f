"""Device building blocks of the row-sharded solvers on one GPU:
the column-block H.V over a row range (wgp_hv_cols), the cached AP block
inverses (wgp_ap_factor / wgp_ap_block_solve) driving sharded.sharded_ap, and
the row-range gradient whose shard partials sum to the full contraction."""
import numpy as np
import pytest
import torch

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import sharded
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def problem(n=700, d=3, s=4, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    X = ((X - X.mean(0)) / X.std(0)).astype(np.float32)
    ls = rng.uniform(0.8, 1.5, d)
    B = rng.standard_normal((n, s)).astype(np.float32)
    return X, ls, 1.1, 0.5, B


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_hv_cols_matches_dense_oracle(mode):
    X, ls, sf, sig, B = problem()
    n, s = B.shape
    H = orc.kernel_matrices(X.astype(np.float64), ls, sf, sig)[0]
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    r0, r1, j0, j1 = 128, 512, 100, 450  # rows and a column block overlapping them (diagonal inside)
    ctx.set_rows(r0, r1)
    rng = np.random.default_rng(1)
    Vb = rng.standard_normal((j1 - j0, s)).astype(np.float32)
    Bl = rng.standard_normal((r1 - r0, s)).astype(np.float32)
    O0 = rng.standard_normal((r1 - r0, s)).astype(np.float32)
    dev = torch.device("cuda")
    Vt = torch.from_numpy(np.ascontiguousarray(Vb.T)).to(dev)
    Bt = torch.from_numpy(np.ascontiguousarray(Bl.T)).to(dev)
    Ot = torch.from_numpy(np.ascontiguousarray(O0.T)).to(dev)
    torch.cuda.synchronize()
    ctx.hv_cols_device(Vt.data_ptr(), j1 - j0, s, j0, j1, Ot.data_ptr(), r1 - r0, mode, Bt.data_ptr(), r1 - r0)
    torch.cuda.synchronize()
    got = Ot.cpu().numpy().T.astype(np.float64)
    hv = H[r0:r1, j0:j1] @ Vb.astype(np.float64)
    ref = {0: hv, 1: Bl - hv, 2: O0 - hv}[mode]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("rows,cols", [((300, 700), (0, 300)), ((128, 512), (100, 450)), ((0, 640), (500, 640))])
def test_hv_block_matches_dense_oracle(rows, cols):
    """wgp_hv_block: any block H[i0:i1, j0:j1] V of the full operator, with
    the diagonal term where the ranges overlap, independent of set_rows."""
    X, ls, sf, sig, B = problem()
    s = B.shape[1]
    H = orc.kernel_matrices(X.astype(np.float64), ls, sf, sig)[0]
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    ctx.set_rows(64, 200)  # must not matter
    (i0, i1), (j0, j1) = rows, cols
    Vb = np.random.default_rng(2).standard_normal((j1 - j0, s)).astype(np.float32)
    Vt = torch.from_numpy(np.ascontiguousarray(Vb.T)).cuda()
    Ot = torch.empty((s, i1 - i0), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ctx.hv_block_device(i0, i1, j0, j1, Vt.data_ptr(), j1 - j0, s, Ot.data_ptr(), i1 - i0)
    torch.cuda.synchronize()
    ref = H[i0:i1, j0:j1] @ Vb.astype(np.float64)
    assert np.linalg.norm(Ot.cpu().numpy().T - ref) / np.linalg.norm(ref) <= 1e-5
    ctx.close()


def test_hv_block_rejects_bad_ranges():
    """wgp_hv_block validates its ranges and leading dimensions like
    wgp_hv_cols (status 2, std::invalid_argument's text)."""
    X, ls, sf, sig, B = problem()
    n = X.shape[0]
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    V = torch.zeros((4, n), device="cuda")
    out = torch.zeros((4, n), device="cuda")
    for i0, i1, j0, j1, ldv, ldo in ((0, 0, 0, 10, n, n), (5, 3, 0, 10, n, n), (0, 10, 0, n + 1, n + 1, n),
                                     (-1, 10, 0, 10, n, n), (0, 10, 0, 10, 5, n), (0, 10, 0, 10, n, 5)):
        with pytest.raises(ValueError):
            ctx.hv_block_device(i0, i1, j0, j1, V.data_ptr(), ldv, 4, out.data_ptr(), ldo)
    ctx.close()


def test_sharded_ap_on_device_matches_oracle():
    """sharded_ap with the device ops (world 1): the reference's AP (block
    residuals formed lazily from the epoch-start residual) in fp32 storage
    with fp64 block solves; epochs within 10% of the fp64
    oracle's and the exact residual at the tolerance."""
    # config-0-like conditioning (d = 8, sigma 0.5), as the solver parity tests:
    # fp32 residual floors stay well below the tolerance
    X, ls, sf, sig, B = problem(n=900, d=8, s=5)
    n = X.shape[0]
    ctx = wg.Context(0)
    ctx.set_data(X)
    ctx.set_hyper([*ls, sf, sig])
    ops = sharded.device_ap_ops(ctx, 0, n)
    st = sharded.sharded_ap(ops, torch.from_numpy(B).cuda(), n, 0, n, block_size=200, tol_mean=1e-2,
                            tol_samples=1e-2)
    o = orc.solve(B, orc.SolverConfig(kind="ap", tol_mean=1e-2, tol_samples=1e-2, block_size=200),
                  X=X.astype(np.float64), ls=ls, sf=sf, sigma=sig)
    assert all(st.converged) and o.all_converged()
    assert abs(st.iterations_used - o.iterations_used) <= max(1, 0.1 * o.iterations_used)
    x = st.solutions.cpu().numpy().astype(np.float64)
    Hx = orc.hv(X.astype(np.float64), ls, sf, sig, x)
    true_rel = np.linalg.norm(B - Hx, axis=0) / np.linalg.norm(B, axis=0)
    assert np.all(true_rel <= 1e-2 * 1.05)
    # the library's own (left-looking) AP reaches the same tolerance in the same epochs
    g = ctx.solve(B, wg.SolverConfig(kind="ap", tol_mean=1e-2, tol_samples=1e-2, block_size=200))
    assert abs(g.iterations_used - st.iterations_used) <= 1
    ctx.close()


@pytest.mark.parametrize("impl", ["tc", "simt"])
def test_row_range_gradient_partials_sum_to_full(impl):
    rng = np.random.default_rng(5)
    n, d, s = 1500, 4, 16
    X = rng.standard_normal((n, d)).astype(np.float32)
    raw = np.array([orc.to_raw("log", v) for v in (*rng.uniform(0.7, 1.4, d), 1.2, 0.4)])
    vy = rng.standard_normal(n).astype(np.float32)
    L = rng.standard_normal((n, s)).astype(np.float32)
    R = rng.standard_normal((n, s)).astype(np.float32)
    ctx = wg.Context(0)
    ctx.set_hv_impl(impl)
    ctx.set_data(X)
    fa, fb = ctx.grad("log", raw, vy, L, R, 0.5 / s)
    parts = []
    for r0, r1 in sharded_rows(n, 3):
        ctx.set_rows(r0, r1)
        parts.append(ctx.grad("log", raw, vy, L, R, 0.5 / s))
    ctx.set_rows(0, n)
    sa = sum(p[0] for p in parts)
    sb = sum(p[1] for p in parts)
    assert np.allclose(sa, fa, rtol=1e-6, atol=1e-7 * np.abs(fa).max())
    assert np.allclose(sb, fb, rtol=1e-6, atol=1e-7 * np.abs(fb).max())
    oa, ob = orc.grad_contractions(X, "log", raw, vy, L, R, 0.5 / s)
    assert np.allclose(sa, oa, rtol=2e-5, atol=1e-5 * np.abs(oa).max())
    # world-1 sharded_grad is the row-range gradient itself
    ga, gb = sharded.sharded_grad(lambda: ctx.grad("log", raw, vy, L, R, 0.5 / s))
    assert np.array_equal(ga, fa) and np.array_equal(gb, fb)
    ctx.close()


def sharded_rows(n, world):
    return [sharded.row_range(n, r, world) for r in range(world)]


@pytest.mark.parametrize("kind", ["cg", "ap"])
def test_sharded_train_on_device_matches_train(kind):
    """The row-sharded outer loop on the device operators (world 1) follows
    the library's own training loop (wgp_train) at a tight solver tolerance:
    the same probes, seeds, warm starts and Adam; trajectories within 1e-3."""
    from paper_2405_18328_b200 import datasets

    p = datasets.config0(n=1024, d=4)
    ctx = wg.Context(0)
    ctx.set_data(p.X)
    cfg = wg.TrainConfig(steps=5, num_probes=8, mode="warm", seed=0, transform="log", estimator="pathwise",
                         rff_features=256, init_noise=0.5,
                         solver=wg.SolverConfig(kind=kind, tol_mean=1e-4, tol_samples=1e-4, block_size=256,
                                                max_iterations=5000))
    ref = ctx.train(p.y, cfg)
    steps = sharded.sharded_train(sharded.device_train_ops(ctx, 0, p.X.shape[0]), p.y, cfg)
    got = np.array([s.constrained_params for s in steps])
    exp = np.array([r.constrained_params for r in ref.steps])
    assert np.max(np.abs(got - exp) / np.abs(exp)) <= 1e-3
    ctx.close()
