"""World-size-2 gloo tests of the row-sharded CG host logic.

The local row-block product is a host fp64 matrix here (the GPU path plugs in
the fused CUDA H.V through ``sharded.device_local_hv``); the test checks that
two ranks reproduce the single-process CG exactly in iteration count and to
rounding in the solutions, and match the oracle's cg_solve.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_18328_b200 import sharded


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=333, s=3, seed=0):
    from oracle import oracle as orc

    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, 3))
    H, _, _ = orc.kernel_matrices(X, [0.9, 1.2, 1.0], 1.1, 0.5)
    B = rng.standard_normal((n, s))
    return H, B


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, B = _problem()
    n = H.shape[0]
    r0, r1 = sharded.row_range(n, rank, world)
    Ht = torch.from_numpy(H[r0:r1])
    st = sharded.sharded_cg(lambda V: Ht @ V, torch.from_numpy(B[r0:r1]).clone(), n,
                            tol_mean=1e-6, tol_samples=1e-6)
    out[rank] = (r0, r1, st.solutions.numpy().copy(), st.iterations_used,
                 st.per_column_relative_residual)
    dist.destroy_process_group()


def test_row_range_partitions_tiles():
    for n in (1, 127, 128, 129, 1000, 13500):
        for w in (1, 2, 3, 8):
            rs = [sharded.row_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
                assert a1 == b0 and a0 % 128 == 0


def test_single_process_matches_oracle():
    from oracle import oracle as orc

    H, B = _problem()
    st = sharded.sharded_cg(lambda V: torch.from_numpy(H) @ V, torch.from_numpy(B), H.shape[0],
                            tol_mean=1e-6, tol_samples=1e-6)
    o = orc.solve(B, orc.SolverConfig(kind="cg", tol_mean=1e-6, tol_samples=1e-6), H=H)
    assert st.iterations_used == o.iterations_used
    # both stop at relative residual 1e-6: solutions agree to that order
    assert np.abs(st.solutions.numpy() - o.solutions).max() <= 1e-5


@pytest.mark.timeout(300)
def test_two_ranks_gloo_match_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    H, B = _problem()
    ref = sharded.sharded_cg(lambda V: torch.from_numpy(H) @ V, torch.from_numpy(B), H.shape[0],
                             tol_mean=1e-6, tol_samples=1e-6)
    sol = np.zeros_like(B)
    for rank in range(world):
        r0, r1, x, it, rel = out[rank]
        sol[r0:r1] = x
        assert abs(it - ref.iterations_used) <= 1  # fp64 summation order differs per shard
        assert np.all(np.array(rel) <= 1e-6 * 1.0001)
    assert np.abs(sol - ref.solutions.numpy()).max() <= 1e-5


# ------------------------------------------------------------------ AP + gradient
def host_ap_ops(H, r0, r1):
    """ApOps over a host fp64 matrix (the device path: sharded.device_ap_ops)."""
    Ht = torch.from_numpy(H)
    HI = Ht[r0:r1]
    chol = {}

    def factor(bs):
        chol.clear()
        n = H.shape[0]
        nb = -(-n // bs)
        for b in range(nb):
            j0, j1 = b * bs, min(n, (b + 1) * bs)
            chol[b] = torch.linalg.cholesky(Ht[j0:j1, j0:j1])
        return nb

    return sharded.ApOps(lambda B, X: B - HI @ X, lambda i0, i1, c0, c1, V: Ht[i0:i1, c0:c1] @ V, factor,
                         lambda b, Rb: torch.cholesky_solve(Rb, chol[b]))


def _worker_ap(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, B = _problem()
    n = H.shape[0]
    r0, r1 = sharded.row_range(n, rank, world)
    st = sharded.sharded_ap(host_ap_ops(H, r0, r1), torch.from_numpy(B[r0:r1]).clone(), n, r0, r1,
                            block_size=100, tol_mean=1e-8, tol_samples=1e-8)
    # gradient: rank partials of the B contraction (rows of L masked to the shard)
    from oracle import oracle as orc

    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, 3))
    raw = np.array([orc.to_raw("softplus", v) for v in (0.9, 1.2, 1.0, 1.1, 0.5)])
    vy, L, R = rng.standard_normal(n), rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    Lm = np.zeros_like(L)
    Lm[r0:r1] = L[r0:r1]
    ga, gb = sharded.sharded_grad(lambda: orc.grad_contractions(X, "softplus", raw, vy, Lm, R, 0.125))
    out[rank] = (r0, r1, st.solutions.numpy().copy(), st.iterations_used, st.per_column_relative_residual, gb)
    dist.destroy_process_group()


def test_sharded_ap_single_process_matches_oracle():
    """Right-looking block Gauss-Seidel with exact epoch refresh = ap_solve."""
    from oracle import oracle as orc

    H, B = _problem()
    n = H.shape[0]
    st = sharded.sharded_ap(host_ap_ops(H, 0, n), torch.from_numpy(B), n, 0, n, block_size=100,
                            tol_mean=1e-8, tol_samples=1e-8)
    o = orc.solve(B, orc.SolverConfig(kind="ap", tol_mean=1e-8, tol_samples=1e-8, block_size=100), H=H)
    assert st.iterations_used == o.iterations_used
    assert np.abs(st.solutions.numpy() - o.solutions).max() <= 1e-8 * np.abs(o.solutions).max() * 100
    assert np.all(np.array(st.per_column_relative_residual) <= 1e-8)


@pytest.mark.timeout(300)
def test_two_ranks_gloo_sharded_ap_and_gradient():
    """Blocks of 100 straddle the rank boundary at 128: R_b is assembled across
    ranks; both ranks reproduce the single-process AP, and the rank partials of
    the gradient contraction sum to the full one."""
    from oracle import oracle as orc

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_ap, args=(world, _free_port(), out), nprocs=world, join=True)
    H, B = _problem()
    n = H.shape[0]
    ref = sharded.sharded_ap(host_ap_ops(H, 0, n), torch.from_numpy(B), n, 0, n, block_size=100,
                             tol_mean=1e-8, tol_samples=1e-8)
    sol = np.zeros_like(B)
    for rank in range(world):
        r0, r1, x, it, rel, gb = out[rank]
        sol[r0:r1] = x
        assert it == ref.iterations_used
        assert np.all(np.array(rel) <= 1e-8)
    assert np.abs(sol - ref.solutions.numpy()).max() <= 1e-10 * np.abs(sol).max() + 1e-12
    rng = np.random.default_rng(4)
    X = rng.standard_normal((n, 3))
    raw = np.array([orc.to_raw("softplus", v) for v in (0.9, 1.2, 1.0, 1.1, 0.5)])
    vy, L, R = rng.standard_normal(n), rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    _, full = orc.grad_contractions(X, "softplus", raw, vy, L, R, 0.125)
    assert np.array_equal(out[0][5], out[1][5])  # identical on every rank
    assert np.allclose(out[0][5], full, rtol=1e-12, atol=1e-12 * np.abs(full).max())


# ------------------------------------------------------------------ outer loop
def host_train_ops(X, r0, r1):
    """TrainOps over host fp64 matrices (the device path: sharded.device_train_ops)."""
    from oracle import oracle as orc

    n, d = X.shape
    state = {}

    def set_hyper(cons):
        state["c"] = np.asarray(cons, dtype=np.float64)
        state["H"] = orc.kernel_matrices(X, state["c"][:d], state["c"][d], state["c"][d + 1])[0]

    def probes(seed, s, F, pathwise, dist_name):
        c = state["c"]
        if pathwise:
            return orc.rff_probes(X, c[:d], c[d], c[d + 1], orc.rff_base(n, d, F, s, seed)).astype(np.float32)
        return orc.sample_probes(n, s, dist_name, seed).astype(np.float32)

    def local_hv(V):
        return (torch.from_numpy(state["H"][r0:r1]) @ V.double()).to(V.dtype)

    def ap_ops():
        ops = host_ap_ops(state["H"], r0, r1)
        return sharded.ApOps(lambda B, Xf: (B.double() - torch.from_numpy(state["H"][r0:r1]) @ Xf.double()).to(B.dtype),
                             lambda i0, i1, c0, c1, V: (torch.from_numpy(state["H"][i0:i1, c0:c1]) @ V.double()).to(V.dtype),
                             ops.factor, ops.block_solve)

    def grad(T, raw, vy, L, R, coef):
        m = np.zeros((n, 1))
        m[r0:r1] = 1.0
        z = np.zeros(n)
        _, qa = orc.grad_contractions(X, T, raw, z, vy[:, None] * m, vy[:, None], 0.5)
        _, qb = orc.grad_contractions(X, T, raw, z, np.asarray(L) * m, np.asarray(R), coef)
        return qa, qb

    return sharded.TrainOps(n, d, r0, r1, set_hyper, probes, local_hv, ap_ops, grad, torch.device("cpu"))


def _train_problem():
    from oracle import oracle as orc

    rng = np.random.default_rng(9)
    X = rng.standard_normal((200, 2)).astype(np.float32).astype(np.float64)
    y = (np.sin(2 * X).sum(1) + 0.1 * rng.standard_normal(200)).astype(np.float32)
    return X, y


def _train_cfg(mod, kind, estimator):
    return mod.TrainConfig(steps=4, num_probes=4, mode="warm", seed=5, transform="log", estimator=estimator,
                           rff_features=64, init_noise=0.5,
                           solver=mod.SolverConfig(kind=kind, tol_mean=1e-6, tol_samples=1e-6, block_size=64,
                                                   max_iterations=5000))


def _worker_train(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2405_18328_b200 as wg

    X, y = _train_problem()
    r0, r1 = sharded.row_range(200, rank, world)
    res = {}
    for kind in ("cg", "ap"):
        steps = sharded.sharded_train(host_train_ops(X, r0, r1), y, _train_cfg(wg, kind, "pathwise"))
        res[kind] = [s.constrained_params for s in steps]
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,estimator", [("cg", "pathwise"), ("cg", "hutchinson"), ("ap", "pathwise")])
def test_sharded_train_single_process_matches_oracle_train(kind, estimator):
    """The sharded outer loop restates wgp_train's semantics (seeds, probes,
    warm starts, gradient assembly, Adam): with host operators it follows the
    oracle's training loop (optimizer.cpp:81-171) to 1e-5."""
    import paper_2405_18328_b200 as wg
    from oracle import oracle as orc

    X, y = _train_problem()
    steps = sharded.sharded_train(host_train_ops(X, 0, 200), y, _train_cfg(wg, kind, estimator))
    o = orc.train(X, y.astype(np.float64), _train_cfg(orc, kind, estimator))
    got = np.array([s.constrained_params for s in steps])
    assert np.allclose(got, o["constrained_params"], rtol=1e-5), (got, o["constrained_params"])


@pytest.mark.timeout(300)
def test_two_ranks_gloo_sharded_train():
    import paper_2405_18328_b200 as wg

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_train, args=(world, _free_port(), out), nprocs=world, join=True)
    X, y = _train_problem()
    for kind in ("cg", "ap"):
        ref = sharded.sharded_train(host_train_ops(X, 0, 200), y, _train_cfg(wg, kind, "pathwise"))
        refc = np.array([s.constrained_params for s in ref])
        assert out[0][kind] == out[1][kind]  # identical on every rank
        assert np.allclose(np.array(out[0][kind]), refc, rtol=1e-6), kind
