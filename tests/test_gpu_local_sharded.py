"""Multi-rank row sharding inside the library on ONE GPU: N contexts joined
by the host-mediated test communicator (wgp_set_comm_local), each driven by
its own thread -- the same sharded code paths as NCCL ranks (own rows, in-place
all-gathers, rank-order reductions, AP block-residual all-reduce, gradient
rank sums), with collectives as host barriers plus device copies (no kernel
waits on another rank's).  Every rank must end with identical results, equal
to the unsharded context's up to the reduction order (H.V rows bitwise)."""
import threading

import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import datasets

pytestmark = pytest.mark.gpu


def on_ranks(nranks, X, fn):
    g = wg.LocalGroup(nranks)
    ctxs = [wg.Context(0) for _ in range(nranks)]
    for r, c in enumerate(ctxs):
        c.set_comm_local(g, r)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            ctxs[r].set_data(X)
            out[r] = fn(ctxs[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in ctxs:
        c.close()
    g.close()
    if errs:
        raise errs[0]
    return out


def problem(n, d=5, s=7, seed=9):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    rhs = rng.standard_normal((n, s)).astype(np.float32)
    return X, rhs, [*rng.uniform(0.8, 1.5, d), 1.1, 0.3]


@pytest.fixture(scope="module")
def ref():
    c = wg.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("nranks,n", [(2, 1000), (3, 1000), (4, 300)])
def test_hv_rows_bitwise(ref, nranks, n):
    X, V, hyp = problem(n, s=17)
    ref.set_data(X)
    ref.set_hyper(hyp)
    want, want64 = ref.hv(V), ref.hv_f64(V.astype(np.float64))

    def fn(c):
        c.set_hyper(hyp)
        return c.shard_info(), c.hv(V), c.hv_f64(V.astype(np.float64))

    outs = on_ranks(nranks, X, fn)
    assert sum(o[0][3] - o[0][2] for o in outs) == n  # the ranks' rows cover [0, n)
    for info, h, h64 in outs:
        assert np.array_equal(h, want) and np.array_equal(h64, want64)


@pytest.mark.parametrize("nranks,n", [(2, 1200), (3, 1200), (4, 300)])
@pytest.mark.parametrize("kind,prec", [("cg", "f64"), ("cg", "f32"), ("ap", "f64")])
def test_solve(ref, nranks, n, kind, prec):
    X, rhs, hyp = problem(n)
    cfg = wg.SolverConfig(kind=kind, tol_mean=1e-5, tol_samples=1e-4, block_size=100, max_iterations=3000)
    ref.set_data(X)
    ref.set_hyper(hyp)
    ref.set_cg_precision(prec)
    want = ref.solve(rhs, cfg)
    ref.set_cg_precision("f64")

    def fn(c):
        c.set_hyper(hyp)
        c.set_cg_precision(prec)
        return c.solve(rhs, cfg)

    outs = on_ranks(nranks, X, fn)
    for o in outs[1:]:  # every rank: the same solve
        assert o.iterations_used == outs[0].iterations_used
        assert np.array_equal(o.solutions, outs[0].solutions)
        assert np.array_equal(o.per_column_relative_residual, outs[0].per_column_relative_residual)
    got = outs[0]
    assert got.all_converged()
    # the rank-order sums reorder the dots' rounding: CG's path drifts at the
    # tolerance level (iterations within 10%, solutions within kappa * tol)
    assert abs(got.iterations_used - want.iterations_used) <= max(2, 0.1 * want.iterations_used)
    assert np.linalg.norm(got.solutions - want.solutions) <= 1e-2 * np.linalg.norm(want.solutions)
    assert np.all(got.per_column_relative_residual <= np.array([1e-5] + [1e-4] * 6) * 1.0001)


@pytest.mark.parametrize("kind", ["cg", "ap"])
def test_train(ref, kind):
    p = datasets.config0(n=1100, d=4)
    cfg = wg.TrainConfig(steps=3, num_probes=6, transform="log", estimator="pathwise", rff_features=128,
                         init_noise=0.5, solver=wg.SolverConfig(kind=kind, tol_mean=0.01, tol_samples=0.01,
                                                                block_size=200, max_iterations=2000))
    ref.set_data(p.X)
    want = ref.train(p.y, cfg)
    outs = on_ranks(3, p.X, lambda c: c.train(p.y, cfg))
    for o in outs[1:]:
        for ra, rb in zip(o.steps, outs[0].steps):
            assert np.array_equal(ra.constrained_params, rb.constrained_params)
            assert ra.solver_iterations == rb.solver_iterations
    for ra, rb in zip(outs[0].steps, want.steps):
        assert abs(ra.solver_iterations - rb.solver_iterations) <= max(2, 0.1 * rb.solver_iterations)
        assert np.allclose(ra.constrained_params, rb.constrained_params, rtol=1e-4)
        assert np.isclose(ra.warm_start_distance, rb.warm_start_distance, rtol=1e-3)


def test_grad(ref):
    X, L, hyp = problem(700, s=5)
    raw = np.log(np.asarray(hyp))
    ref.set_data(X)
    want = ref.grad("log", raw, L[:, 0], L, L, 0.1)
    outs = on_ranks(3, X, lambda c: c.grad("log", raw, L[:, 0], L, L, 0.1))
    for a, b in outs:
        assert np.array_equal(a, outs[0][0]) and np.array_equal(b, outs[0][1])
        assert np.allclose(a, want[0], rtol=1e-9) and np.allclose(b, want[1], rtol=1e-9)
