"""Row sharding inside the library (wgp_set_comm, NCCL) on one
GPU: a one-rank communicator runs every sharded code path -- the in-place
all-gathers of the direction / iterate / result, the column reductions
finished on the gathered per-rank totals (dist_finish), AP's block-residual
all-reduce, the gradient's rank sum, all inside the captured CG / AP graphs
-- and must reproduce the unsharded context bitwise.  (This sandbox has one
GPU; the rank-count logic is covered by tests/test_shard_rows_cpu.py and the
gloo tests of the Python mirror, tests/test_sharding_cpu.py.)"""
import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import datasets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    a = wg.Context(0)
    b = wg.Context(0)
    b.set_comm(0, 1, wg.nccl_unique_id())
    yield a, b
    b.close()
    a.close()


def problem(n=1500, d=6, s=9, seed=4):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    rhs = rng.standard_normal((n, s)).astype(np.float32)
    hyp = [*rng.uniform(0.8, 1.5, d), 1.1, 0.3]
    return X, rhs, hyp


def test_shard_info(pair):
    _, b = pair
    X, _, hyp = problem()
    b.set_data(X)
    assert b.shard_info() == (0, 1, 0, 1500, 1536)


def test_hv_matches_unsharded(pair):
    a, b = pair
    X, V, hyp = problem(s=17)
    for c in (a, b):
        c.set_data(X)
        c.set_hyper(hyp)
    assert np.array_equal(a.hv(V), b.hv(V))
    V64 = V.astype(np.float64)
    assert np.array_equal(a.hv_f64(V64), b.hv_f64(V64))


@pytest.mark.parametrize("kind,prec", [("cg", "f64"), ("cg", "f32"), ("ap", "f64")])
def test_solve_matches_unsharded(pair, kind, prec):
    a, b = pair
    X, rhs, hyp = problem()
    cfg = wg.SolverConfig(kind=kind, tol_mean=1e-4, tol_samples=1e-3, block_size=256, max_iterations=3000)
    out = []
    for c in (a, b):
        c.set_data(X)
        c.set_hyper(hyp)
        c.set_cg_precision(prec)
        out.append(c.solve(rhs, cfg))
        c.set_cg_precision("f64")
    ga, gb = out
    assert gb.all_converged()
    if kind == "ap":
        # the unsharded AP closes most epochs with the incremental residual
        # R0 - H dX, the sharded one with B - H X: equal up to rounding
        assert abs(ga.iterations_used - gb.iterations_used) <= 1
        assert np.linalg.norm(ga.solutions - gb.solutions) <= 1e-4 * np.linalg.norm(ga.solutions)
        return
    assert ga.iterations_used == gb.iterations_used
    assert np.array_equal(ga.solutions, gb.solutions)
    assert np.array_equal(ga.per_column_relative_residual, gb.per_column_relative_residual)


@pytest.mark.parametrize("kind", ["cg", "ap"])
def test_train_matches_unsharded(pair, kind):
    a, b = pair
    p = datasets.config0(n=900, d=4)
    cfg = wg.TrainConfig(steps=4, num_probes=6, transform="log", estimator="pathwise", rff_features=128,
                         init_noise=0.5, solver=wg.SolverConfig(kind=kind, tol_mean=0.01, tol_samples=0.01,
                                                                block_size=200, max_iterations=2000))
    tr = []
    for c in (a, b):
        c.set_data(p.X)
        tr.append(c.train(p.y, cfg))
    ta, tb = tr
    if kind == "ap":  # see test_solve_matches_unsharded
        for ra, rb in zip(ta.steps, tb.steps):
            assert abs(ra.solver_iterations - rb.solver_iterations) <= 1
            assert np.allclose(ra.constrained_params, rb.constrained_params, rtol=1e-5)
        return
    for ra, rb in zip(ta.steps, tb.steps):
        assert ra.solver_iterations == rb.solver_iterations
        assert np.array_equal(ra.constrained_params, rb.constrained_params)
        assert ra.warm_start_distance == rb.warm_start_distance
    assert np.array_equal(ta.final_solutions, tb.final_solutions)


def test_grad_matches_unsharded(pair):
    a, b = pair
    X, L, hyp = problem(s=5)
    raw = np.log(np.asarray(hyp))
    outs = []
    for c in (a, b):
        c.set_data(X)
        outs.append(c.grad("log", raw, L[:, 0], L, L, 0.1))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_sgd_is_single_gpu(pair):
    _, b = pair
    X, rhs, hyp = problem(n=300)
    b.set_data(X)
    b.set_hyper(hyp)
    with pytest.raises(ValueError, match="row-sharded"):
        b.solve(rhs, wg.SolverConfig(kind="sgd", max_iterations=10))
