"""Pins the oracle's CG / AP / SGD control flow to the reference's solver tests.

Ports of /root/reference/proj/tests/solvers_test.cpp and acceptance C2
(acceptance_main.cpp:111-155), run on the oracle with a dense H (the
reference's own representation) and, where it matters, matrix-free.
"""
import numpy as np
import pytest

from oracle import dense_ref
from oracle import oracle as orc


def random_spd(n, lo, hi, rng):  # test_util.hpp:24-34
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    h = q @ np.diag(rng.uniform(lo, hi, n)) @ q.T
    return 0.5 * (h + h.T)


def cfg(kind, tol=1e-8, **kw):  # solvers_test.cpp:14-24
    c = orc.SolverConfig(kind=kind, tol_mean=tol, tol_samples=tol, block_size=32,
                         minibatch_size=1 << 20, max_iterations=20000)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_identity_one_cg_iteration():  # :34-42
    rng = np.random.default_rng(1)
    rhs = rng.standard_normal((12, 3))
    st = orc.solve(rhs, cfg("cg"), H=np.eye(12))
    assert st.iterations_used == 1 and st.all_converged()
    assert np.abs(st.solutions - rhs).max() <= 1e-14


def test_2x2_diagonal():  # :44-53
    st = orc.solve(np.array([[2.0], [3.0]]), cfg("cg", 1e-12), H=np.diag([2.0, 3.0]))
    assert st.iterations_used <= 2
    assert np.allclose(st.solutions[:, 0], 1.0, atol=1e-10)


@pytest.mark.parametrize("kind", ["cg", "ap", "sgd"])
def test_exact_warm_start_zero_passes(kind):  # :55-68
    rng = np.random.default_rng(2)
    H = random_spd(40, 0.5, 4.0, rng)
    rhs = rng.standard_normal((40, 4))
    exact = np.linalg.solve(H, rhs)
    st = orc.solve(rhs, cfg(kind, 1e-6, learning_rate=1.0), init=exact, H=H)
    assert st.iterations_used == 0 and st.all_converged()


def test_cg_within_n_iterations():  # :70-85
    rng = np.random.default_rng(3)
    for rep in range(3):
        n = 40 + 30 * rep
        H = random_spd(n, 0.5, 5.0, rng)
        rhs = rng.standard_normal((n, 2))
        st = orc.solve(rhs, cfg("cg", 1e-10, max_iterations=10 * n), H=H)
        assert st.iterations_used <= n
        for j in range(2):
            assert np.linalg.norm(rhs[:, j] - H @ st.solutions[:, j]) / np.linalg.norm(rhs[:, j]) <= 1e-8


@pytest.mark.parametrize("kind", ["cg", "ap", "sgd"])
def test_zero_rhs_column(kind):  # :87-100
    H = np.eye(5) * 2.0
    rhs = np.zeros((5, 2))
    rhs[0, 1] = 1.0
    st = orc.solve(rhs, cfg(kind, 1e-10, learning_rate=5.0), H=H)
    assert st.converged[0]
    assert np.abs(st.solutions[:, 0]).max() == 0.0
    assert st.per_column_relative_residual[0] == 0.0


def test_cg_hilbert():  # :102-115
    n = 10
    H = 1.0 / (np.arange(n)[:, None] + np.arange(n)[None, :] + 1.0) + 1e-8 * np.eye(n)
    b = np.ones((n, 1))
    st = orc.solve(b, cfg("cg", 1e-6, max_iterations=5000), H=H)
    assert np.linalg.norm(b[:, 0] - H @ st.solutions[:, 0]) / np.linalg.norm(b) <= 1e-5


def test_ap_single_block_direct():  # :117-126
    rng = np.random.default_rng(4)
    H = random_spd(25, 0.5, 3.0, rng)
    rhs = rng.standard_normal((25, 3))
    st = orc.solve(rhs, cfg("ap", 1e-10, block_size=4000), H=H)
    assert st.iterations_used == 1
    assert np.abs(st.solutions - np.linalg.solve(H, rhs)).max() <= 1e-10


def test_ap_diagonal_one_epoch():  # :128-137
    st = orc.solve(np.array([[1.0], [2.0], [3.0], [4.0]]), cfg("ap", 1e-12, block_size=2),
                   H=np.diag([1.0, 2.0, 3.0, 4.0]))
    assert st.iterations_used == 1
    assert np.abs(st.solutions - 1.0).max() <= 1e-14


def test_ap_residual_nonincreasing():  # :139-153
    rng = np.random.default_rng(5)
    H = random_spd(200, 0.2, 4.0, rng)
    rhs = rng.standard_normal((200, 2))
    prev = np.linalg.norm(rhs)
    for epochs in range(1, 26, 3):
        st = orc.solve(rhs, cfg("ap", 1e-14, block_size=50, max_iterations=epochs), H=H)
        now = np.linalg.norm(rhs - H @ st.solutions)
        assert now <= prev * (1 + 1e-12) + 1e-14
        prev = now


def test_sgd_identity_coordinate_descent():  # :155-169
    rng = np.random.default_rng(6)
    rhs = rng.standard_normal((30, 2))
    st = orc.solve(rhs, cfg("sgd", 1e-12, minibatch_size=10, momentum=0.0, learning_rate=10.0,
                              max_iterations=500, seed=99), H=np.eye(30))
    assert st.all_converged()
    assert np.abs(st.solutions - rhs).max() <= 1e-12


def test_full_batch_heavy_ball():  # :171-188
    rng = np.random.default_rng(7)
    n = 100
    H = random_spd(n, 0.5, 2.0, rng)
    rhs = rng.standard_normal((n, 2))
    lam = np.linalg.eigvalsh(H).max()
    st = orc.solve(rhs, cfg("sgd", 1e-6, minibatch_size=n, momentum=0.9,
                              learning_rate=1.0 / lam, max_iterations=10 * n), H=H)
    assert st.all_converged()
    for j in range(2):
        assert np.linalg.norm(rhs[:, j] - H @ st.solutions[:, j]) / np.linalg.norm(rhs[:, j]) <= 1e-6


def test_sgd_stored_residual_proxy():  # :190-213
    rng = np.random.default_rng(8)
    n = 500
    X = rng.uniform(size=(n, 2))
    H, _, _ = orc.kernel_matrices(X, [0.8, 1.2], 1.0, 0.4)
    rhs = rng.standard_normal((n, 3))
    c = orc.SolverConfig(kind="sgd", tol_mean=0.01, tol_samples=0.1, minibatch_size=250,
                         momentum=0.9, learning_rate=1.0, max_iterations=40000, seed=5)
    st = orc.solve(rhs, c, H=H)
    assert st.all_converged()
    for j in range(3):
        stored = np.linalg.norm(st.residuals[:, j]) / np.linalg.norm(rhs[:, j])
        assert st.per_column_relative_residual[j] <= 2.0 * stored


@pytest.mark.parametrize("kind", ["cg", "ap", "sgd"])
def test_all_solvers_match_direct(kind):  # :215-235
    rng = np.random.default_rng(9)
    n = 120
    X = rng.uniform(size=(n, 3))
    H, _, _ = orc.kernel_matrices(X, np.ones(3), 1.0, 1.0)
    rhs = rng.standard_normal((n, 4))
    exact = np.linalg.solve(H, rhs)
    st = orc.solve(rhs, cfg(kind, 1e-8, learning_rate=1.5, max_iterations=100000), H=H)
    assert st.all_converged()
    for j in range(4):
        assert np.linalg.norm(st.solutions[:, j] - exact[:, j]) / np.linalg.norm(exact[:, j]) <= 1e-6


@pytest.mark.parametrize("kind", ["cg", "ap", "sgd"])
def test_matrix_free_equals_dense(kind):
    """The matrix-free operator reproduces the dense-H control flow exactly
    (iteration counts equal, solutions to rounding)."""
    rng = np.random.default_rng(10)
    n = 150
    X = rng.standard_normal((n, 3))
    ls = np.array([0.7, 1.2, 0.9])
    H, _, _ = orc.kernel_matrices(X, ls, 1.1, 0.3)
    rhs = rng.standard_normal((n, 3))
    c = cfg(kind, 1e-6, block_size=40, minibatch_size=50, learning_rate=2.0, seed=3)
    a = orc.solve(rhs, c, H=H)
    b = orc.solve(rhs, c, X=X, ls=ls, sf=1.1, sigma=0.3)
    assert a.iterations_used == b.iterations_used
    assert np.abs(a.solutions - b.solutions).max() <= 1e-9 * np.abs(a.solutions).max()


def test_cg_matches_dense_numpy_restatement():
    rng = np.random.default_rng(12)
    n = 90
    H = random_spd(n, 0.1, 3.0, rng)
    rhs = rng.standard_normal((n, 4))
    st = orc.solve(rhs, cfg("cg", 1e-9), H=H)
    X, it, conv = dense_ref.cg_solve(H, rhs, np.zeros_like(rhs), 1e-9, 1e-9, 20000)
    assert st.iterations_used == it
    assert np.abs(st.solutions - X).max() <= 1e-9


@pytest.mark.parametrize("kind", ["cg", "ap", "sgd"])
def test_bitwise_determinism(kind):  # :237-255
    rng = np.random.default_rng(10)
    H = random_spd(60, 0.5, 3.0, rng)
    rhs = rng.standard_normal((60, 3))
    init = 0.1 * rng.standard_normal((60, 3))
    c = cfg(kind, 1e-6, minibatch_size=20, learning_rate=5.0, seed=1234)
    a = orc.solve(rhs, c, init=init, H=H)
    b = orc.solve(rhs, c, init=init, H=H, nthreads=1)
    assert np.array_equal(a.solutions, b.solutions)
    assert np.array_equal(a.residuals, b.residuals)
    assert a.iterations_used == b.iterations_used and a.converged == b.converged


def test_per_column_tolerances():  # :257-275
    rng = np.random.default_rng(11)
    H = random_spd(80, 0.5, 6.0, rng)
    rhs = rng.standard_normal((80, 5))
    c = orc.SolverConfig(kind="cg", tol_mean=1e-6, tol_samples=1e-2)
    st = orc.solve(rhs, c, H=H)
    assert st.all_converged()
    assert st.per_column_relative_residual[0] <= 1e-5
    assert all(st.per_column_relative_residual[1:] <= 1e-1)
    loose = orc.solve(rhs, orc.SolverConfig(kind="cg", tol_mean=1e-2, tol_samples=1e-2), H=H)
    assert loose.iterations_used <= st.iterations_used


def test_non_pd_reported():  # :277-286
    H = np.array([[1.0, 2.0], [2.0, 1.0]])
    b = np.array([[1.0], [0.0]])
    with pytest.raises(orc.OracleNumericalError, match="not positive definite"):
        orc.solve(b, cfg("cg"), H=H)
    with pytest.raises(orc.OracleNumericalError, match="not positive definite"):
        orc.solve(b, cfg("ap", block_size=2), H=H)


def test_sgd_divergence_message():  # :288-297
    rng = np.random.default_rng(12)
    H = random_spd(20, 1.0, 5.0, rng)
    b = rng.standard_normal((20, 1))
    with pytest.raises(orc.OracleNumericalError, match="smaller learning rate"):
        orc.solve(b, cfg("sgd", 1e-8, learning_rate=1e6, max_iterations=100000), H=H)


def test_config_validation():  # :299-313
    for bad in (dict(tol_mean=0.0), dict(tol_samples=1.0), dict(block_size=0), dict(minibatch_size=0)):
        c = orc.SolverConfig(**bad)
        with pytest.raises(orc.OracleInvalidArgument):
            orc.solve(np.ones((3, 1)), c, H=np.eye(3))


def test_acceptance_c2_small():
    """acceptance_main.cpp:111-155 at 4 instances (the full criterion runs 20)."""
    rng = np.random.default_rng(7)
    worst, cg_max = 0.0, 0
    for inst in range(4):
        n = 300
        X = rng.uniform(size=(n, 3))
        ls = rng.uniform(0.5, 1.5, 3)
        sf, sig = rng.uniform(0.5, 1.5), 0.3 + 0.3 * rng.uniform(0.5, 1.5)
        H, _, _ = orc.kernel_matrices(X, ls, sf, sig)
        rhs = rng.standard_normal((n, 5))
        exact = np.linalg.solve(H, rhs)
        lam = np.linalg.eigvalsh(H).max()
        for kind in ("cg", "ap", "sgd"):
            c = orc.SolverConfig(kind=kind, tol_mean=1e-8, tol_samples=1e-8, block_size=100,
                                 minibatch_size=n, momentum=0.9, learning_rate=0.9 * n / lam,
                                 max_iterations=50000, seed=11 + inst)
            st = orc.solve(rhs, c, H=H)
            if kind == "cg":
                cg_max = max(cg_max, st.iterations_used)
            rel = np.linalg.norm(st.solutions - exact, axis=0) / np.linalg.norm(exact, axis=0)
            worst = max(worst, rel.max())
    assert worst <= 1e-6
    assert cg_max <= 300
