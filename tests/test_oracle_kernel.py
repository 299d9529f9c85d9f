"""Pins the CPU oracle's kernel arithmetic to the reference's known answers.

Ports of /root/reference/proj/tests/kernel_test.cpp and acceptance C1
(acceptance_main.cpp:71-108), plus a cross-check against the independent
dense numpy restatement (oracle/dense_ref.py).
"""
import math

import numpy as np
import pytest

from oracle import dense_ref
from oracle import oracle as orc


def test_splitmix_and_derive_seed_known_values():
    # common.hpp:25-36 re-derived independently in Python
    def sm(x):
        M = (1 << 64) - 1
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    for b, s in [(0, 1), (12, 7), (2**63 + 5, 0x736F6C7665)]:
        assert orc.splitmix64(b) == sm(b)
        assert orc.derive_seed(b, s) == sm(sm(b) ^ sm((s + 0x51ED2701AB0A3C11) & ((1 << 64) - 1)))


def test_softplus_roundtrip():  # kernel_test.cpp:31-37
    for expo in np.arange(-6.0, 6.0001, 0.25):
        v = 10.0**expo
        back = orc.softplus(orc.softplus_inverse(v))
        assert abs(back - v) / v <= 1e-12


def test_softplus_derivative_fd():  # kernel_test.cpp:39-45
    for x in (-30.0, -2.0, -0.1, 0.0, 0.3, 5.0, 40.0):
        h = 1e-5
        fd = (orc.softplus(x + h) - orc.softplus(x - h)) / (2 * h)
        assert abs(orc.softplus_derivative(x) - fd) <= 1e-9


def test_softplus_inverse_rejects_nonpositive():
    with pytest.raises(orc.OracleInvalidArgument):
        orc.softplus_inverse(0.0)


def test_log_transform_roundtrip():
    for v in (1e-6, 0.5, 1.0, 3.0, 1e6):
        assert abs(orc.to_constrained("log", orc.to_raw("log", v)) - v) <= 1e-12 * v


def test_matern_at_zero_distance():  # kernel_test.cpp:47-56
    rng = np.random.default_rng(7)
    for rep in range(10):
        x = rng.standard_normal(3)
        sf = 1.3
        assert orc.matern32(x, x, np.full(3, 0.5 + rep * 0.3), sf) == pytest.approx(sf * sf, rel=1e-14)


def test_matern_closed_form_unit_distance():  # kernel_test.cpp:58-67, acceptance C1
    v = orc.matern32([0.0], [1.0], [1.0], 1.0)
    expected = (1 + math.sqrt(3)) * math.exp(-math.sqrt(3))
    assert abs(v - expected) <= 1e-12
    assert v == pytest.approx(0.4833577245, rel=1e-9)


def test_matern_monotone_in_lengthscale():  # kernel_test.cpp:69-81
    a, b = np.array([0.1, 0.4]), np.array([0.9, -0.2])
    prev = 0.0
    for ls in (0.5, 1.0, 2.0, 8.0, 64.0, 1024.0):
        v = orc.matern32(a, b, [ls, ls], 1.7)
        assert v > prev
        prev = v
    assert prev == pytest.approx(1.7 * 1.7, rel=1e-4)


def test_matern_symmetry_and_bounds():  # kernel_test.cpp:94-106
    rng = np.random.default_rng(21)
    ls = np.full(4, 0.8)
    for _ in range(200):
        x, x2 = rng.standard_normal(4), rng.standard_normal(4)
        k12, k21 = orc.matern32(x, x2, ls, 1.2), orc.matern32(x2, x, ls, 1.2)
        assert k12 == k21
        assert 0.0 < k12 < 1.2 * 1.2


def test_system_matrix_n1():  # kernel_test.cpp:108-115
    H, _, _ = orc.kernel_matrices(np.array([[0.3, -0.7]]), [1.0, 1.0], 1.5, 0.2)
    assert H[0, 0] == pytest.approx(1.5**2 + 0.2**2, rel=1e-14)


def test_system_matrix_duplicate_rows():  # kernel_test.cpp:117-130
    X = np.array([[0.1, 0.2], [0.1, 0.2], [0.8, 0.4]])
    H, K, _ = orc.kernel_matrices(X, [1.0, 1.0], 1.1, 1e-3)
    assert H[0, 1] == pytest.approx(1.1**2, rel=1e-14)
    np.linalg.cholesky(H)
    assert abs(np.linalg.eigvalsh(K).min()) <= 1e-12


def test_system_matrix_invariants():  # kernel_test.cpp:132-144
    rng = np.random.default_rng(3)
    X = rng.uniform(size=(50, 3))
    H, _, _ = orc.kernel_matrices(X, np.ones(3), 1.0, 1.0)
    assert np.abs(H - H.T).max() == 0.0
    assert np.abs(np.diag(H) - 2.0).max() <= 1e-12
    assert np.linalg.eigvalsh(H).min() >= 1.0 - 1e-10


def test_system_entries_match_pairwise():  # kernel_test.cpp:146-158
    rng = np.random.default_rng(11)
    X = rng.uniform(size=(20, 3))
    ls = np.array([0.6, 1.4, 2.2])
    H, _, _ = orc.kernel_matrices(X, ls, 0.9, 0.15)
    for i in range(20):
        for j in range(20):
            e = orc.matern32(X[i], X[j], ls, 0.9) + (0.15**2 if i == j else 0.0)
            assert abs(H[i, j] - e) <= 1e-12


def test_kernel_matrices_match_dense_numpy_restatement():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((64, 5))
    ls = rng.uniform(0.5, 2.0, 5)
    H, K, D = orc.kernel_matrices(X, ls, 1.3, 0.4)
    H2, K2, D2 = dense_ref.kernel_matrices(X, ls, 1.3, 0.4)
    for a, b in ((H, H2), (K, K2)):
        assert np.abs(a - b).max() <= 1e-13
    # decay = exp(-sqrt3 R) is first-order in R = sqrt(D); the Gram-trick residue
    # D_ii ~ 1e-16 (summation-order dependent, kernel.cpp:111-115) shows up as ~1e-8.
    assert np.abs(D - D2).max() <= 1e-6


@pytest.mark.parametrize("transform", ["softplus", "log"])
def test_derivatives_match_finite_differences(transform):
    """kernel_test.cpp:160-176 / acceptance C1: dH/dtheta_raw vs central FD (h=1e-5),
    checked through the oracle's streamed contractions against E_ij basis."""
    rng = np.random.default_rng(17)
    for rep in range(3):
        X = rng.uniform(size=(40, 2))
        ls = np.array([0.4 + 0.3 * rep, 1.0 + 0.2 * rep])
        raw = np.array([orc.to_raw(transform, v) for v in (*ls, 0.8 + 0.1 * rep, 0.1 + 0.05 * rep)])
        derivs = dense_ref.derivative_matrices(X, transform, raw)
        for k in range(4):
            up, dn = raw.copy(), raw.copy()
            up[k] += 1e-5
            dn[k] -= 1e-5
            cu = [orc.to_constrained(transform, r) for r in up]
            cd = [orc.to_constrained(transform, r) for r in dn]
            Hu, _, _ = orc.kernel_matrices(X, cu[:2], cu[2], cu[3])
            Hd, _, _ = orc.kernel_matrices(X, cd[:2], cd[2], cd[3])
            fd = (Hu - Hd) / 2e-5
            rel = np.linalg.norm(fd - derivs[k]) / np.linalg.norm(derivs[k])
            assert rel <= 1e-6


@pytest.mark.parametrize("transform", ["softplus", "log"])
def test_streamed_contractions_match_explicit(transform):
    """kernel_test.cpp:207-222 with the estimator's low-rank A and B."""
    rng = np.random.default_rng(13)
    n, d, s = 30, 3, 4
    X = rng.uniform(size=(n, d))
    raw = np.array([orc.to_raw(transform, v) for v in (0.5, 1.1, 1.9, 1.2, 0.25)])
    vy = rng.standard_normal(n)
    L, R = rng.standard_normal((n, s)), rng.standard_normal((n, s))
    coef = 0.5 / s
    oa, ob = orc.grad_contractions(X, transform, raw, vy, L, R, coef)
    A = 0.5 * np.outer(vy, vy)
    B = coef * L @ R.T
    for k, D in enumerate(dense_ref.derivative_matrices(X, transform, raw)):
        assert abs(oa[k] - np.sum(D * A)) <= 1e-12 * max(1, abs(oa[k]))
        assert abs(ob[k] - np.sum(D * B)) <= 1e-12 * max(1, abs(ob[k]))


def test_matrix_free_hv_matches_dense():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((200, 6))
    ls = rng.uniform(0.5, 2, 6)
    V = rng.standard_normal((200, 7))
    H, _, _ = dense_ref.kernel_matrices(X, ls, 1.1, 0.3)
    out = orc.hv(X, ls, 1.1, 0.3, V)
    assert np.abs(out - H @ V).max() <= 1e-12
    out2 = orc.dense_matmul(H, V)
    assert np.abs(out2 - H @ V).max() <= 1e-12
    rows = orc.hv_rows(X, ls, 1.1, 0.3, V, 50, 90)
    assert np.array_equal(rows, out[50:90])


def test_hv_thread_count_independent():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((300, 4))
    V = rng.standard_normal((300, 3))
    a = orc.hv(X, np.ones(4), 1.0, 0.5, V, nthreads=1)
    b = orc.hv(X, np.ones(4), 1.0, 0.5, V, nthreads=4)
    assert np.array_equal(a, b)
