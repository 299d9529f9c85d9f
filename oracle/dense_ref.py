"""Independent dense numpy restatement of the reference's Eigen expressions.

TEST INFRASTRUCTURE ONLY -- used to pin the matrix-free C++ oracle
(warmgp_oracle.cpp) against a second, line-by-line transcription of the
reference's dense code (/root/reference/proj/src/*.cpp).  Never imported by
the product package.
"""
from __future__ import annotations

import numpy as np

SQRT3 = 1.7320508075688772


# kernel.cpp:14-31
def softplus(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > 0, x + np.log1p(np.exp(-np.abs(x))), np.log1p(np.exp(np.minimum(x, 0))))


def softplus_inverse(v):
    v = np.asarray(v, dtype=np.float64)
    return np.where(v > 0.6931471805599453, v + np.log1p(-np.exp(-v)), np.log(np.expm1(v)))


def softplus_derivative(x):
    x = np.asarray(x, dtype=np.float64)
    return 1.0 / (1.0 + np.exp(-x))


def constrained(transform, raw):
    return np.exp(raw) if transform == "log" else softplus(raw)


def chain(transform, raw):
    return np.exp(raw) if transform == "log" else softplus_derivative(raw)


# kernel.cpp:101-139
def scaled_sqdist(X, ls):
    Xs = X * (1.0 / np.asarray(ls))[None, :]
    sq = np.sum(Xs * Xs, axis=1)
    G = Xs @ Xs.T
    G = np.tril(G) + np.tril(G, -1).T  # mirrored from the lower triangle
    D = (sq[:, None] + sq[None, :]) - 2.0 * G
    return np.maximum(D, 0.0)


def kernel_matrices(X, ls, sf, sigma):
    R = np.sqrt(scaled_sqdist(X, ls))
    decay = np.exp(-SQRT3 * R)
    K = sf * sf * (1.0 + SQRT3 * R) * decay
    H = K.copy()
    H[np.diag_indices_from(H)] += sigma * sigma
    return H, K, decay


# kernel.cpp:160-199 (raw-space derivative matrices, transform-aware chain)
def derivative_matrices(X, transform, raw):
    n, d = X.shape
    ls = constrained(transform, raw[:d])
    sf = float(constrained(transform, raw[d]))
    sigma = float(constrained(transform, raw[d + 1]))
    _, K, decay = kernel_matrices(X, ls, sf, sigma)
    out = []
    for k in range(d):
        scale = 3.0 * sf * sf * chain(transform, raw[k]) / ls[k] ** 3
        diff = X[:, k][:, None] - X[:, k][None, :]
        D = scale * decay * diff * diff
        np.fill_diagonal(D, 0.0)
        out.append(D)
    out.append((2.0 * chain(transform, raw[d]) / sf) * K)
    out.append(np.eye(n) * (2.0 * sigma * chain(transform, raw[d + 1])))
    return out


# estimator.cpp:39-61 (explicit-matrix route)
def assemble_gradient(v_y, probe_solves, probes, derivs):
    s = probes.shape[1]
    quad = np.array([0.5 * v_y @ (D @ v_y) for D in derivs])
    trace = np.array([0.5 / s * np.sum(probe_solves * (D @ probes)) for D in derivs])
    return quad, trace


# exact.cpp:36-50
def exact_gradient(X, y, transform, raw):
    n, d = X.shape
    ls = constrained(transform, raw[:d])
    sf = float(constrained(transform, raw[d]))
    sigma = float(constrained(transform, raw[d + 1]))
    H, _, _ = kernel_matrices(X, ls, sf, sigma)
    L = np.linalg.cholesky(H)
    alpha = np.linalg.solve(L.T, np.linalg.solve(L, y))
    Hinv = np.linalg.inv(H)
    derivs = derivative_matrices(X, transform, raw)
    return np.array([0.5 * alpha @ (D @ alpha) - 0.5 * np.sum(Hinv * D) for D in derivs])


# solvers.cpp:81-139, dense
def cg_solve(H, rhs, init, tol_mean, tol_samples, max_it):
    n, s = rhs.shape
    bn = np.linalg.norm(rhs, axis=0)
    tols = np.array([tol_mean] + [tol_samples] * (s - 1))
    if max_it <= 0:
        max_it = 10 * n
    X = init.copy()
    R = rhs - H @ X
    P = np.zeros_like(rhs)
    rs = np.sum(R * R, axis=0)
    conv = np.zeros(s, dtype=bool)
    for j in range(s):
        if bn[j] == 0 or np.sqrt(rs[j]) <= tols[j] * bn[j]:
            conv[j] = True
        else:
            P[:, j] = R[:, j]
    it = 0
    while not conv.all() and it < max_it:
        it += 1
        HP = H @ P
        refresh = it % 50 == 0
        for j in range(s):
            if conv[j]:
                continue
            pHp = P[:, j] @ HP[:, j]
            if not pHp > 0:
                raise FloatingPointError("cg_solve: non-positive curvature")
            a = rs[j] / pHp
            X[:, j] += a * P[:, j]
            if refresh:
                R[:, j] = rhs[:, j] - H @ X[:, j]
            else:
                R[:, j] -= a * HP[:, j]
            rn = R[:, j] @ R[:, j]
            if np.sqrt(rn) <= tols[j] * bn[j]:
                conv[j] = True
                P[:, j] = 0
            else:
                P[:, j] = R[:, j] + (rn / rs[j]) * P[:, j]
            rs[j] = rn
    return X, it, conv


def predict(X_train, y, X_test, ls, sf, sigma):
    """exact.cpp:52-77 (dense fp64): latent means and variances at X_test."""
    X_train = np.asarray(X_train, np.float64)
    X_test = np.asarray(X_test, np.float64)
    H, _, _ = kernel_matrices(X_train, ls, sf, sigma)
    L = np.linalg.cholesky(H)
    alpha = np.linalg.solve(L.T, np.linalg.solve(L, np.asarray(y, np.float64)))
    ls = np.asarray(ls, np.float64)
    d = (((X_train[:, None, :] - X_test[None, :, :]) / ls) ** 2).sum(-1)
    r = np.sqrt(d)
    Ks = sf * sf * (1.0 + np.sqrt(3.0) * r) * np.exp(-np.sqrt(3.0) * r)  # n x m
    means = Ks.T @ alpha
    W = np.linalg.solve(L.T, np.linalg.solve(L, Ks))
    var = sf * sf - (Ks * W).sum(0)
    return means, np.maximum(var, 0.0), sigma * sigma
