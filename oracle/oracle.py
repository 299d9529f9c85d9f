"""ctypes front end of the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module -- as the checker or as the timed CPU reference arm, never
as the thing measured or shipped.  The product package
(``paper_2405_18328_b200``) never imports it.

The C++ library (warmgp_oracle.cpp) is a fp64 restatement of the reference
``warmgp`` (/root/reference/proj); see oracle.h for the parity pin.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

OK, INVALID, NUMERICAL = 0, 2, 3
SOLVER_KINDS = {"cg": 0, "ap": 1, "sgd": 2}
MODES = {"warm": 0, "cold": 1, "cold-fixed": 2}
TRANSFORMS = {"softplus": 0, "log": 1}
ESTIMATORS = {"hutchinson": 0, "pathwise": 1}
DISTS = {"gaussian": 0, "rademacher": 1}


class OracleNumericalError(RuntimeError):
    """NumericalError of the reference (exit code 3)."""


class OracleInvalidArgument(ValueError):
    """std::invalid_argument of the reference (exit code 2)."""


class _SolverCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("tol_mean", C.c_double), ("tol_samples", C.c_double),
                ("max_iterations", C.c_int), ("block_size", C.c_int),
                ("minibatch_size", C.c_int), ("momentum", C.c_double),
                ("learning_rate", C.c_double), ("seed", C.c_uint64),
                ("f32_vectors", C.c_int)]


class _SolveState(C.Structure):
    _fields_ = [("solutions", C.POINTER(C.c_double)), ("residuals", C.POINTER(C.c_double)),
                ("per_column_relative_residual", C.POINTER(C.c_double)),
                ("converged", C.POINTER(C.c_int)), ("iterations_used", C.c_int)]


class _TrainCfg(C.Structure):
    _fields_ = [("steps", C.c_int), ("learning_rate", C.c_double), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double), ("num_probes", C.c_int),
                ("probe_distribution", C.c_int), ("mode", C.c_int), ("solver", _SolverCfg),
                ("init_constrained", C.c_double), ("seed", C.c_uint64), ("transform", C.c_int),
                ("estimator", C.c_int), ("rff_features", C.c_int), ("init_noise", C.c_double),
                ("init_signal", C.c_double), ("exact_gradients", C.c_int)]


class _Trace(C.Structure):
    _fields_ = [("raw_params", C.POINTER(C.c_double)),
                ("constrained_params", C.POINTER(C.c_double)),
                ("gradient", C.POINTER(C.c_double)), ("solver_iterations", C.POINTER(C.c_int)),
                ("per_column_relative_residual", C.POINTER(C.c_double)),
                ("warm_start_distance", C.POINTER(C.c_double)),
                ("probe_seed", C.POINTER(C.c_uint64)),
                ("final_solutions", C.POINTER(C.c_double))]


def build() -> str:
    """Compile the oracle with its committed Makefile (g++ -fopenmp)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        for name in ("or_splitmix64", "or_derive_seed"):
            getattr(_lib, name).restype = C.c_uint64
        _lib.or_splitmix64.argtypes = [C.c_uint64]
        _lib.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        _lib.or_split_order.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
        _lib.or_synthesize_draws.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p]
        for name in ("or_softplus", "or_softplus_inverse", "or_softplus_derivative"):
            getattr(_lib, name).restype = C.c_double
            getattr(_lib, name).argtypes = [C.c_double]
        for name in ("or_to_constrained", "or_to_raw", "or_chain"):
            getattr(_lib, name).restype = C.c_double
            getattr(_lib, name).argtypes = [C.c_int, C.c_double]
        _lib.or_matern32.restype = C.c_double
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pi(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _check(rc):
    if rc == OK:
        return
    msg = lib().or_last_error().decode()
    if rc == NUMERICAL:
        raise OracleNumericalError(msg)
    raise OracleInvalidArgument(msg)


# --------------------------------------------------------------------- common
def splitmix64(x: int) -> int:
    return int(lib().or_splitmix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def derive_seed(base: int, stream: int) -> int:
    return int(lib().or_derive_seed(C.c_uint64(base), C.c_uint64(stream)))


def split_order(n: int, split_seed: int) -> np.ndarray:
    """dataset.cpp:118-124: split_standardize's row permutation."""
    out = np.empty(int(n), dtype=np.int64)
    _check(lib().or_split_order(int(n), C.c_uint64(split_seed), out.ctypes.data))
    return out


def synthesize(n, d, lengthscales, signal, noise, seed):
    """dataset.cpp:167-190: X ~ U[0,1]^d and y = chol(K + noise^2 I) xi with the
    reference's draws (bitwise X and xi; y up to Cholesky rounding).
    The 4-argument form synthesize(n, d, noise, seed) is lengthscales = 1, signal = 1."""
    X = np.empty((n, d))
    xi = np.empty(n)
    _check(lib().or_synthesize_draws(int(n), int(d), C.c_uint64(seed), X.ctypes.data, xi.ctypes.data))
    H = kernel_matrices(X, np.broadcast_to(np.asarray(lengthscales, dtype=np.float64), (d,)), signal, noise)[0]
    return X, np.linalg.cholesky(H) @ xi


def softplus(x):
    return lib().or_softplus(float(x))


def softplus_inverse(v):
    r = lib().or_softplus_inverse(float(v))
    if np.isnan(r):
        raise OracleInvalidArgument(lib().or_last_error().decode())
    return r


def softplus_derivative(x):
    return lib().or_softplus_derivative(float(x))


def to_constrained(transform, raw):
    return lib().or_to_constrained(TRANSFORMS.get(transform, transform), float(raw))


def to_raw(transform, v):
    return lib().or_to_raw(TRANSFORMS.get(transform, transform), float(v))


def matern32(x, x2, ls, sf):
    x = np.ascontiguousarray(x, dtype=np.float64)
    x2 = np.ascontiguousarray(x2, dtype=np.float64)
    ls = np.ascontiguousarray(ls, dtype=np.float64)
    return lib().or_matern32(_p(x), _p(x2), C.c_int(x.size), _p(ls), C.c_double(sf))


# --------------------------------------------------------------------- kernel
def kernel_matrices(X, ls, sf, sigma):
    X = _f64(X)
    n, d = X.shape
    H = np.empty((n, n), order="F")
    K = np.empty((n, n), order="F")
    D = np.empty((n, n), order="F")
    _check(lib().or_build_kernel_matrices(_p(X), C.c_int64(n), C.c_int(d), _p(_f64(ls)),
                                          C.c_double(sf), C.c_double(sigma), _p(H), _p(K), _p(D)))
    return H, K, D


def hv(X, ls, sf, sigma, V, nthreads=0):
    X = _f64(X)
    V = _f64(V).reshape(X.shape[0], -1, order="F")
    n, d = X.shape
    out = np.empty_like(V)
    _check(lib().or_hv(_p(X), C.c_int64(n), C.c_int(d), _p(_f64(ls)), C.c_double(sf),
                       C.c_double(sigma), _p(V), C.c_int(V.shape[1]), _p(out), C.c_int(nthreads)))
    return out


def hv_rows(X, ls, sf, sigma, V, r0, r1, nthreads=0):
    X = _f64(X)
    V = _f64(V).reshape(X.shape[0], -1, order="F")
    n, d = X.shape
    out = np.empty((r1 - r0, V.shape[1]), order="F")
    _check(lib().or_hv_rows(_p(X), C.c_int64(n), C.c_int(d), _p(_f64(ls)), C.c_double(sf),
                            C.c_double(sigma), _p(V), C.c_int(V.shape[1]), C.c_int64(r0),
                            C.c_int64(r1), _p(out), C.c_int(nthreads)))
    return out


def dense_matmul(H, V, nthreads=0):
    H = _f64(H)
    V = _f64(V).reshape(H.shape[0], -1, order="F")
    out = np.empty_like(V)
    _check(lib().or_dense_matmul(_p(H), C.c_int64(H.shape[0]), _p(V), C.c_int(V.shape[1]),
                                 _p(out), C.c_int(nthreads)))
    return out


# --------------------------------------------------------------------- solvers
@dataclass
class SolverConfig:
    """solvers.hpp:20-32 (defaults identical)."""
    kind: str = "cg"
    tol_mean: float = 0.01
    tol_samples: float = 0.1
    max_iterations: int = 0
    block_size: int = 2000
    minibatch_size: int = 1000
    momentum: float = 0.9
    learning_rate: float = 10.0
    seed: int = 0
    f32_vectors: bool = False  # CG in the fp32 arithmetic of the GPU path

    def _c(self):
        return _SolverCfg(SOLVER_KINDS[self.kind], self.tol_mean, self.tol_samples,
                          self.max_iterations, self.block_size, self.minibatch_size,
                          self.momentum, self.learning_rate, self.seed, int(self.f32_vectors))


@dataclass
class SolveState:
    solutions: np.ndarray
    residuals: np.ndarray
    per_column_relative_residual: np.ndarray
    converged: list
    iterations_used: int

    def all_converged(self):
        return all(self.converged)


def solve(rhs, config: SolverConfig, init=None, *, H=None, X=None, ls=None, sf=None,
          sigma=None, nthreads=0) -> SolveState:
    """solvers.cpp:265-279.  Dense H (reference representation) or matrix-free X."""
    rhs = _f64(rhs)
    if rhs.ndim == 1:
        rhs = rhs.reshape(-1, 1, order="F")
    n, s = rhs.shape
    init = np.zeros_like(rhs) if init is None else _f64(init).reshape(n, s, order="F")
    sol = np.empty_like(rhs)
    res = np.empty_like(rhs)
    pcr = np.empty(s)
    conv = np.zeros(s, dtype=np.int32)
    st = _SolveState(_p(sol), _p(res), _p(pcr), _pi(conv), 0)
    cfg = config._c()
    if H is not None:
        H = _f64(H)
        rc = lib().or_solve(_p(H), None, C.c_int64(n), C.c_int(0), None, C.c_double(0),
                            C.c_double(0), C.byref(cfg), _p(rhs), _p(init), C.c_int(s),
                            C.byref(st), C.c_int(nthreads))
    else:
        X = _f64(X)
        rc = lib().or_solve(None, _p(X), C.c_int64(n), C.c_int(X.shape[1]), _p(_f64(ls)),
                            C.c_double(sf), C.c_double(sigma), C.byref(cfg), _p(rhs), _p(init),
                            C.c_int(s), C.byref(st), C.c_int(nthreads))
    _check(rc)
    return SolveState(sol, res, pcr, [bool(c) for c in conv], st.iterations_used)


# --------------------------------------------------------------------- estimator
def sample_probes(n, s, dist="gaussian", seed=0):
    out = np.empty((n, s), order="F")
    _check(lib().or_sample_probes(C.c_int64(n), C.c_int(s), C.c_int(DISTS.get(dist, dist)),
                                  C.c_uint64(seed), _p(out)))
    return out


def rff_base(n, d, F, s, seed):
    oz = np.empty((F, d))  # row-major: f-major
    chi2 = np.empty(F)
    b = np.empty(F)
    w = np.empty((F, s), order="F")
    eps = np.empty((n, s), order="F")
    _check(lib().or_rff_base(C.c_int64(n), C.c_int(d), C.c_int(F), C.c_int(s), C.c_uint64(seed),
                             _p(oz), _p(chi2), _p(b), _p(w), _p(eps)))
    return dict(omega_z=oz, chi2=chi2, phase_b=b, w=w, eps=eps)


def rff_probes(X, ls, sf, sigma, base, nthreads=0):
    X = _f64(X)
    n, d = X.shape
    F, s = base["w"].shape
    out = np.empty((n, s), order="F")
    oz = np.ascontiguousarray(base["omega_z"], dtype=np.float64)
    _check(lib().or_rff_probes(_p(X), C.c_int64(n), C.c_int(d), _p(_f64(ls)), C.c_double(sf),
                               C.c_double(sigma), C.c_int(F), C.c_int(s), _p(oz),
                               _p(_f64(base["chi2"])), _p(_f64(base["phase_b"])),
                               _p(_f64(base["w"])), _p(_f64(base["eps"])), _p(out),
                               C.c_int(nthreads)))
    return out


def grad_contractions(X, transform, raw, vy, L, R, coef_b, nthreads=0):
    """Raw-space <dH_k, A>, <dH_k, B> with A = vy vy^T / 2, B = coef_b L R^T."""
    X = _f64(X)
    n, d = X.shape
    L = _f64(L).reshape(n, -1, order="F")
    R = _f64(R).reshape(n, -1, order="F")
    oa = np.empty(d + 2)
    ob = np.empty(d + 2)
    _check(lib().or_grad_contractions(_p(X), C.c_int64(n), C.c_int(d),
                                      C.c_int(TRANSFORMS.get(transform, transform)),
                                      _p(_f64(raw)), _p(_f64(vy)), _p(L), _p(R),
                                      C.c_int(L.shape[1]), C.c_double(coef_b), _p(oa), _p(ob),
                                      C.c_int(nthreads)))
    return oa, ob


def exact_gradient(X, y, transform, raw, nthreads=0):
    X = _f64(X)
    n, d = X.shape
    g = np.empty(d + 2)
    _check(lib().or_exact_gradient(_p(X), _p(_f64(y)), C.c_int64(n), C.c_int(d),
                                   C.c_int(TRANSFORMS.get(transform, transform)), _p(_f64(raw)),
                                   _p(g), C.c_int(nthreads)))
    return g


def exact_mll(X, y, transform, raw, nthreads=0):
    X = _f64(X)
    n, d = X.shape
    m = C.c_double(0)
    _check(lib().or_exact_mll(_p(X), _p(_f64(y)), C.c_int64(n), C.c_int(d),
                              C.c_int(TRANSFORMS.get(transform, transform)), _p(_f64(raw)),
                              C.byref(m), C.c_int(nthreads)))
    return m.value


def warm_start_distance(X, ls, sf, sigma, init, sol, nthreads=0):
    X = _f64(X)
    n, d = X.shape
    init = _f64(init).reshape(n, -1, order="F")
    sol = _f64(sol).reshape(n, -1, order="F")
    out = C.c_double(0)
    _check(lib().or_warm_start_distance(_p(X), C.c_int64(n), C.c_int(d), _p(_f64(ls)),
                                        C.c_double(sf), C.c_double(sigma), _p(init), _p(sol),
                                        C.c_int(init.shape[1]), C.byref(out), C.c_int(nthreads)))
    return out.value


def adam_step(raw, grad, m, v, t, lr=0.1, beta1=0.9, beta2=0.999, eps=1e-8):
    """In-place on raw/m/v (float64 arrays)."""
    _check(lib().or_adam_step(_p(raw), _p(_f64(grad)), _p(m), _p(v), C.c_int(raw.size),
                              C.c_int(t), C.c_double(lr), C.c_double(beta1), C.c_double(beta2),
                              C.c_double(eps)))


# --------------------------------------------------------------------- optimizer
@dataclass
class TrainConfig:
    """optimizer.hpp:23-38 plus the BASELINE extensions."""
    steps: int = 100
    learning_rate: float = 0.1
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    num_probes: int = 16
    probe_distribution: str = "gaussian"
    mode: str = "warm"
    solver: SolverConfig = field(default_factory=SolverConfig)
    init_constrained: float = 1.0
    seed: int = 0
    transform: str = "softplus"
    estimator: str = "hutchinson"
    rff_features: int = 1000
    init_noise: float = 0.0
    init_signal: float = 0.0
    exact_gradients: bool = False

    def _c(self):
        return _TrainCfg(self.steps, self.learning_rate, self.adam_beta1, self.adam_beta2,
                         self.adam_eps, self.num_probes, DISTS[self.probe_distribution],
                         MODES[self.mode], self.solver._c(), self.init_constrained, self.seed,
                         TRANSFORMS[self.transform], ESTIMATORS[self.estimator],
                         self.rff_features, self.init_noise, self.init_signal,
                         int(self.exact_gradients))


def train(X, y, config: TrainConfig, nthreads=0):
    X = _f64(X)
    n, d = X.shape
    p, T, sp = d + 2, config.steps, config.num_probes + 1
    out = dict(raw_params=np.zeros((T, p)), constrained_params=np.zeros((T, p)),
               gradient=np.zeros((T, p)), solver_iterations=np.zeros(T, dtype=np.int32),
               per_column_relative_residual=np.zeros((T, sp)),
               warm_start_distance=np.zeros(T), probe_seed=np.zeros(T, dtype=np.uint64),
               final_solutions=np.zeros((n, sp), order="F"))
    tr = _Trace(_p(out["raw_params"]), _p(out["constrained_params"]), _p(out["gradient"]),
                _pi(out["solver_iterations"]), _p(out["per_column_relative_residual"]),
                _p(out["warm_start_distance"]),
                out["probe_seed"].ctypes.data_as(C.POINTER(C.c_uint64)),
                _p(out["final_solutions"]))
    cfg = config._c()
    _check(lib().or_train(_p(X), _p(_f64(y)), C.c_int64(n), C.c_int(d), C.byref(cfg),
                          C.byref(tr), C.c_int(nthreads)))
    return out
