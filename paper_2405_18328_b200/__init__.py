"""B200-native hot path of warm-started iterative-GP marginal-likelihood
optimisation (arXiv 2405.18328), behind the reference library's API.

The compute lives in ``libwarmgp_b200.so`` (sm_100a CUDA + C++ host runtime,
C-ABI in ``include/warmgp_b200.h``).  This module is the Python mirror of
the reference ``warmgp`` C++ API (proj/include/warmgp/*.hpp): the same type
names, fields, defaults, error classes and message texts, so tests read like
the reference's own.  There is no CPU fallback: without the built library or
without a B200 every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

__all__ = [
    "NumericalError", "DeviceError", "Context", "Hyperparameters", "SolverConfig", "SolveState",
    "TrainConfig", "StepRecord", "OptTrace", "KernelOperator", "solve", "train",
    "sample_probes", "GradientEstimate", "assemble_gradient_streamed", "warm_start_distance",
    "adam_step", "derive_seed", "library_path", "load", "device_count", "train_exact",
    "exact_mll", "exact_gradient", "predict", "test_metrics", "PredictiveDistribution", "TestMetrics",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libwarmgp_b200.so"
_lib = None

WGP_OK, WGP_INVALID, WGP_NUMERICAL, WGP_DEVICE = 0, 2, 3, 4
HV_TC, HV_SIMT, HV_TC_F16 = 0, 1, 2
# tc: tcgen05 3xTF32 (default); simt: CUDA-core fp32; tc_f16: tcgen05 with
# fp16x3 K.V over column-scaled V (half the K.V tensor work, same operand split)
_HV_IMPLS = {"tc": HV_TC, "simt": HV_SIMT, "tc_f16": HV_TC_F16}
CG_F64, CG_F32 = 0, 1
_CG_PRECISIONS = {"f64": CG_F64, "f32": CG_F32}
_KINDS = {"cg": 0, "ap": 1, "sgd": 2}
_MODES = {"warm": 0, "cold": 1, "cold-fixed": 2}
_TRANSFORMS = {"softplus": 0, "log": 1}
_ESTIMATORS = {"hutchinson": 0, "pathwise": 1}
_DISTS = {"gaussian": 0, "rademacher": 1}


class NumericalError(RuntimeError):
    """warmgp::NumericalError (proj/include/warmgp/common.hpp:13-16), exit code 3."""


class DeviceError(RuntimeError):
    """CUDA / device failure (exit code 4 in the C-ABI)."""


# ----------------------------------------------------------------- C structs
class _SolverCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("tol_mean", C.c_double), ("tol_samples", C.c_double),
                ("max_iterations", C.c_int), ("block_size", C.c_int),
                ("minibatch_size", C.c_int), ("momentum", C.c_double),
                ("learning_rate", C.c_double), ("seed", C.c_uint64)]


class _SolveState(C.Structure):
    _fields_ = [("solutions", C.POINTER(C.c_float)), ("residuals", C.POINTER(C.c_float)),
                ("per_column_relative_residual", C.POINTER(C.c_double)),
                ("converged", C.POINTER(C.c_int)), ("iterations_used", C.c_int)]


class _SolveStateF64(C.Structure):
    _fields_ = [("solutions", C.POINTER(C.c_double)), ("residuals", C.POINTER(C.c_double)),
                ("per_column_relative_residual", C.POINTER(C.c_double)),
                ("converged", C.POINTER(C.c_int)), ("iterations_used", C.c_int)]


class _TrainCfg(C.Structure):
    _fields_ = [("steps", C.c_int), ("learning_rate", C.c_double), ("adam_beta1", C.c_double),
                ("adam_beta2", C.c_double), ("adam_eps", C.c_double), ("num_probes", C.c_int),
                ("probe_distribution", C.c_int), ("mode", C.c_int), ("solver", _SolverCfg),
                ("init_constrained", C.c_double), ("seed", C.c_uint64), ("transform", C.c_int),
                ("estimator", C.c_int), ("rff_features", C.c_int), ("init_noise", C.c_double),
                ("init_signal", C.c_double), ("warm_start_distance", C.c_int),
                ("exact_gradients", C.c_int), ("record_solver_state", C.c_int)]


class _Trace(C.Structure):
    _fields_ = [("raw_params", C.POINTER(C.c_double)),
                ("constrained_params", C.POINTER(C.c_double)),
                ("gradient", C.POINTER(C.c_double)), ("solver_iterations", C.POINTER(C.c_int)),
                ("per_column_relative_residual", C.POINTER(C.c_double)),
                ("warm_start_distance", C.POINTER(C.c_double)),
                ("probe_seed", C.POINTER(C.c_uint64)), ("solver_ms", C.POINTER(C.c_double)),
                ("step_ms", C.POINTER(C.c_double)), ("final_solutions", C.POINTER(C.c_float)),
                ("warm_distance_ms", C.POINTER(C.c_double)), ("solver_init", C.POINTER(C.c_float)),
                ("solver_solutions", C.POINTER(C.c_float))]


EXPORTS = [
    "wgp_last_error", "wgp_version", "wgp_device_count", "wgp_create", "wgp_destroy",
    "wgp_set_hv_impl", "wgp_stream", "wgp_set_data", "wgp_set_hyper", "wgp_set_rows", "wgp_hv",
    "wgp_hv_device", "wgp_solve", "wgp_grad", "wgp_sample_probes", "wgp_rff_probes", "wgp_train",
    "wgp_adam_step", "wgp_derive_seed", "wgp_launch_count", "wgp_profile", "wgp_profile_read",
    "wgp_exact", "wgp_predict", "wgp_split_order", "wgp_hv_cols", "wgp_hv_block", "wgp_ap_factor", "wgp_ap_block_solve",
    "wgp_set_split_global", "wgp_set_cg_precision", "wgp_hv_f64", "wgp_solve_f64",
    "wgp_nccl_unique_id", "wgp_set_comm", "wgp_shard_info", "wgp_shard_rows",
    "wgp_local_group_create", "wgp_local_group_destroy", "wgp_set_comm_local",
]


def library_path() -> str:
    # WGP_LIBRARY: an alternative build of the same library (A/B timing of
    # kernel variants in one process tree); default the in-tree build
    return os.environ.get("WGP_LIBRARY") or os.path.join(_HERE, _LIB_NAME)


def load():
    """Load the in-tree CUDA library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing; run __graft_entry__.build() "
                          "(this package has no CPU fallback)")
    lib = C.CDLL(path)
    lib.wgp_last_error.restype = C.c_char_p
    lib.wgp_version.restype = C.c_char_p
    lib.wgp_stream.restype = C.c_void_p
    lib.wgp_stream.argtypes = [C.c_void_p]
    lib.wgp_launch_count.restype = C.c_uint64
    lib.wgp_profile.argtypes = [C.c_void_p, C.c_int]
    lib.wgp_profile_read.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)]
    lib.wgp_derive_seed.restype = C.c_uint64
    lib.wgp_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    lib.wgp_split_order.argtypes = [C.c_int64, C.c_uint64, C.c_void_p]
    lib.wgp_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.wgp_destroy.argtypes = [C.c_void_p]
    lib.wgp_set_hv_impl.argtypes = [C.c_void_p, C.c_int]
    lib.wgp_set_cg_precision.argtypes = [C.c_void_p, C.c_int]
    lib.wgp_hv_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_solve_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_nccl_unique_id.argtypes = [C.c_void_p]
    lib.wgp_set_comm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    lib.wgp_shard_info.argtypes = [C.c_void_p] + [C.c_void_p] * 5
    lib.wgp_shard_rows.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.wgp_local_group_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    lib.wgp_local_group_destroy.argtypes = [C.c_void_p]
    lib.wgp_set_comm_local.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    lib.wgp_set_data.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
    lib.wgp_set_hyper.argtypes = [C.c_void_p, C.c_void_p]
    lib.wgp_set_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    lib.wgp_hv.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_hv_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64]
    lib.wgp_hv_block.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                 C.c_int, C.c_void_p, C.c_int64]
    lib.wgp_hv_cols.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                C.c_int64, C.c_int, C.c_void_p, C.c_int64]
    lib.wgp_ap_factor.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_ap_block_solve.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.wgp_grad.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_int, C.c_double, C.c_void_p, C.c_void_p]
    lib.wgp_sample_probes.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
    lib.wgp_rff_probes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
    lib.wgp_train.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.wgp_exact.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.wgp_predict.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p]
    lib.wgp_adam_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                  C.c_double, C.c_double, C.c_double, C.c_double]
    _lib = lib
    return lib


def _check(rc: int):
    if rc == WGP_OK:
        return
    msg = load().wgp_last_error().decode()
    if rc == WGP_NUMERICAL:
        raise NumericalError(msg)
    if rc == WGP_INVALID:
        raise ValueError(msg)
    raise DeviceError(msg)


def launch_count() -> int:
    """Kernels this library has launched in this process (all contexts)."""
    return int(load().wgp_launch_count())


def device_count() -> int:
    return int(load().wgp_device_count())


def split_order(n: int, split_seed: int) -> np.ndarray:
    """dataset.cpp:118-124: split_standardize's row permutation (host
    mt19937_64 Fisher-Yates, bitwise the reference's)."""
    out = np.empty(int(n), dtype=np.int64)
    _check(load().wgp_split_order(int(n), C.c_uint64(split_seed), out.ctypes.data))
    return out


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0; broadcast the bytes)."""
    buf = (C.c_ubyte * 128)()
    _check(load().wgp_nccl_unique_id(buf))
    return bytes(buf)


class LocalGroup:
    """TEST INFRASTRUCTURE (wgp_local_group_create): a host-mediated
    communicator for `nranks` contexts on one GPU, each driven by its own
    Python thread (ctypes releases the GIL in library calls)."""

    def __init__(self, nranks: int):
        self._lib = load()
        h = C.c_void_p()
        _check(self._lib.wgp_local_group_create(nranks, C.byref(h)))
        self._h = h
        self.nranks = nranks

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wgp_local_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_rows(n: int, rank: int, nranks: int):
    """The library's row partition (wgp_shard_rows): (own0, own1, ld)."""
    a, b, ld = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    _check(load().wgp_shard_rows(n, rank, nranks, C.byref(a), C.byref(b), C.byref(ld)))
    return int(a.value), int(b.value), int(ld.value)


def derive_seed(base: int, stream: int) -> int:
    """common.hpp:34-36."""
    return int(load().wgp_derive_seed(C.c_uint64(base), C.c_uint64(stream)))


def _f32(a, n=None, what="solve: rhs row count mismatch"):
    """fp32 column-major n x s; with n given, the row count must match (the
    reference's check_shapes, solvers.cpp:58-67, raises the same way)."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float32))
    if a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    if n is not None and a.shape[0] != n:
        raise ValueError(what)
    return a


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- reference types
def _softplus(x):
    return float(np.logaddexp(0.0, x))


def _softplus_inverse(v):
    if not v > 0:
        raise ValueError("softplus_inverse: argument must be positive")
    return float(v + np.log1p(-np.exp(-v))) if v > 0.6931471805599453 else float(np.log(np.expm1(v)))


@dataclass
class Hyperparameters:
    """kernel.hpp:19-50: raw (unconstrained) values [lengthscales..., signal, noise];
    constrained through softplus (reference) or exp (``transform="log"``)."""
    raw: np.ndarray
    transform: str = "softplus"

    @classmethod
    def from_constrained(cls, lengthscales, signal_scale, noise_scale, transform="softplus"):
        inv = (lambda v: float(np.log(v))) if transform == "log" else _softplus_inverse
        vals = [*np.atleast_1d(lengthscales), signal_scale, noise_scale]
        if transform == "log" and any(not v > 0 for v in vals):
            raise ValueError("log transform: argument must be positive")
        return cls(np.array([inv(float(v)) for v in vals]), transform)

    @classmethod
    def constant_constrained(cls, input_dim, value, transform="softplus"):
        return cls.from_constrained(np.full(input_dim, value), value, value, transform)

    @property
    def input_dim(self):
        return self.raw.size - 2

    @property
    def num_params(self):
        return self.raw.size

    def to_constrained_vector(self):
        f = np.exp if self.transform == "log" else np.vectorize(_softplus)
        return np.asarray(f(self.raw), dtype=np.float64)

    def lengthscales(self):
        return self.to_constrained_vector()[:-2]

    def signal_scale(self):
        return float(self.to_constrained_vector()[-2])

    def noise_scale(self):
        return float(self.to_constrained_vector()[-1])


@dataclass
class SolverConfig:
    """solvers.hpp:20-32 (identical defaults)."""
    kind: str = "cg"
    tol_mean: float = 0.01
    tol_samples: float = 0.1
    max_iterations: int = 0
    block_size: int = 2000
    minibatch_size: int = 1000
    momentum: float = 0.9
    learning_rate: float = 10.0
    seed: int = 0

    def validate(self):  # solvers.cpp:31-37
        if not (0 < self.tol_mean < 1) or not (0 < self.tol_samples < 1):
            raise ValueError("SolverConfig: tolerances must lie in (0, 1)")
        if self.block_size < 1:
            raise ValueError("SolverConfig: block_size must be >= 1")
        if self.minibatch_size < 1:
            raise ValueError("SolverConfig: minibatch_size must be >= 1")
        if self.max_iterations < 0:
            raise ValueError("SolverConfig: max_iterations must be >= 0")

    def _c(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown solver kind: {self.kind}")
        return _SolverCfg(_KINDS[self.kind], self.tol_mean, self.tol_samples, self.max_iterations,
                          self.block_size, self.minibatch_size, self.momentum,
                          self.learning_rate, self.seed)


@dataclass
class SolveState:
    """solvers.hpp:38-46."""
    solutions: np.ndarray
    residuals: np.ndarray
    per_column_relative_residual: np.ndarray
    converged: List[bool]
    iterations_used: int

    def all_converged(self):
        return all(self.converged)


@dataclass
class GradientEstimate:
    """estimator.hpp:36-41."""
    quadratic_term: np.ndarray
    trace_term: np.ndarray

    def gradient(self):
        return self.quadratic_term - self.trace_term


@dataclass
class TrainConfig:
    """optimizer.hpp:23-38 plus the BASELINE extensions (transform, estimator,
    rff_features, init_noise, init_signal)."""
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
    warm_start_distance: bool = True
    exact_gradients: bool = False  # train_exact (optimizer.hpp:83-86)
    record_solver_state: bool = False  # keep per-step init / solutions (optimizer.hpp:35)

    def validate(self):
        if self.steps < 1:
            raise ValueError("TrainConfig: steps must be >= 1")
        if self.num_probes < 1:
            raise ValueError("TrainConfig: num_probes must be >= 1")
        self.solver.validate()

    def _c(self):
        return _TrainCfg(self.steps, self.learning_rate, self.adam_beta1, self.adam_beta2,
                         self.adam_eps, self.num_probes, _DISTS[self.probe_distribution],
                         _MODES[self.mode], self.solver._c(), self.init_constrained, self.seed,
                         _TRANSFORMS[self.transform], _ESTIMATORS[self.estimator],
                         self.rff_features, self.init_noise, self.init_signal,
                         int(self.warm_start_distance), int(self.exact_gradients),
                         int(self.record_solver_state))


@dataclass
class StepRecord:
    """optimizer.hpp:54-67 (device timings instead of wall clock)."""
    step: int
    raw_params: np.ndarray
    constrained_params: np.ndarray
    gradient: np.ndarray
    solver_iterations: int
    solver_ms: float
    step_ms: float
    per_column_relative_residual: np.ndarray
    warm_start_distance: float
    probe_seed: int
    warm_distance_ms: float = 0.0  # device time of the warm-start-distance H.V (inside step_ms)
    solver_init: Optional[np.ndarray] = None       # with record_solver_state (optimizer.hpp:65)
    solver_solutions: Optional[np.ndarray] = None  # (optimizer.hpp:66)


@dataclass
class OptTrace:
    """optimizer.hpp:69-76."""
    steps: List[StepRecord]
    final_solutions: Optional[np.ndarray] = None

    def back(self):
        return self.steps[-1]

    def total_solver_iterations(self, first=1, last=1 << 30):
        return sum(r.solver_iterations for r in self.steps if first <= r.step <= last)

    def final_hyperparameters(self, input_dim, transform="softplus"):
        """optimizer.cpp:67-70: the last step's parameters."""
        c = np.asarray(self.steps[-1].constrained_params)
        return Hyperparameters.from_constrained(c[:input_dim], c[input_dim], c[input_dim + 1], transform)

    def raw_params(self):
        return np.array([r.raw_params for r in self.steps])


# ----------------------------------------------------------------- context
class Context:
    """One device context (C-ABI ``wgp_ctx``): owns the stream, the points and
    every device buffer, including the warm-start state of ``train``."""

    def __init__(self, device: int = 0, hv_impl: str = "tc", cg_precision: str = "f64"):
        self._lib = load()
        h = C.c_void_p()
        _check(self._lib.wgp_create(device, C.byref(h)))
        self._h = h
        self.n = 0
        self.d = 0
        self.set_hv_impl(hv_impl)
        self.set_cg_precision(cg_precision)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wgp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self) -> int:
        return int(self._lib.wgp_stream(self._h) or 0)

    def profile(self, enable: bool = True):
        """Bracket every tensor-core H.V kernel launch with CUDA events."""
        _check(self._lib.wgp_profile(self._h, int(enable)))

    def profile_read(self):
        """(summed kernel ms, launches) since the last read; resets."""
        ms, k = C.c_double(0.0), C.c_int(0)
        _check(self._lib.wgp_profile_read(self._h, C.byref(ms), C.byref(k)))
        return float(ms.value), int(k.value)

    def set_hv_impl(self, impl: str):
        if impl not in _HV_IMPLS:
            raise ValueError(f"unknown H.V implementation {impl!r}; one of {sorted(_HV_IMPLS)}")
        _check(self._lib.wgp_set_hv_impl(self._h, _HV_IMPLS[impl]))

    def set_cg_precision(self, precision: str):
        """CG on fp64 state over the fp64-accumulating operator ("f64", default:
        the reference's iteration counts) or on fp32 state over the H.V engine
        ("f32": faster, more iterations on ill-conditioned systems)."""
        if precision not in _CG_PRECISIONS:
            raise ValueError(f"unknown CG precision {precision!r}; one of {sorted(_CG_PRECISIONS)}")
        _check(self._lib.wgp_set_cg_precision(self._h, _CG_PRECISIONS[precision]))

    def set_comm(self, rank: int, nranks: int, unique_id: bytes):
        """Attach an NCCL communicator (one process per GPU): the context's
        solvers, H.V and outer loop then run row-sharded over the ranks
        (wgp_set_comm; call before set_data)."""
        if len(unique_id) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(self._lib.wgp_set_comm(self._h, rank, nranks, buf))

    def set_comm_local(self, group: "LocalGroup", rank: int):
        """Join a LocalGroup as `rank` (test infrastructure: multi-rank sharding
        on one GPU; call before set_data)."""
        _check(self._lib.wgp_set_comm_local(self._h, group._h, rank))

    def shard_info(self):
        """(rank, nranks, own0, own1, ld) of the context's row sharding."""
        r, nr = C.c_int(0), C.c_int(0)
        a, b, ld = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        _check(self._lib.wgp_shard_info(self._h, C.byref(r), C.byref(nr), C.byref(a), C.byref(b), C.byref(ld)))
        return int(r.value), int(nr.value), int(a.value), int(b.value), int(ld.value)

    def set_data(self, X):
        X = _f32(X)
        self.n, self.d = X.shape
        self._X = X
        _check(self._lib.wgp_set_data(self._h, _ptr(X), X.shape[0], X.shape[1]))

    def set_hyper(self, constrained):
        c = np.ascontiguousarray(constrained, dtype=np.float64)
        if c.size != self.d + 2:
            raise ValueError("Hyperparameters: raw vector must have input_dim + 2 entries")
        _check(self._lib.wgp_set_hyper(self._h, _ptr(c)))

    def set_rows(self, r0: int, r1: int):
        _check(self._lib.wgp_set_rows(self._h, r0, r1))

    def hv(self, V, rows=None):
        """H V for host V (n x s) -> host (rows x s)."""
        V = _f32(V, self.n, "hv: V row count mismatch")
        m = self.n if rows is None else rows
        out = np.empty((m, V.shape[1]), dtype=np.float32, order="F")
        _check(self._lib.wgp_hv(self._h, _ptr(V), V.shape[1], _ptr(out)))
        return out

    def hv_f64(self, V, rows=None):
        """fp64 H V (the fp64 CG operator) for host V (n x s) -> host fp64 (rows x s)."""
        V = np.asfortranarray(np.asarray(V, dtype=np.float64))
        if V.ndim == 1:
            V = V.reshape(-1, 1, order="F")
        if V.shape[0] != self.n:
            raise ValueError("hv: V row count mismatch")
        m = self.n if rows is None else rows
        out = np.empty((m, V.shape[1]), dtype=np.float64, order="F")
        _check(self._lib.wgp_hv_f64(self._h, _ptr(V), V.shape[1], _ptr(out)))
        return out

    def hv_device(self, V_ptr: int, ldv: int, s: int, out_ptr: int, ldo: int):
        """Device-pointer H V on the context stream (asynchronous)."""
        _check(self._lib.wgp_hv_device(self._h, C.c_void_p(V_ptr), ldv, s, C.c_void_p(out_ptr), ldo))

    def hv_block_device(self, i0: int, i1: int, j0: int, j1: int, V_ptr: int, ldv: int, s: int, out_ptr: int,
                        ldo: int) -> None:
        """out = H[i0:i1, j0:j1] V (wgp_hv_block; device pointers, column-major,
        V rows j0.., out rows i0..)."""
        _check(self._lib.wgp_hv_block(self._h, i0, i1, j0, j1, C.c_void_p(V_ptr), ldv, s, C.c_void_p(out_ptr), ldo))

    def hv_cols_device(self, V_ptr: int, ldv: int, s: int, j0: int, j1: int, out_ptr: int, ldo: int,
                       mode: int = 0, B_ptr: int = 0, ldb: int = 0):
        """Device-pointer column block over the set_rows rows: out = (mode 0) H[rows, j0:j1] V,
        (1) B - that, (2) out -= that; V holds the block's j1 - j0 rows, B / out the local rows."""
        _check(self._lib.wgp_hv_cols(self._h, C.c_void_p(V_ptr), ldv, s, j0, j1, C.c_void_p(out_ptr), ldo, mode,
                                     C.c_void_p(B_ptr or None), ldb))

    def set_split_global(self, flag: bool):
        """J splits keyed on the global n (bitwise shard-invariant rows) or on the local rows."""
        _check(self._lib.wgp_set_split_global(self._h, int(bool(flag))))

    def ap_factor(self, block_size: int) -> int:
        """Factor and invert every diagonal block (solvers.cpp:151-165); returns the block count."""
        nb = C.c_int64(0)
        _check(self._lib.wgp_ap_factor(self._h, int(block_size), C.byref(nb)))
        return int(nb.value)

    def ap_block_solve_device(self, block: int, Rb_ptr: int, s: int, delta_ptr: int):
        """delta_b = H_bb^-1 R_b (fp64 device, size x s column-major)."""
        _check(self._lib.wgp_ap_block_solve(self._h, int(block), C.c_void_p(Rb_ptr), s, C.c_void_p(delta_ptr)))

    def solve(self, rhs, config: SolverConfig, init=None) -> SolveState:
        rhs = _f32(rhs, self.n)
        n, s = rhs.shape
        if s < 1:
            raise ValueError("solve: rhs needs at least one column")
        if init is not None:
            init = _f32(init)
            if init.shape != rhs.shape:
                raise ValueError("solve: init shape must match rhs")
        sol = np.empty((n, s), dtype=np.float32, order="F")
        res = np.empty((n, s), dtype=np.float32, order="F")
        pcr = np.empty(s)
        conv = np.zeros(s, dtype=np.int32)
        st = _SolveState(sol.ctypes.data_as(C.POINTER(C.c_float)),
                         res.ctypes.data_as(C.POINTER(C.c_float)),
                         pcr.ctypes.data_as(C.POINTER(C.c_double)),
                         conv.ctypes.data_as(C.POINTER(C.c_int)), 0)
        cfg = config._c()
        _check(self._lib.wgp_solve(self._h, C.byref(cfg), _ptr(rhs),
                                   _ptr(init) if init is not None else None, s, C.byref(st)))
        return SolveState(sol, res, pcr, [bool(c) for c in conv], st.iterations_used)

    def solve_f64(self, rhs, config: SolverConfig, init=None) -> SolveState:
        """wgp_solve_f64: fp64 rhs / init / solutions (the reference's MatrixXd);
        with fp64 CG nothing is rounded to fp32 on the way."""
        def f64(a):
            a = np.asfortranarray(np.asarray(a, dtype=np.float64))
            return a.reshape(-1, 1, order="F") if a.ndim == 1 else a
        rhs = f64(rhs)
        if rhs.shape[0] != self.n:
            raise ValueError("solve: rhs row count mismatch")
        n, s = rhs.shape
        if s < 1:
            raise ValueError("solve: rhs needs at least one column")
        if init is not None:
            init = f64(init)
            if init.shape != rhs.shape:
                raise ValueError("solve: init shape must match rhs")
        sol = np.empty((n, s), order="F")
        res = np.empty((n, s), order="F")
        pcr = np.empty(s)
        conv = np.zeros(s, dtype=np.int32)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        st = _SolveStateF64(dp(sol), dp(res), dp(pcr), conv.ctypes.data_as(C.POINTER(C.c_int)), 0)
        cfg = config._c()
        _check(self._lib.wgp_solve_f64(self._h, C.byref(cfg), _ptr(rhs),
                                       _ptr(init) if init is not None else None, s, C.byref(st)))
        return SolveState(sol, res, pcr, [bool(c) for c in conv], st.iterations_used)

    def predict(self, X_test, y, config: "SolverConfig" = None) -> "PredictiveDistribution":
        """predict (exact.cpp:52-77) through iterative solves (`config`, default
        CG at tolerance 1e-4) at the context's hyperparameters."""
        config = config or SolverConfig(kind="cg", tol_mean=1e-4, tol_samples=1e-4, max_iterations=10000)
        config.validate()
        Xt = _f32(X_test)
        m = Xt.shape[0]
        if m and Xt.shape[1] != self.d:
            raise ValueError("predict: input dimension mismatch")
        y = np.ascontiguousarray(y, dtype=np.float32).ravel()
        if y.size != self.n:
            raise ValueError("predict: X_train and y disagree on n")
        mean = np.zeros(m)
        var = np.zeros(m)
        nv = C.c_double(0.0)
        cfg = config._c()
        _check(self._lib.wgp_predict(self._h, _ptr(Xt), m, _ptr(y), C.byref(cfg), _ptr(mean), _ptr(var),
                                     C.byref(nv)))
        return PredictiveDistribution(mean, var, float(nv.value))

    def exact_mll(self, y, raw, transform="softplus"):
        """exact_mll (exact.cpp:25-36) on the device in fp64 for the context's data."""
        return self._exact(y, raw, transform, want_grad=False)[0]

    def exact_gradient(self, y, raw, transform="softplus"):
        """exact_gradient (exact.cpp:38-50): raw-space gradient of the exact MLL."""
        return self._exact(y, raw, transform, want_grad=True)[1]

    def _exact(self, y, raw, transform, want_grad):
        y = np.ascontiguousarray(y, dtype=np.float32).ravel()
        if y.size != self.n:
            raise ValueError(("exact_gradient" if want_grad else "exact_mll") + ": X and y disagree on n")
        r = np.ascontiguousarray(raw, dtype=np.float64)
        if r.size != self.d + 2:
            raise ValueError("Hyperparameters: raw vector must have input_dim + 2 entries")
        mll = C.c_double(0.0)
        g = np.zeros(self.d + 2)
        _check(self._lib.wgp_exact(self._h, _TRANSFORMS[transform], _ptr(r), _ptr(y), C.byref(mll),
                                   _ptr(g) if want_grad else None))
        return float(mll.value), g

    def grad(self, transform, raw, vy, L, R, coef_b):
        raw = np.ascontiguousarray(raw, dtype=np.float64)
        vy = np.ascontiguousarray(vy, dtype=np.float32)
        if vy.size != self.n:
            raise ValueError("assemble_gradient_streamed: shape mismatch")
        L = _f32(L, self.n, "assemble_gradient_streamed: shape mismatch")
        R = _f32(R, self.n, "assemble_gradient_streamed: shape mismatch")
        if L.shape[1] != R.shape[1]:
            raise ValueError("assemble_gradient_streamed: shape mismatch")
        oa, ob = np.empty(raw.size), np.empty(raw.size)
        _check(self._lib.wgp_grad(self._h, _TRANSFORMS.get(transform, transform), _ptr(raw),
                                  _ptr(vy), _ptr(L), _ptr(R), L.shape[1], coef_b, _ptr(oa), _ptr(ob)))
        return oa, ob

    def rff_probes(self, F, s, seed):
        out = np.empty((self.n, s), dtype=np.float32, order="F")
        _check(self._lib.wgp_rff_probes(self._h, F, s, C.c_uint64(seed), _ptr(out)))
        return out

    def train(self, y, config: TrainConfig) -> OptTrace:
        config.validate()
        y = np.ascontiguousarray(y, dtype=np.float32).ravel()
        if y.size != self.n:
            raise ValueError("train: X and y disagree on n")
        T, p, sp = config.steps, self.d + 2, config.num_probes + 1
        arr = dict(raw=np.zeros((T, p)), con=np.zeros((T, p)), grad=np.zeros((T, p)),
                   it=np.zeros(T, dtype=np.int32), pcr=np.zeros((T, sp)), wsd=np.zeros(T),
                   seed=np.zeros(T, dtype=np.uint64), sms=np.zeros(T), tms=np.zeros(T),
                   fin=np.zeros((self.n, sp), dtype=np.float32, order="F"), wms=np.zeros(T))
        rec = config.record_solver_state
        if rec:  # steps x (n x sp column-major)
            arr["sinit"] = np.zeros((T, sp, self.n), dtype=np.float32)
            arr["ssol"] = np.zeros((T, sp, self.n), dtype=np.float32)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
        tr = _Trace(dp(arr["raw"]), dp(arr["con"]), dp(arr["grad"]),
                    arr["it"].ctypes.data_as(C.POINTER(C.c_int)), dp(arr["pcr"]), dp(arr["wsd"]),
                    arr["seed"].ctypes.data_as(C.POINTER(C.c_uint64)), dp(arr["sms"]),
                    dp(arr["tms"]), fp(arr["fin"]), dp(arr["wms"]),
                    fp(arr["sinit"]) if rec else None, fp(arr["ssol"]) if rec else None)
        cfg = config._c()
        _check(self._lib.wgp_train(self._h, _ptr(y), C.byref(cfg), C.byref(tr)))
        steps = [StepRecord(t + 1, arr["raw"][t].copy(), arr["con"][t].copy(), arr["grad"][t].copy(),
                            int(arr["it"][t]), float(arr["sms"][t]), float(arr["tms"][t]),
                            arr["pcr"][t].copy(), float(arr["wsd"][t]), int(arr["seed"][t]),
                            float(arr["wms"][t]),
                            arr["sinit"][t].T.copy(order="F") if rec else None,
                            arr["ssol"][t].T.copy(order="F") if rec else None)
                 for t in range(T)]
        return OptTrace(steps, arr["fin"])


# ----------------------------------------------------------------- reference-style free functions
class KernelOperator:
    """Matrix-free stand-in for the dense ``H`` argument of ``solve``
    (solvers.hpp:50-55): the inputs X and the hyperparameters, never H."""

    def __init__(self, X, hyper: Hyperparameters, device: int = 0, ctx: Optional[Context] = None,
                 hv_impl: str = "tc"):
        self.ctx = ctx or Context(device, hv_impl)
        self.ctx.set_data(X)
        self.hyper = hyper
        self.ctx.set_hyper(hyper.to_constrained_vector())

    @property
    def n(self):
        return self.ctx.n

    def matvec(self, V):
        return self.ctx.hv(V)


def solve(op: KernelOperator, rhs, config: SolverConfig, init=None) -> SolveState:
    """solvers.cpp:265-279 over the matrix-free operator."""
    config.validate()
    return op.ctx.solve(rhs, config, init)


def train(X, y, config: TrainConfig, device: int = 0, ctx: Optional[Context] = None,
          hv_impl: str = "tc") -> OptTrace:
    """optimizer.cpp:175-177 (run_loop :81-171) on the device."""
    X = _f32(X)
    if X.shape[0] < 1:
        raise ValueError("train: dataset is empty")
    if np.asarray(y).size != X.shape[0]:
        raise ValueError("train: X and y disagree on n")
    ctx = ctx or Context(device, hv_impl)
    ctx.set_data(X)
    return ctx.train(y, config)


@dataclass
class PredictiveDistribution:
    """exact.hpp PredictiveDistribution: latent means / variances + noise variance."""
    means: np.ndarray
    variances: np.ndarray
    noise_variance: float = 0.0


@dataclass
class TestMetrics:
    """exact.hpp TestMetrics."""
    rmse: float = 0.0
    mean_loglik: float = 0.0


def test_metrics(pred: PredictiveDistribution, y_test) -> TestMetrics:
    """exact.cpp:79-92: RMSE and mean predictive log-likelihood (latent
    variance + noise variance)."""
    y_test = np.asarray(y_test, dtype=np.float64).ravel()
    if pred.means.size != y_test.size:
        raise ValueError("test_metrics: prediction/target length mismatch")
    if y_test.size == 0:
        return TestMetrics()
    err = pred.means - y_test
    var = pred.variances + pred.noise_variance
    return TestMetrics(float(np.sqrt(np.mean(err ** 2))),
                       float(np.mean(-0.5 * (np.log(var) + 1.8378770664093453) - 0.5 * err ** 2 / var)))


def predict(X_train, y, X_test, hyper: "Hyperparameters", config: "SolverConfig" = None, device: int = 0,
            ctx: Optional[Context] = None) -> PredictiveDistribution:
    """exact.cpp:52-77 on the device through iterative solves."""
    ctx = ctx or Context(device)
    ctx.set_data(_f32(X_train))
    ctx.set_hyper(hyper.to_constrained_vector())
    return ctx.predict(X_test, y, config)


def train_exact(X, y, config: TrainConfig, device: int = 0, ctx: Optional[Context] = None) -> OptTrace:
    """optimizer.cpp:179-181: the same loop with the exact Cholesky gradient
    (fp64, dense, on the device; n <= 20000)."""
    import dataclasses
    return train(X, y, dataclasses.replace(config, exact_gradients=True), device, ctx)


def exact_mll(X, y, hyper: "Hyperparameters", device: int = 0, ctx: Optional[Context] = None) -> float:
    """exact.cpp:25-36 on the device (fp64)."""
    ctx = ctx or Context(device)
    ctx.set_data(_f32(X))
    return ctx.exact_mll(y, hyper.raw, hyper.transform)


def exact_gradient(X, y, hyper: "Hyperparameters", device: int = 0, ctx: Optional[Context] = None) -> np.ndarray:
    """exact.cpp:38-50 on the device (fp64): raw-space gradient."""
    ctx = ctx or Context(device)
    ctx.set_data(_f32(X))
    return ctx.exact_gradient(y, hyper.raw, hyper.transform)


def sample_probes(n: int, s: int, distribution: str = "gaussian", seed: int = 0) -> np.ndarray:
    """estimator.cpp:21-37 (host mt19937_64; values of the reference rounded to fp32)."""
    out = np.empty((n, s), dtype=np.float32, order="F")
    _check(load().wgp_sample_probes(n, s, _DISTS[distribution], C.c_uint64(seed), _ptr(out)))
    return out


def assemble_gradient_streamed(op: KernelOperator, v_y, probe_solves, probes) -> GradientEstimate:
    """estimator.cpp:63-82: Frobenius contractions with A = v_y v_y^T / 2 and
    B = V Z^T / (2s), streamed by the fused gradient kernel."""
    s = np.asarray(probes).reshape(op.n, -1).shape[1]
    qa, qb = op.ctx.grad(op.hyper.transform, op.hyper.raw, v_y, probe_solves, probes, 0.5 / s)
    op.ctx.set_hyper(op.hyper.to_constrained_vector())
    return GradientEstimate(qa, qb)


def warm_start_distance(op: KernelOperator, init, solution) -> float:
    """estimator.cpp:84-95, evaluated with the device operator."""
    D = _f32(init) - _f32(solution)
    HD = op.matvec(D).astype(np.float64)
    return float(np.sqrt(max(np.mean(np.sum(D * HD, axis=0)) / op.n, 0.0)))


def adam_step(raw, grad, m, v, t, config: TrainConfig = TrainConfig()):
    """optimizer.cpp:48-65 (in place on float64 arrays)."""
    for a in (raw, m, v):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("adam_step: float64 contiguous arrays required")
    g = np.ascontiguousarray(grad, dtype=np.float64)
    if not (g.size == raw.size == m.size == v.size):
        raise ValueError("adam_step: shape mismatch")
    _check(load().wgp_adam_step(_ptr(raw), _ptr(g), _ptr(m), _ptr(v), raw.size, t,
                                config.learning_rate, config.adam_beta1, config.adam_beta2,
                                config.adam_eps))
