"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-side pieces (probe RNG, seeds, Adam) match the
oracle bitwise.  No compute entry point is called without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2405_18328_b200 as wg
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "warmgp_b200.h")).read()
    return sorted(set(re.findall(r"\b(wgp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(wg.library_path())
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(wg.EXPORTS)


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {wg.library_path()} 2>&1").read()
    assert "sm_100a" in out


def test_no_device_is_a_loud_error():
    if wg.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(wg.DeviceError, match="no CPU fallback"):
        wg.Context(0)


def test_probes_bitwise_match_reference_rng():
    for dist in ("gaussian", "rademacher"):
        a = wg.sample_probes(257, 5, dist, 42)
        b = orc.sample_probes(257, 5, dist, 42)
        assert np.array_equal(a, b.astype(np.float32))


def test_derive_seed_matches():
    for b, s in [(0, 1), (12, 7), (99, 0x736F6C7665)]:
        assert wg.derive_seed(b, s) == orc.derive_seed(b, s)


def test_adam_matches_oracle():
    rng = np.random.default_rng(0)
    raw1, m1, v1 = np.zeros(5), np.zeros(5), np.zeros(5)
    raw2, m2, v2 = np.zeros(5), np.zeros(5), np.zeros(5)
    for t in range(1, 30):
        g = rng.standard_normal(5)
        wg.adam_step(raw1, g, m1, v1, t)
        orc.adam_step(raw2, g, m2, v2, t)
    assert np.array_equal(raw1, raw2)
    with pytest.raises(wg.NumericalError, match="step 3"):
        wg.adam_step(raw1, np.array([np.nan] * 5), m1, v1, 3)


def test_config_validation_messages():
    with pytest.raises(ValueError, match="tolerances"):
        wg.SolverConfig(tol_mean=0.0).validate()
    with pytest.raises(ValueError, match="block_size"):
        wg.SolverConfig(block_size=0).validate()
    with pytest.raises(ValueError, match="steps"):
        wg.TrainConfig(steps=0).validate()


def test_hyperparameters_roundtrip():
    for tr in ("softplus", "log"):
        h = wg.Hyperparameters.from_constrained([0.5, 2.0], 1.3, 0.1, tr)
        assert np.allclose(h.to_constrained_vector(), [0.5, 2.0, 1.3, 0.1], rtol=1e-12)
        assert h.input_dim == 2 and h.num_params == 4
