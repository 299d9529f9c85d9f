"""CPU restatement of the int8-slice fp64 product of csrc/hv_i8.cu (DESIGN.md
4.1c), checked with exact Python integers: the balanced base-256 digits of V,
the unsigned bytes of K, the class sums that the int32 tensor-core
accumulators hold, and the bound on what dropping classes 0..2 costs.  (The
device kernel itself is checked against the fp64 oracle and the DMMA engine
in tests/test_gpu_parity.py.)"""
import math

import numpy as np
import pytest

KBYTES, VBYTES, KEEP = 5, 7, 3  # K: 39-bit unsigned; V: 7 balanced signed bytes; classes i + j >= 3


def k_int(k, sf2):
    """rint(k 2^eK) with sf^2 2^eK in [2^38, 2^39) (hv_i8.cu: eK from sf^2's exponent)."""
    e = 38 - (math.frexp(sf2)[1] - 1)
    return int(round(k * 2.0 ** e)), e


def col_exp(vmax):
    """2^e_c putting the column max into [2^53, 2^54) (hv_i8.cu col_exp)."""
    if not vmax > 0 or not math.isfinite(vmax):
        return 0
    return max(-1000, min(1000, 54 - math.frexp(vmax)[1]))


def balanced_digits(v, n=VBYTES):
    """v = sum_j d_j 256^j with d_j in [-128, 127] (least significant first)."""
    out = []
    for _ in range(n):
        d = ((v & 0xFF) ^ 0x80) - 0x80
        out.append(d)
        v = (v - d) >> 8
    return out, v


def test_balanced_digits_roundtrip():
    rng = np.random.default_rng(0)
    for v in list(rng.integers(-2**54, 2**54, 2000)) + [0, 1, -1, 2**54 - 1, -(2**54 - 1), 127, 128, -128, -129]:
        v = int(v)
        d, rest = balanced_digits(v)
        assert rest == 0 and all(-128 <= x <= 127 for x in d)
        assert sum(x * 256 ** j for j, x in enumerate(d)) == v


def test_k_bytes_exact_above_sf2_2m15():
    """K is k itself (exactly) for k >= sf^2 2^-15: fp32 k has 24 significant bits."""
    rng = np.random.default_rng(1)
    for sf2 in (0.37, 1.0, 1.9, 7.5, 2.0 ** -20):
        sf2 = float(np.float32(sf2))
        ks = (sf2 * rng.uniform(2.0 ** -15, 1.0, 500)).astype(np.float32)
        for k in ks:
            K, e = k_int(float(k), sf2)
            assert 0 <= K < 2 ** 39
            assert K * 2.0 ** -e == float(k)
            b = [(K >> (8 * i)) & 0xFF for i in range(KBYTES)]
            assert sum(x * 256 ** i for i, x in enumerate(b)) == K


@pytest.mark.parametrize("seed", [2, 3, 4])
def test_class_sums_reproduce_the_product(seed):
    """sum over kept byte classes w = i + j >= 3 of 256^w sum_{i+j=w} K_i V_j, each
    class an exact integer sum (the int32 accumulators), equals the exact
    integer product up to the dropped classes, which stay below 2^-60 of the
    column's bound |K|max |V|max n; the int32 headroom covers 192 tiles of 64
    points between drains (hv_i8.cu kChunk)."""
    rng = np.random.default_rng(seed)
    n = 300
    sf2 = float(np.float32(rng.uniform(0.3, 2.0)))
    k = (sf2 * rng.uniform(0, 1, n) ** 3).astype(np.float32)
    v = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, n)
    e = col_exp(float(np.abs(v).max()))
    Vi = [int(round(x * 2.0 ** e)) for x in v]
    Ki = [k_int(float(x), sf2)[0] for x in k]
    kb = [[(K >> (8 * i)) & 0xFF for i in range(KBYTES)] for K in Ki]
    vb = [balanced_digits(V)[0] for V in Vi]
    classes = {}
    for a in range(n):
        for i in range(KBYTES):
            for j in range(VBYTES):
                classes[i + j] = classes.get(i + j, 0) + kb[a][i] * vb[a][j]
    exact = sum(K * V for K, V in zip(Ki, Vi))
    assert sum(c * 256 ** w for w, c in classes.items()) == exact
    kept = sum(c * 256 ** w for w, c in classes.items() if w >= KEEP)
    bound = 2 ** 39 * 2 ** 54 * n
    assert abs(kept - exact) <= 2.0 ** -60 * bound
    # one class over 192 tiles of 64 points: <= 5 pairs x 255 x 128 per point
    assert 5 * 255 * 128 * 64 * 192 < 2 ** 31
