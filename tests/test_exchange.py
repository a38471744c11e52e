"""The exact all-reduce encoding of the cross-CTA exchange (DESIGN.md §4.2,
csrc/xchg.cuh): partials split into three 41-bit limbs of a 2^-80
fixed-point number, summed as integers by red.add with an arrival count in
the top 12 bits of every word, and reconstructed from the three integer
sums as (L2*2^2 + L1*2^-39) + L0*2^-80.  The device result must lie within
one ulp of the exact sum of the truncated partials up to the
2048-participant limit (8 GPUs x 148 CTAs fit with room) -- including limbs
near their maximum, where a narrower data field would carry into the
arrival count -- and, being a function of the integer sums alone, not
depend on the order of the partials."""
import ctypes as C
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_1208_0945_b200 import _native

SCALE = 2 ** 80


def _device_sum(vals):
    lib = _native.lib()
    a = np.ascontiguousarray(vals, dtype=np.float64)
    out = C.c_double(0.0)
    st = C.c_int32(-1)
    rc = lib.bsccs_debug_exchange_sum(0, a.ctypes.data_as(C.c_void_p), len(a), C.byref(out), C.byref(st))
    assert rc == 0, _native.lib().bsccs_last_error()
    return out.value, st.value


def _exact(vals):
    total = sum(math.floor(Fraction(float(v)) * SCALE) for v in vals)
    return float(Fraction(total, SCALE))


def _cases(rng):
    top = 2.0 ** 43
    yield "uniform (total overflows)", rng.uniform(0, top, 2048)
    yield "uniform below 2^37", rng.uniform(0, 2.0 ** 37, 2048)
    yield "gradient-like", rng.uniform(0, 1e5, 148)
    yield "tiny", rng.uniform(0, 1e-20, 1184)
    yield "mixed", np.concatenate([rng.uniform(0, 1e6, 500), rng.uniform(0, 1e-12, 500), np.zeros(24)])
    # middle limb (2^-39 .. 2^2 bits) all ones: v = 4 - 2^-39 for every participant
    yield "max middle limb", np.full(2048, 4.0 - 2.0 ** -39)
    # every limb at its maximum
    yield "max limbs", np.full(2048, np.nextafter(top, 0))
    yield "one", np.array([1.0])
    yield "sub-resolution", np.full(300, 2.0 ** -81)


@pytest.mark.gpu
def test_exchange_sum_is_the_correctly_rounded_exact_sum():
    rng = np.random.default_rng(7)
    for name, vals in _cases(rng):
        got, st = _device_sum(vals)
        exp = _exact(vals)
        total_big = sum(math.floor(Fraction(float(v)) * SCALE) for v in vals) >= 2 ** 128
        if total_big:
            assert st == 2, name
            continue
        assert st == 0, name
        assert abs(got - exp) <= math.ulp(exp), (name, got, exp)
        got2, _ = _device_sum(np.ascontiguousarray(vals[::-1]))
        assert got2 == got, name  # order-independent, bit for bit


@pytest.mark.gpu
def test_exchange_range_errors():
    _, st = _device_sum(np.array([1.0, 2.0 ** 43]))
    assert st == 1
    _, st = _device_sum(np.array([-1.0]))
    assert st == 1
    _, st = _device_sum(np.array([np.nan]))
    assert st == 1
    # totals at or above 2^48 cannot be reconstructed: flagged, not wrapped
    _, st = _device_sum(np.full(64, 2.0 ** 42))
    assert st == 2
    got, st = _device_sum(np.full(31, 2.0 ** 43 - 1.0))
    assert st == 0 and abs(got - 31 * (2.0 ** 43 - 1.0)) <= math.ulp(31 * 2.0 ** 43)


def test_exchange_word_capacity():
    """host-side restatement of the static_asserts in xchg.cuh"""
    limb_bits, cnt_shift, max_p = 41, 52, 2048
    assert max_p * (2 ** limb_bits - 1) < 2 ** cnt_shift      # limb sums never reach the count
    assert max_p < 2 ** (64 - cnt_shift)                      # the count holds every arrival
    assert 3 * limb_bits == 123 and 2.0 ** (3 * limb_bits - 80) == 2.0 ** 43
    assert 8 * 148 <= max_p                                    # one node of B200s, one CTA per SM
