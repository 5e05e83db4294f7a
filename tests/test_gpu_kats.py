"""Remaining known-answer tests of the reference (SURVEY 8c pins) restated on
the GPU: identities and inverses, the nc = 1 bitwise degeneracy of every
operator (mc_ops.hpp:10, T/test_mct.cpp:499-525), accuracy claims checked
against exact rational arithmetic, and the MC-SGD tiny-update pin.
"""
from fractions import Fraction

import numpy as np
import pytest

from mcgen import assert_bits, config_values, split

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _exact(x):
    return sum(Fraction(float(c)) for c in x)


def test_identities_and_inverses(gr):
    """T/test_mct.cpp:197-241, 243-272, 302-348: scaling_n(x, 1) = x and
    x * 0 = 0; add_mcn(x, 0) = x, add_mcn(x, -x) = 0; mul_mcn(x, 1) = x and
    the zero fast path."""
    rng = np.random.default_rng(5)
    x = split(config_values(rng, 4096), 2, np.float32)
    one = np.ones(4096, np.float32)
    assert_bits(gr.run("scaling_n", x, one), x, "scaling_n(x, 1)")
    assert_bits(gr.run("scaling_n", x, np.zeros(4096, np.float32)), np.zeros_like(x), "scaling_n(x, 0)")
    assert_bits(gr.run("add_mcn", x, np.zeros_like(x)), x, "add_mcn(x, 0)")
    assert_bits(gr.run("add_mcn", x, -x), np.zeros_like(x), "add_mcn(x, -x)")
    ones = np.zeros_like(x)
    ones[:, 0] = 1.0
    assert_bits(gr.run("mul_mcn", x, ones), x, "mul_mcn(x, 1)")
    assert_bits(gr.run("mul_mcn", x, np.zeros_like(x)), np.zeros_like(x), "mul_mcn(x, 0)")
    assert_bits(gr.run("mul_mcn", np.zeros_like(x), x), np.zeros_like(x), "mul_mcn(0, x)")


def test_division_pins(gr):
    """T/test_mct.cpp:274-300, 421-436: 1/3 within 2^-45, x/x within 2^-44 of
    1, div_n(1, 3) == div_mcn(1, 3) bitwise, (1/3) * 3 within 2^-45."""
    f = np.float32
    third = gr.run("div_mcn", np.array([[1.0, 0.0]], f), np.array([[3.0, 0.0]], f))
    assert abs(_exact(third[0]) - Fraction(1, 3)) <= Fraction(1, 3) * Fraction(1, 2**45)
    assert_bits(gr.run("div_n", np.array([1.0], f), np.array([[3.0, 0.0]], f)), third, "div_n(1, 3)")
    back = gr.run("scaling_n", third, np.array([3.0], f))
    assert abs(_exact(back[0]) - 1) <= Fraction(1, 2**45)
    rng = np.random.default_rng(6)
    x = split(config_values(rng, 2000) + 0.5, 2, f)
    q = gr.run("div_mcn", x, x)
    assert max(abs(_exact(r) - 1) for r in q) <= Fraction(1, 2**44)


def test_mul_fast_vs_slow_and_add_gain(gr):
    """T/test_mct.cpp:253-272, 330-348: mul_mcn (fast) within 2^-45 of
    mul_mcn_slow; add_mcn at nc = 2 at least 10^3 times more accurate than
    nc = 1 (median relative error against exact sums)."""
    rng = np.random.default_rng(7)
    n = 3000
    xv, yv = config_values(rng, n), config_values(rng, n) + 0.5
    x2, y2 = split(xv, 2, np.float32), split(yv, 2, np.float32)
    fast, slow = gr.run("mul_mcn", x2, y2), gr.run("mul_mcn_slow", x2, y2)
    for a, b in zip(fast[:500], slow[:500]):
        ea, eb = _exact(a), _exact(b)
        assert abs(ea - eb) <= abs(eb) * Fraction(1, 2**45)
    x1, y1 = split(xv, 1, np.float32), split(yv, 1, np.float32)
    s2, s1 = gr.run("add_mcn", x2, y2), gr.run("add_mcn", x1, y1)
    e2, e1 = [], []
    for i in range(400):
        want = _exact(x2[i]) + _exact(y2[i])
        if want == 0:
            continue
        e2.append(abs(float((_exact(s2[i]) - want) / want)))
        e1.append(abs(float((_exact(s1[i]) - (_exact(x1[i]) + _exact(y1[i]))) / want)) + 1e-30)
    assert np.median(e2) * 1e3 <= max(np.median(e1), 2.0**-24 / 4)


@pytest.mark.parametrize("bits", [16, 32, 64])
def test_single_component_is_plain_arithmetic(gr, bits):
    """nc = 1 degenerates bitwise to working-precision arithmetic for every
    operator (mc_ops.hpp:10; T/test_mct.cpp:499-525)."""
    dt = {16: np.float16, 32: np.float32, 64: np.float64}[bits]
    rng = np.random.default_rng(8 + bits)
    lo, hi = (-4, 4) if bits == 16 else (-8, 8)
    a = config_values(rng, 5000, lo, hi).astype(dt)
    b = (config_values(rng, 5000, lo, hi) + 0.5).astype(dt)
    x, y = a[:, None], b[:, None]
    with np.errstate(all="ignore"):
        assert_bits(gr.run("add_mcn", x, y)[:, 0], a + b, "add")
        assert_bits(gr.run("mul_mcn", x, y)[:, 0], a * b, "mul")
        assert_bits(gr.run("mul_mcn_slow", x, y)[:, 0], a * b, "mul_slow")
        assert_bits(gr.run("div_mcn", x, y)[:, 0], a / b, "div")
        assert_bits(gr.run("div_n", a, y)[:, 0], a / b, "div_n")
        assert_bits(gr.run("square_mcn", x)[:, 0], a * a, "square")
        assert_bits(gr.run("grow_expn", x, b)[:, 0], a + b, "grow")
        assert_bits(gr.run("scaling_n", x, b)[:, 0], a * b, "scaling")


def test_sgd_tiny_update_survives(gr):
    """T/test_optim.cpp:49-61: an MC-SGD step on a binary16 nc = 2 weight 1.0
    with update 2^-20 keeps it exactly (1, -2^-20): the second component
    carries what binary16 alone would lose."""
    w = np.array([[1.0, 0.0]], np.float16)
    out = gr.run("grow_expn", w, np.array([-(2.0**-20)], np.float16))
    assert out[0, 0] == 1.0 and out[0, 1] == np.float16(-(2.0**-20))
    plain = gr.run("grow_expn", w[:, :1], np.array([-(2.0**-20)], np.float16))
    assert plain[0, 0] == 1.0  # nc = 1: the update is lost
