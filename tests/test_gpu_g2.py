"""The certified binary32 nc=2 tier (csrc/mcf_g2.cuh) under inputs built to sit
on its margins: exact quotients and reciprocals (remainders exactly zero),
half-ulp ties in the second component, powers of two (where the gap below is
half the gap above), products near the 2^-100 underflow guard and near
overflow, zero second components, mixed with config-0 values.  Every element
must be bit-identical to the oracle whether the shortcut accepts it or the
register / literal path takes over.
"""
import numpy as np
import pytest

from mcgen import assert_bits, config_values, split

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _pairs(rng, n, lo=-8, hi=8):
    """compressed binary32 pairs of several kinds, shuffled together"""
    k = n // 8
    out = []
    out.append(split(config_values(rng, k, lo, hi), 2, np.float32))  # generic
    ints = rng.integers(1, 1 << 12, k) * rng.choice([-1.0, 1.0], k) * np.exp2(rng.integers(-6, 7, k))
    out.append(split(ints, 2, np.float32))  # short significands: exact products / quotients
    p2 = rng.choice([-1.0, 1.0], k) * np.exp2(rng.integers(-20, 21, k).astype(np.float64))
    out.append(split(p2, 2, np.float32))  # powers of two
    # second component exactly half an ulp of an even leading component (a tie)
    c0 = config_values(rng, k, lo, hi).astype(np.float32)
    c0 = (c0.view(np.uint32) & np.uint32(0xFFFFFFFE)).view(np.float32)
    ulp = np.spacing(np.abs(c0)).astype(np.float64)
    t = np.stack([c0, (rng.choice([-0.5, 0.5], k) * ulp).astype(np.float32)], -1)
    out.append(t)
    # powers of two with a second component toward zero (gap below is halved)
    c0 = (rng.choice([-1.0, 1.0], k) * np.exp2(rng.integers(-8, 9, k).astype(np.float64))).astype(np.float32)
    c1 = (-np.sign(c0) * np.spacing(np.abs(c0)) * rng.uniform(0.05, 0.25, k)).astype(np.float32)
    out.append(np.stack([c0, c1], -1))
    out.append(split(config_values(rng, k, -52, -45), 2, np.float32))  # products near 2^-100
    out.append(split(config_values(rng, k, 58, 66), 2, np.float32))  # products near overflow
    z = split(config_values(rng, n - 7 * k, lo, hi), 2, np.float32)
    z[:, 1] = 0
    out.append(z)
    a = np.concatenate(out)
    return a[rng.permutation(a.shape[0])]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_g2_ops_bitwise_on_margins(gr, port, seed):
    rng = np.random.default_rng(900 + seed)
    n = 1 << 17
    x = _pairs(rng, n)
    y = _pairs(rng, n)
    ok = np.abs(y[:, 0]) > 0
    y = y[ok]
    x = x[: y.shape[0]]
    v = x[rng.permutation(x.shape[0]), 0].copy()
    assert_bits(gr.run("scaling_n", x, v), port.scaling_n(x, v), "scaling_n")
    assert_bits(gr.run("add_mcn", x, y), port.add_mcn(x, y), "add_mcn")
    xn = x.copy()
    xn[: y.shape[0] // 2, 0] = -y[: y.shape[0] // 2, 0]  # cancelling leads
    assert_bits(gr.run("add_mcn", xn, y), port.add_mcn(xn, y), "add_mcn cancelling")
    assert_bits(gr.run("square_mcn", x), port.square_mcn(x), "square_mcn")
    assert_bits(gr.run("div_n", v, y), port.div_n(v, y), "div_n")
    assert_bits(gr.run("div_mcn", x, y), port.div_mcn(x, y), "div_mcn")
    assert_bits(gr.run("mul_mcn", x, y), port.mul_mcn(x, y), "mul_mcn")
    # exact quotients: x = k * y with short k, and reciprocals of powers of two
    kk = split(rng.integers(1, 64, y.shape[0]).astype(np.float64), 2, np.float32)
    xy = gr.run("mul_mcn_slow", kk, y)
    assert_bits(gr.run("div_mcn", xy, y), port.div_mcn(xy, y), "div_mcn exact quotients")
    one = np.ones(y.shape[0], np.float32)
    assert_bits(gr.run("div_n", one, y), port.div_n(one, y), "div_n reciprocals")


@pytest.mark.parametrize("seed", [11, 12])
def test_one_digit_division_core_near_exact_quotients(gr, port, seed):
    """The wide tier's one-digit core (mcf_w2.cuh div_core1) replaces the second
    and third quotient digits by the remainder's quotient R and certifies the
    second component against an absolute margin of |R| 2^-42.  Inputs built to
    stress exactly that: x = q y (1 + eps) with q of at most 24 or 48 bits and eps
    from 2^-26 down to 2^-80 and zero (R tiny or zero against q0; the second
    component many binades below it), quotients whose first digit is corrected by
    R (x1 and y1 of opposite effect, |R| about half a step of q0), and divisors
    of Mul-MCN whose reciprocal is nearly a power of two.  Bit-identical to the
    oracle whichever tier ends up taking the element."""
    rng = np.random.default_rng(7700 + seed)
    n = 1 << 16
    y64 = config_values(rng, n, -6, 6)
    y64 += np.sign(y64) * 0.5
    y = split(y64, 2, np.float32)
    yv = y[:, 0].astype(np.float64) + y[:, 1].astype(np.float64)
    bits = rng.choice([6, 12, 24, 30, 48], n)
    q = np.ldexp(rng.integers(1, 1 << 52, n).astype(np.float64), -52) + 1.0
    q = np.ldexp(np.floor(np.ldexp(q, bits - 1)), -(bits - 1)) * rng.choice([-1.0, 1.0], n)
    eps = np.where(rng.uniform(0, 1, n) < 0.2, 0.0, rng.choice([-1.0, 1.0], n) * np.exp2(-rng.uniform(26, 80, n)))
    xl = q.astype(np.longdouble) * yv.astype(np.longdouble) * (1 + eps.astype(np.longdouble))
    x0 = xl.astype(np.float32)
    x1 = (xl - x0.astype(np.longdouble)).astype(np.float32)
    x = np.stack([x0, x1], -1)
    keep = np.isfinite(x).all(-1) & (x0.astype(np.float32) + x1 == x0)
    x, y = x[keep], y[keep]
    assert x.shape[0] > n // 2
    assert_bits(gr.run("div_mcn", x, y), port.div_mcn(x, y), "div_mcn near-exact")
    v = x[:, 0].copy()
    assert_bits(gr.run("div_n", v, y), port.div_n(v, y), "div_n near-exact")
    # first digit corrected by the remainder: y1 at its largest, x1 of the sign that moves the quotient across a step
    y2 = y.copy()
    y2[:, 1] = (np.spacing(np.abs(y2[:, 0])) * rng.choice([-0.5, 0.5, -0.49, 0.49], y2.shape[0])).astype(np.float32)
    y2 = y2[(y2[:, 0] + y2[:, 1]) == y2[:, 0]]
    x2 = x[: y2.shape[0]]
    assert_bits(gr.run("div_mcn", x2, y2), port.div_mcn(x2, y2), "div_mcn half-ulp y1")
    # Mul-MCN: divisors whose reciprocal sits next to a power of two
    p2 = np.exp2(rng.integers(-6, 7, x.shape[0]).astype(np.float64)) * rng.choice([-1.0, 1.0], x.shape[0])
    yn = split(p2 * (1 + rng.choice([-1.0, 1.0], x.shape[0]) * np.exp2(-rng.uniform(20, 60, x.shape[0]))), 2, np.float32)
    assert_bits(gr.run("mul_mcn", x, yn), port.mul_mcn(x, yn), "mul_mcn reciprocal near a power of two")
    assert_bits(gr.run("mul_mcn", x, y), port.mul_mcn(x, y), "mul_mcn near-exact operands")
