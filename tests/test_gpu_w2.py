"""The wide certified tier (csrc/mcf_w2.cuh: Div-MCN, DivN, Mul-MCN and Exp-MCN in
binary64) on inputs placed at its guards and decline paths.  Whether the wide
tier accepts an element or hands it to the binary32 tier / register / literal
path, every element must be bit-identical to the oracle:

* operands at and beyond the +-2^40 window, quotient digits reaching the
  binary32 subnormal range (q2 normal-or-zero guard), products near 2^-86 /
  2^-100 (exact low parts);
* second components too far below the first for x0 + x1 to be one binary64,
  and at the limit (leading bits 28-30 binades apart);
* zeros, exact quotients (q1 = 0), single-component divisors, subnormal
  operands, +-Inf and NaN;
* Exp-MCN over the whole binary32 range of x0 (results near underflow and
  overflow), x1 across the 2^-12 bound of the polynomial, zero and subnormal x1.
"""
import numpy as np
import pytest

import oracle
from mcgen import assert_bits, config_values, split

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _scaled_pairs(rng, n, exps):
    """compressed pairs split from binary64 values m 2^e, e drawn from `exps`"""
    v = rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n) * np.exp2(rng.choice(exps, n).astype(np.float64))
    return split(v, 2, np.float32)


def _far_second(rng, n, gaps):
    """(c0, c1) with c1's leading bit `gap` binades below c0's (gap > 29: c0 + c1 is not one binary64)"""
    c0 = (rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    g = rng.choice(gaps, n)
    c1 = (rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n) * np.exp2(-g.astype(np.float64))).astype(np.float32)
    return np.stack([c0, c1], -1)


def _special(n):
    f = np.float32
    vals = np.array([0.0, -0.0, 1.0, -1.0, 3.0, 0.5, 2.0 ** 40, 2.0 ** -40, 2.0 ** 41, 2.0 ** -41, 1e-45, -1e-45,
                     2.0 ** -126, 2.0 ** -127, 3.4e38, np.inf, -np.inf, np.nan, 7.0, 1.0 / 3.0], dtype=f)
    c0 = np.resize(vals, n)
    return np.stack([c0, np.zeros(n, f)], -1)


@pytest.mark.parametrize("seed", [1, 2])
def test_division_tier_at_its_guards(gr, port, seed):
    rng = np.random.default_rng(4200 + seed)
    n = 1 << 15
    window = np.arange(36, 45)  # across the 2^40 edge on both sides
    cases = []
    # (x, y): y at the window edges, x generic / x at the edges, y generic
    cases.append((split(config_values(rng, n, -8, 8), 2, np.float32), _scaled_pairs(rng, n, window)))
    cases.append((split(config_values(rng, n, -8, 8), 2, np.float32), _scaled_pairs(rng, n, -window)))
    cases.append((_scaled_pairs(rng, n, window), split(config_values(rng, n, -8, 8) + 0.5, 2, np.float32)))
    # small numerators over large divisors: digits down to the subnormal range
    cases.append((_scaled_pairs(rng, n, np.arange(-40, -30)), _scaled_pairs(rng, n, np.arange(30, 41))))
    # second components far below the first (x0 + x1, y0 + y1 not one binary64), and at the limit
    cases.append((_far_second(rng, n, np.arange(25, 60)), _far_second(rng, n, np.arange(25, 60))))
    cases.append((_far_second(rng, n, [28, 29, 30]), _far_second(rng, n, [28, 29, 30])))
    # single-component divisors / numerators, exact quotients
    y1 = split(config_values(rng, n, -8, 8) + 0.5, 2, np.float32)
    y1[:, 1] = 0
    cases.append((split(config_values(rng, n, -8, 8), 2, np.float32), y1))
    k = rng.integers(1, 256, n).astype(np.float32)
    xq = np.stack([(y1[:, 0].astype(np.float64) * k).astype(np.float32), np.zeros(n, np.float32)], -1)
    cases.append((xq, y1))
    # special values against each other
    sp = _special(n)
    cases.append((sp, np.roll(sp, 7, axis=0)))
    for i, (x, y) in enumerate(cases):
        with np.errstate(all="ignore"):
            assert_bits(gr.run("div_mcn", x, y), port.div_mcn(x, y), f"div_mcn case {i}")
            assert_bits(gr.run("mul_mcn", x, y), port.mul_mcn(x, y), f"mul_mcn case {i}")
            v = x[:, 0].copy()
            assert_bits(gr.run("div_n", v, y), port.div_n(v, y), f"div_n case {i}")


def test_exp_tier_over_the_range(gr, port):
    rng = np.random.default_rng(4300)
    n = 1 << 16
    f = np.float32
    x0 = rng.uniform(-104.0, 89.5, n).astype(f)  # exp from the subnormal range to overflow
    # x1: config-like residuals, values across the 2^-12 bound, zeros, subnormals
    kinds = rng.integers(0, 5, n)
    x1 = (rng.uniform(-1, 1, n) * np.spacing(np.abs(x0)) * 0.5).astype(f)
    big = (rng.uniform(-1, 1, n) * np.exp2(rng.integers(-14, -9, n).astype(np.float64))).astype(f)
    x1 = np.where(kinds == 1, big, x1)
    x1 = np.where(kinds == 2, f(0.0), x1)
    x1 = np.where(kinds == 3, f(-0.0), x1)
    x1 = np.where(kinds == 4, (rng.integers(-8, 9, n) * 1.4e-45).astype(f), x1)
    x = np.stack([x0, x1], -1)
    x[:8, 0] = [0.0, -0.0, 88.7, 88.8, -87.3, -103.9, np.inf, -np.inf]
    x[8, 0] = np.nan
    with np.errstate(all="ignore"):
        assert_bits(gr.run("exp_mcn", x), port.exp_mcn(x, oracle.EXP_CR), "exp_mcn over the range")
