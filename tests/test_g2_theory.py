"""CPU check of the certified binary32 nc=2 tiers (csrc/mcf_g2.cuh, and the wide
long-division tier csrc/mcf_w2.cuh: rows w2div / w2mul for the three-digit
core, w1div / w1mul for the one-digit core the kernels use, w2mslow / w2msq for
the direct product and its square, emulated with a wide format of 2 p + 5 bits).

tools/g2_verify.cpp runs the SAME header on an emulated binary format with p
significand bits and compares it with the reference's algorithms restated in
that format (renorm_kernel with its pass cap, scale_raw, add_kernel,
div_kernel, mul_fast_kernel, square_kernel, grow_kernel; mc_ops.hpp:41-282):

* exhaustively over every compressed operand pair in an exponent window for
  small p, where every rounding boundary, tie and power of two is hit;
* on sampled config-0 operands at p = 24.

Required: no accepted case differs from the reference bit for bit, and the
reference never ends a renormalization at its pass cap (the certification
argument assumes it ends compressed).  At p = 24 the shortcut must accept
essentially every config-0 element (it is the fast path).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g2v(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("g2") / "g2v")
    src = os.path.join(ROOT, "tools", "g2_verify.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fopenmp", src, "-o", exe], check=True)
    return exe


ROWS = {"scale", "square", "div", "mul", "add", "grow", "w2div", "w2mul", "w2scale", "w1div", "w1mul", "w2mslow", "w2msq"}
# the one-digit core's margin (2^10 units of the remainder quotient's last
# place) is wider than the whole rounding interval of the emulated format
# below p = 6: it accepts nothing there and is checked at p = 6 instead
ONE_DIGIT = {"w1div", "w1mul"}


def _run(exe, *args, env=None):
    r = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, **(env or {})))
    rows = {}
    for line in r.stdout.splitlines():
        m = re.match(r"p=\s*(\d+) (\w+)\s+cases\s+(\d+)\s+accepted\s+([\d.]+)%\s+mismatches (\d+)\s+cap-hits (\d+)", line)
        if m:
            rows[m.group(2)] = dict(cases=int(m.group(3)), acc=float(m.group(4)), bad=int(m.group(5)),
                                    cap=int(m.group(6)))
    assert set(rows) == ROWS, r.stdout + r.stderr
    return rows, r.returncode


@pytest.mark.parametrize("p,k", [(4, 5), (5, 3)])
def test_exhaustive_small_precision(g2v, p, k):
    rows, rc = _run(g2v, "small", p, k)
    for op, r in rows.items():
        assert r["bad"] == 0, (op, r)
        assert r["cap"] == 0, (op, r)
        assert r["cases"] > 0 and (r["acc"] > 0 or op in ONE_DIGIT), (op, r)
    assert rc == 0


def test_one_digit_core_exhaustive_p6(g2v):
    """Every compressed pair at p = 6 (second components up to one binade below
    the first's last place) through the one-digit division core, with the
    margin set FOUR TIMES BELOW the certified one (2^8 units; at 2^10 the
    margin covers the whole rounding interval of this small format): every
    accepted case -- a superset of what the certified margin would accept --
    is bit-identical to the reference's three-digit div_kernel / Mul-MCN.
    (The same run over second components six binades down, 826.7 M divisions
    and 275.3 M multiplications, has zero mismatches: DESIGN 4.3c.)"""
    rows, rc = _run(g2v, "small", 6, 0, env={"G2_ONLY1": "1", "G2_LG1": "8"})
    for op in ONE_DIGIT:
        r = rows[op]
        assert r["bad"] == 0 and r["cap"] == 0, (op, r)
        assert r["cases"] > 5_000_000 and r["acc"] > 10.0, (op, r)
    assert rc == 0


@pytest.mark.parametrize("p", [8, 10, 12])
def test_one_digit_core_sampled_mid_precisions(g2v, p):
    """The certified margin itself at precisions where it leaves room: sampled
    config-0 operands, accepted cases bit-identical."""
    rows, rc = _run(g2v, "sample", p, 1000000, env={"G2_ONLY1": "1"})
    for op in ONE_DIGIT:
        r = rows[op]
        assert r["bad"] == 0 and r["cap"] == 0, (op, r)
        assert r["acc"] > 15.0, (op, r)
    assert rc == 0


def test_one_digit_margin_is_needed(g2v):
    """The verifier can see a margin that is too small: at 2^4 units (64x below
    the certified one) accepted divisions differ from the reference."""
    rows, rc = _run(g2v, "small", 6, 0, env={"G2_ONLY1": "1", "G2_LG1": "4"})
    assert rows["w1div"]["bad"] > 0 and rc != 0


def test_sampled_binary32(g2v):
    rows, rc = _run(g2v, "sample", 24, 300000)
    for op, r in rows.items():
        assert r["bad"] == 0 and r["cap"] == 0, (op, r)
        # add: half the samples are near-cancelling sums; ties with two nonzero
        # tail terms decline (~0.3% of random sums)
        # w2mul: two chained wide divisions, each declining ~1e-5 of the samples
        assert r["acc"] > (99.5 if op == "add" else 99.9 if op in ONE_DIGIT else 99.98 if op == "w2mul" else 99.99), (op, r)
    assert rc == 0
