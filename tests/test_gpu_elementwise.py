"""Bitwise parity of the CUDA elementwise operators with the oracle and with
golden vectors from the reference (through the C-ABI of include/mcf_gpu.h).

Parity rule: every component bit-identical, +0.0 padding
included; NaNs compare equal regardless of payload.  Exp-MCN is compared with
the oracle's correctly-rounded-exp mode (the GPU computes a correctly rounded
binary64 exp; the reference calls libm, see test_exp_vs_reference_libm).
"""
import os

import numpy as np
import pytest

import oracle
from mcgen import DT, assert_bits, config_values, nasty_mc, random_mc, split

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_elementwise.npz"))
KEYS = sorted({"_".join(k.split("_")[:2]) for k in G.files})


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _inputs(seed, n, nc, bits, nasty):
    rng = np.random.default_rng(seed)
    dt = DT[bits]
    lo, hi = (-4, 4) if bits == 16 else (-8, 8)
    x = random_mc(rng, n, nc, dt, lo, hi)
    y = random_mc(rng, n, nc, dt, lo, hi)
    if nasty:
        x = np.concatenate([x, nasty_mc(rng, n // 2, nc, dt)])
        y = np.concatenate([y, nasty_mc(rng, n // 2, nc, dt)])
    yd = y.copy()
    yd[..., 0] = (yd[..., 0].astype(np.float64) + np.sign(yd[..., 0]) * 0.5).astype(dt)
    v = (rng.uniform(-1, 1, x.shape[0]) * np.exp2(rng.uniform(lo, hi, x.shape[0]))).astype(dt)
    return x, y, yd, v


CASES = [(32, nc) for nc in (1, 2, 3, 4, 5, 8)] + [(16, 2), (16, 3), (64, 2), (64, 3)]


@pytest.mark.parametrize("bits,nc", CASES)
@pytest.mark.parametrize("nasty", [False, True])
def test_ops_bitwise_vs_oracle(gr, port, bits, nc, nasty):
    x, y, yd, v = _inputs(100 * nc + bits, 3000, nc, bits, nasty)
    assert_bits(gr.run("grow_expn", x, v), port.grow_expn(x, v), "grow_expn")
    assert_bits(gr.run("scaling_n", x, v), port.scaling_n(x, v), "scaling_n")
    if nc < 8:
        assert_bits(gr.run("scaling_n", x, v, expanded=True), port.scaling_n(x, v, True), "scaling_n expanded")
    assert_bits(gr.run("div_n", v, yd), port.div_n(v, yd), "div_n")
    assert_bits(gr.run("add_mcn", x, y), port.add_mcn(x, y), "add_mcn")
    assert_bits(gr.run("div_mcn", x, yd), port.div_mcn(x, yd), "div_mcn")
    assert_bits(gr.run("mul_mcn", x, y), port.mul_mcn(x, y), "mul_mcn")
    assert_bits(gr.run("mul_mcn_slow", x, y), port.mul_mcn_slow(x, y), "mul_mcn_slow")
    assert_bits(gr.run("square_mcn", x), port.square_mcn(x), "square_mcn")
    assert_bits(gr.run("negate", x), port.negate(x), "negate")
    assert_bits(gr.run("approx", x), port.approx(x), "approx")
    for r_nc in sorted({1, nc, max(1, nc - 1), min(8, nc + 1)}):
        assert_bits(gr.run("renormalize", x, r_nc), port.renormalize(x, r_nc), f"renormalize ->{r_nc}")
        assert_bits(gr.run("simple_renorm", x, r_nc), port.simple_renorm(x, r_nc), f"simple_renorm ->{r_nc}")
    lim = 4.0 if bits == 16 else 10.0
    xe = np.clip(x.astype(np.float64), -lim, lim).astype(x.dtype)
    assert_bits(gr.run("exp_mcn", xe), port.exp_mcn(xe, oracle.EXP_CR), "exp_mcn (CR)")


@pytest.mark.parametrize("bits", [16, 32, 64])
def test_eft_arrays(gr, port, bits):
    rng = np.random.default_rng(bits)
    lo, hi = (-6, 6) if bits == 16 else (-60, 60)
    a = (rng.uniform(-1, 1, 5001) * np.exp2(rng.uniform(lo, hi, 5001))).astype(DT[bits])
    b = (rng.uniform(-1, 1, 5001) * np.exp2(rng.uniform(lo, hi, 5001))).astype(DT[bits])
    s, e = gr.run("two_sum", a, b)
    s2, e2 = port.two_sum(a, b)
    assert_bits(s, s2, "two_sum s")
    assert_bits(e, e2, "two_sum e")
    p, q = gr.run("two_prod", a, b)
    p2, q2 = port.two_prod(a, b)
    assert_bits(p, p2, "two_prod p")
    assert_bits(q, q2, "two_prod e")


@pytest.mark.parametrize("key", KEYS)
def test_golden_reference_vectors(gr, key):
    """GPU against outputs of the reference itself (tests/golden/)."""
    x, y, yd, v, xe = (G[f"{key}_{s}"] for s in ("x", "y", "yd", "v", "xe"))
    nc = x.shape[-1]
    assert_bits(gr.run("grow_expn", x, v), G[f"{key}_grow_expn"], "grow_expn")
    assert_bits(gr.run("scaling_n", x, v), G[f"{key}_scaling_n"], "scaling_n")
    assert_bits(gr.run("scaling_n", x, v, expanded=True), G[f"{key}_scaling_n_x"], "scaling_n expanded")
    assert_bits(gr.run("div_n", v, yd), G[f"{key}_div_n"], "div_n")
    assert_bits(gr.run("add_mcn", x, y), G[f"{key}_add_mcn"], "add_mcn")
    assert_bits(gr.run("div_mcn", x, yd), G[f"{key}_div_mcn"], "div_mcn")
    assert_bits(gr.run("mul_mcn", x, y), G[f"{key}_mul_mcn"], "mul_mcn")
    assert_bits(gr.run("mul_mcn_slow", x, y), G[f"{key}_mul_mcn_slow"], "mul_mcn_slow")
    assert_bits(gr.run("square_mcn", x), G[f"{key}_square_mcn"], "square_mcn")
    assert_bits(gr.run("negate", x), G[f"{key}_negate"], "negate")
    assert_bits(gr.run("approx", x), G[f"{key}_approx"], "approx")
    assert_bits(gr.run("renormalize", x, nc), G[f"{key}_renormalize"], "renormalize")
    assert_bits(gr.run("simple_renorm", x, nc), G[f"{key}_simple_renorm"], "simple_renorm")
    assert_bits(gr.run("exp_mcn", xe), G[f"{key}_exp_mcn_cr"], "exp_mcn (CR)")
    a, b = G[f"{key}_a"], G[f"{key}_b"]
    assert_bits(np.stack(gr.run("two_sum", a, b)), G[f"{key}_two_sum"], "two_sum")
    assert_bits(np.stack(gr.run("two_prod", a, b)), G[f"{key}_two_prod"], "two_prod")


def test_exp_vs_reference_libm(gr, port):
    """GPU exp vs the unmodified reference: any difference must sit on an
    element whose libm binary64 exp differs from the correctly rounded one."""
    for key in KEYS:
        xe = G[f"{key}_xe"]
        got = gr.run("exp_mcn", xe)
        want = G[f"{key}_exp_mcn"]
        same = np.all((got == want) | (np.isnan(got) & np.isnan(want)), axis=-1)
        for i in np.nonzero(~same)[0]:
            comps = xe[i].astype(np.float64)
            assert any(port.libm_exp(c) != port.cr_exp(c)[0] for c in comps), f"{key}[{i}] unexplained"


def test_config0_full_size_bitwise(gr, port):
    """BASELINE config 0 at its full size (2^24 elements, fp32, nc=2): every
    operator bit-identical to the oracle on every element."""
    n = 1 << 24
    rng = np.random.default_rng(2024)
    x = split(config_values(rng, n), 2, np.float32)
    yv = config_values(rng, n)
    y = split(yv, 2, np.float32)
    yd = split(yv + np.sign(yv) * 0.5, 2, np.float32)
    v = config_values(rng, n).astype(np.float32)
    xe = split(np.clip(config_values(rng, n), -10, 10), 2, np.float32)
    assert_bits(gr.run("grow_expn", x, v), port.grow_expn(x, v), "grow_expn")
    assert_bits(gr.run("scaling_n", x, v), port.scaling_n(x, v), "scaling_n")
    assert_bits(gr.run("add_mcn", x, y), port.add_mcn(x, y), "add_mcn")
    assert_bits(gr.run("square_mcn", x), port.square_mcn(x), "square_mcn")
    sub = slice(0, 1 << 21)  # the issue-bound ops on a 2^21 slice keep the oracle under a minute
    assert_bits(gr.run("div_n", v[sub], yd[sub]), port.div_n(v[sub], yd[sub]), "div_n")
    assert_bits(gr.run("div_mcn", x[sub], yd[sub]), port.div_mcn(x[sub], yd[sub]), "div_mcn")
    assert_bits(gr.run("mul_mcn", x[sub], yd[sub]), port.mul_mcn(x[sub], yd[sub]), "mul_mcn")
    assert_bits(gr.run("exp_mcn", xe[sub]), port.exp_mcn(xe[sub], oracle.EXP_CR), "exp_mcn")


def test_broadcast_operands(gr, port):
    rng = np.random.default_rng(7)
    x = random_mc(rng, 6 * 5, 2, np.float32).reshape(6, 5, 2)
    vs = np.float32(rng.uniform(-3, 3))
    v5 = rng.uniform(-3, 3, 5).astype(np.float32)
    for v in (np.array([vs]), v5):
        want_g = port.grow_expn(x, np.tile(v, 6) if v.size == 5 else v)
        assert_bits(gr.run("grow_expn", x, v), want_g.reshape(x.shape), "grow broadcast")
        want_s = port.scaling_n(x, np.tile(v, 6) if v.size == 5 else v)
        assert_bits(gr.run("scaling_n", x, v), want_s.reshape(x.shape), "scaling broadcast")
        want_d = port.div_n(np.tile(v, 6) if v.size == 5 else v, x)
        assert_bits(gr.run("div_n", v, x), want_d.reshape(x.shape), "div_n broadcast")


def test_reference_known_answers(gr):
    """KATs of T/test_mct.cpp restated on the GPU."""
    f = np.float32
    assert_bits(gr.run("renormalize", np.array([[2.0**-40, 1.0]], f), 2), np.array([[1.0, 2.0**-40]], f))
    assert_bits(gr.run("renormalize", np.zeros((1, 3), f), 2), np.zeros((1, 2), f))
    assert_bits(gr.run("simple_renorm", np.array([[1.0, 0.0, 2.0**-30]], f), 3), np.array([[1.0, 2.0**-30, 0.0]], f))
    assert_bits(gr.run("grow_expn", np.array([[1.0, 0.0]], f), np.array([2.0**-30], f)), np.array([[1.0, 2.0**-30]], f))
    assert_bits(gr.run("square_mcn", np.array([[1.0, 0.0]], f)), np.array([[1.0, 0.0]], f))
    assert_bits(gr.run("square_mcn", np.zeros((1, 2), f)), np.zeros((1, 2), f))
    assert_bits(gr.run("exp_mcn", np.zeros((1, 2), f)), np.array([[1.0, 0.0]], f))
    assert_bits(gr.run("div_n", np.array([0.4375], f), np.array([[1.0, 0.0]], f)), np.array([[0.4375, 0.0]], f))
    q = gr.run("div_mcn", np.array([[1.0, 0.0]], f), np.zeros((1, 2), f))
    assert not np.isfinite(q[0, 0])
    h = np.float16
    assert np.isinf(gr.run("exp_mcn", np.array([[12.0, 0.0]], h))[0, 0])
    s, e = gr.run("two_sum", np.array([1.0], f), np.array([2.0**-30], f))
    assert s[0] == 1.0 and e[0] == 2.0**-30
    p, e = gr.run("two_prod", np.array([1 + 2.0**-23], f), np.array([1 + 2.0**-23], f))
    assert p[0] == 1 + 2.0**-22 and e[0] == 2.0**-46


def test_errors_mirror_reference(gr):
    import torch

    import paper_2207_08867_b200 as mcf

    t = torch.zeros((2, 9), device="cuda")
    with pytest.raises(ValueError, match="1 <= nc <= 8"):
        mcf.square_mcn(t)
    x = torch.zeros((2, 2, 2), device="cuda")
    with pytest.raises(ValueError, match="trailing suffix"):
        mcf.scaling_n(x, torch.zeros(3, device="cuda"))
    with pytest.raises(mcf.UnsupportedOperation):
        mcf.mm_mcn(x, x)


def test_host_entry_points_match_device(port):
    """mcf.host (the reference's host calling model) equals the oracle."""
    import paper_2207_08867_b200 as mcf

    x, y, yd, v = _inputs(5, 200000, 2, 32, True)
    assert_bits(mcf.host.add_mcn(x, y), port.add_mcn(x, y), "host add")
    assert_bits(mcf.host.grow_expn(x, v), port.grow_expn(x, v), "host grow")
    assert_bits(mcf.host.div_n(v, yd), port.div_n(v, yd), "host div_n")
    assert_bits(mcf.host.scaling_n(x, v[:1]), port.scaling_n(x, v[:1]), "host scaling scalar")
    assert_bits(mcf.host.approx(x), port.approx(x), "host approx")


@pytest.mark.parametrize("nc", [2, 3])
def test_binary64_fast_paths_full_tiles(gr, port, nc):
    """Binary64 register fast paths on enough elements for
    the TMA tile kernel, plus a ragged tail, every operator bitwise."""
    x, y, yd, v = _inputs(900 + nc, 300_001, nc, 64, False)
    for name, args, ref in (("grow_expn", (x, v), port.grow_expn(x, v)),
                            ("scaling_n", (x, v), port.scaling_n(x, v)),
                            ("div_n", (v, yd), port.div_n(v, yd)),
                            ("add_mcn", (x, y), port.add_mcn(x, y)),
                            ("div_mcn", (x, yd), port.div_mcn(x, yd)),
                            ("mul_mcn", (x, y), port.mul_mcn(x, y)),
                            ("square_mcn", (x,), port.square_mcn(x)),
                            ("exp_mcn", (np.clip(x, -10, 10),), port.exp_mcn(np.clip(x, -10, 10), oracle.EXP_CR))):
        assert_bits(gr.run(name, *args), ref, f"b64 nc{nc} {name}")
