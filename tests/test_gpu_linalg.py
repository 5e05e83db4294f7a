"""MC contractions on the GPU (linalg.hpp) against the oracle.

Reference-order plans (SEQUENTIAL, PAIRWISE_TREE) run the reference's DotCore
per output and must be bit-identical to it; MC x MC follows SURVEY 8c recipe
B bit for bit.  The throughput plan (FAST) uses a different summation and is
checked against binary128 truth with the tolerance of BASELINE.json's
north star: median and max relative error each <= 4x the reference's own on
the same sampled outputs.
"""
import os

import numpy as np
import pytest

import oracle
from mcgen import DT, assert_bits, random_mc

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_elementwise.npz"))


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def wp(rng, shape, bits, lo=-3, hi=3):
    n = int(np.prod(shape))
    return (rng.uniform(-1, 1, n) * np.exp2(rng.uniform(lo, hi, n))).astype(DT[bits]).reshape(shape)


@pytest.mark.parametrize("bits,nc", [(32, 1), (32, 2), (32, 3), (32, 4), (16, 2), (64, 2), (16, 1), (64, 1)])
def test_mm_reference_order_bitwise(gr, port, bits, nc):
    rng = np.random.default_rng(bits * 10 + nc)
    x = random_mc(rng, 33 * 70, nc, DT[bits], -3, 3).reshape(33, 70, nc)
    w = wp(rng, (70, 45), bits)
    assert_bits(gr.run("mm_mcn", x, w), port.mm_mcn(x, w), "mm_mcn")
    xb = random_mc(rng, 3 * 5 * 9, nc, DT[bits], -3, 3).reshape(3, 5, 9, nc)
    wb = wp(rng, (3, 9, 4), bits)
    assert_bits(gr.run("bmm_mcn", xb, wb), port.bmm_mcn(xb, wb), "bmm_mcn")
    w2 = wp(rng, (9, 4), bits)
    assert_bits(gr.run("matmul_mcn", xb, w2), port.bmm_mcn(xb, w2), "matmul 3/2")
    v = wp(rng, (70,), bits)
    assert_bits(gr.run("mv_mcn", x, v), port.mv_mcn(x, v), "mv_mcn")
    assert_bits(gr.run("dot_mcn", x[0], v), port.dot_mcn(x[0], v), "dot_mcn")


@pytest.mark.parametrize("nc", [1, 2, 3])
def test_pairwise_tree_bitwise(gr, port, nc):
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(nc)
    x = random_mc(rng, 8 * 100, nc, np.float32, -3, 3).reshape(8, 100, nc)
    w = wp(rng, (100, 6), 32)
    for leaf in (1, 4):
        got = gr.run("mm_mcn", x, w, plan=(mcf.PAIRWISE_TREE, leaf))
        assert_bits(got, port.bmm_mcn(x, w, oracle.PAIRWISE_TREE, leaf), f"tree leaf={leaf}")


@pytest.mark.parametrize("k,leaf", [(1, 1), (7, 1), (31, 2), (33, 1), (100, 40), (3000, 1), (4097, 5), (20000, 64)])
def test_pairwise_tree_warp_split_bitwise(gr, port, k, leaf):
    """The warp-parallel tree (5 levels across lanes, leaves and deeper levels
    per lane) on K that leave some top-level nodes as leaves, odd splits and
    long K: the same tree as linalg.hpp:59-76, bit for bit."""
    import paper_2207_08867_b200 as mcf

    for nc in (2, 3):
        rng = np.random.default_rng(k + leaf + nc)
        x = random_mc(rng, 3 * k, nc, np.float32, -3, 3).reshape(3, k, nc)
        w = wp(rng, (k, 2), 32)
        got = gr.run("mm_mcn", x, w, plan=(mcf.PAIRWISE_TREE, leaf))
        assert_bits(got, port.bmm_mcn(x, w, oracle.PAIRWISE_TREE, leaf), f"tree k={k} leaf={leaf} nc={nc}")


def test_single_component_equals_plain_matmul(gr, port):
    """T/test_linalg.cpp:297-314: nc=1 mm == matmul2d bitwise."""
    rng = np.random.default_rng(48)
    for bits in (16, 32, 64):
        a = wp(rng, (4, 6), bits, -1, 1)
        b = wp(rng, (6, 3), bits, -1, 1)
        got = gr.run("mm_mcn", a[..., None], b)[..., 0]
        assert_bits(got, port.matmul2d(a, b), f"nc=1 mm b{bits}")


def test_golden_contractions(gr):
    for key in ("b32_nc2", "b32_nc3", "b16_nc3", "b64_nc2", "b32_nc1"):
        xm, wm, ym = G[f"{key}_mm_x"], G[f"{key}_mm_w"], G[f"{key}_mm_y"]
        assert_bits(gr.run("mm_mcn", xm, wm), G[f"{key}_mm"], f"{key} mm")
        import paper_2207_08867_b200 as mcf

        assert_bits(gr.run("mm_mcn", xm, wm, plan=(mcf.PAIRWISE_TREE, 2)), G[f"{key}_mm_tree"], f"{key} tree")
        assert_bits(gr.run("mm_mcmc", xm, ym), G[f"{key}_mmmc"], f"{key} mm_mcmc")


@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 3), (16, 2), (64, 2), (32, 4)])
def test_mcmc_recipe_b_bitwise(gr, port, bits, nc):
    rng = np.random.default_rng(7 * nc + bits)
    lo, hi = (-3, 3) if bits != 16 else (-6, 0)
    x = random_mc(rng, 20 * 50, nc, DT[bits], lo, hi).reshape(20, 50, nc)
    y = random_mc(rng, 50 * 12, nc, DT[bits], lo, hi).reshape(50, 12, nc)
    rows = np.repeat(np.arange(20), 12)
    cols = np.tile(np.arange(12), 20)
    assert_bits(gr.run("mm_mcmc", x, y), port.mm_mcmc_sampled(x, y, rows, cols).reshape(20, 12, nc), "mm_mcmc")
    xd = random_mc(rng, 9 * 300, nc, DT[bits], lo, hi).reshape(9, 300, nc)
    yd = random_mc(rng, 9 * 300, nc, DT[bits], lo, hi).reshape(9, 300, nc)
    assert_bits(gr.run("dot_mcmc", xd, yd), port.dot_mcmc(xd, yd), "dot_mcmc")


def test_reference_kats(gr):
    """T/test_linalg.cpp:57-66, 87-98, 114-123."""
    f = np.float32
    x = np.zeros((17, 2), f)
    x[:, 0] = 1
    d = gr.run("dot_mcn", x, np.ones(17, f))
    assert d[0] == 17.0 and d[1] == 0.0
    assert np.all(gr.run("dot_mcn", x, np.zeros(17, f)) == 0)
    eye = np.zeros((3, 3, 2), f)
    for i in range(3):
        eye[i, i, 0] = 1
    v = np.array([2.0, -1.5, 0.25], f)
    assert np.array_equal(gr.run("mv_mcn", eye, v)[:, 0], v)
    import paper_2207_08867_b200 as mcf

    with pytest.raises(ValueError, match=r"\(3,5\).*\(3,2\)"):
        import torch

        mcf.matmul_mcn(torch.zeros((3, 5, 2), device="cuda"), torch.zeros((3, 2), device="cuda"))


# ---- MCF_FAST: tolerance against binary128 truth -----------------------------------

def _relerr_stats(e):
    e = np.asarray(e, np.float64)
    return float(np.median(e)), float(np.max(e))


def _check_within_4x(gpu_err, ref_err, what):
    gm, gx = _relerr_stats(gpu_err)
    rm, rx = _relerr_stats(ref_err)
    msg = (f"{what}: GPU median 2^{np.log2(max(gm, 1e-300)):.1f} max 2^{np.log2(max(gx, 1e-300)):.1f}; "
           f"reference median 2^{np.log2(max(rm, 1e-300)):.1f} max 2^{np.log2(max(rx, 1e-300)):.1f}")
    print(msg)
    assert gm <= 4 * rm and gx <= 4 * rx, msg


def test_fast_mm_mct_nc2_within_reference_error(gr, port):
    """BASELINE config 2 distribution (A nc=2 split from fp64 U[-1,1], B fp32
    U[-1,1]) at the full K = 4096, on a 32 x 32 block of outputs."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(2)
    m, k, n = 32, 4096, 48
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows = np.repeat(np.arange(m), n)
    cols = np.tile(np.arange(n), m)
    ref = port.mm_mcn_sampled(x, w, rows, cols)
    gerr = port.relerr_mm_mct(x, w, rows, cols, got.reshape(-1, 2))
    rerr = port.relerr_mm_mct(x, w, rows, cols, ref)
    _check_within_4x(gerr, rerr, "mm MC(nc=2) x T, K=4096")


def test_fast_mv_nc3_within_reference_error(gr, port):
    """BASELINE config 1a distribution (nc=3, U(-1,1) 2^U(-8,8)), K = 4096."""
    import paper_2207_08867_b200 as mcf
    from mcgen import config_values

    rng = np.random.default_rng(3)
    m, k = 96, 4096
    x = random_mc(rng, m * k, 3, np.float32).reshape(m, k, 3)
    v = config_values(rng, k).astype(np.float32)
    got = gr.run("mv_mcn", x, v, plan=mcf.FAST)
    rows = np.arange(m)
    cols = np.zeros(m, np.int64)
    w = v.reshape(k, 1)
    ref = port.mm_mcn_sampled(x, w, rows, cols)
    gerr = port.relerr_mm_mct(x, w, rows, cols, got)
    rerr = port.relerr_mm_mct(x, w, rows, cols, ref)
    _check_within_4x(gerr, rerr, "mv MC(nc=3) x T, K=4096")


@pytest.mark.parametrize("nc", [2, 3])
def test_fast_dot_mcmc_within_recipe_b_error(gr, port, nc):
    """BASELINE config 1b: independent MC x MC dots of length 4096."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(4 + nc)
    b, k = 48, 4096
    x = random_mc(rng, b * k, nc, np.float32).reshape(b, k, nc)
    y = random_mc(rng, b * k, nc, np.float32).reshape(b, k, nc)
    got = gr.run("dot_mcmc", x, y, plan=mcf.FAST)
    ref = port.dot_mcmc(x, y)
    # truth: each dot as a 1 x k times k x 1 MC x MC product
    gerr, rerr = [], []
    for i in range(b):
        r0, c0 = np.array([0]), np.array([0])
        gerr.append(port.relerr_mm_mcmc(x[i:i + 1], y[i].reshape(k, 1, nc), r0, c0, got[i:i + 1])[0])
        rerr.append(port.relerr_mm_mcmc(x[i:i + 1], y[i].reshape(k, 1, nc), r0, c0, ref[i:i + 1])[0])
    _check_within_4x(gerr, rerr, f"dot MC x MC nc={nc}")


def test_fast_mm_mcmc_fp32_nc2_within_recipe_b_error(gr, port):
    """BASELINE config 4 (fp32 nc=2 split from fp64 U[-1,1]) on a K=4096 slab."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(6)
    m, k, n = 16, 4096, 24
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    y = split(rng.uniform(-1, 1, k * n), 2, np.float32).reshape(k, n, 2)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows = np.repeat(np.arange(m), n)
    cols = np.tile(np.arange(n), m)
    ref = port.mm_mcmc_sampled(x, y, rows, cols)
    gerr = port.relerr_mm_mcmc(x, y, rows, cols, got.reshape(-1, 2))
    rerr = port.relerr_mm_mcmc(x, y, rows, cols, ref)
    _check_within_4x(gerr, rerr, "mm MC x MC fp32 nc=2, K=4096")


def test_fast_mm_mcmc_fp16_nc3_within_recipe_b_error(gr, port):
    """BASELINE config 4 fp16 variant: nc=3 binary16 split from U[-1,1]/64."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(7)
    m, k, n = 16, 4096, 24
    x = split(rng.uniform(-1, 1, m * k) / 64, 3, np.float16).reshape(m, k, 3)
    y = split(rng.uniform(-1, 1, k * n) / 64, 3, np.float16).reshape(k, n, 3)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows = np.repeat(np.arange(m), n)
    cols = np.tile(np.arange(n), m)
    ref = port.mm_mcmc_sampled(x, y, rows, cols)
    gerr = port.relerr_mm_mcmc(x, y, rows, cols, got.reshape(-1, 3))
    rerr = port.relerr_mm_mcmc(x, y, rows, cols, ref)
    _check_within_4x(gerr, rerr, "mm MC x MC fp16 nc=3, K=4096")


def test_fast_plan_ragged_shapes_and_fallback(gr, port):
    """Odd shapes exercise the tile edges; shapes without a fast kernel fall
    back to the reference order (bitwise)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(8)
    x = random_mc(rng, 77 * 130, 2, np.float32, -2, 2).reshape(77, 130, 2)
    w = wp(rng, (130, 70), 32, -2, 2)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    ref = port.mm_mcn(x, w)
    rows = np.repeat(np.arange(77), 70)
    cols = np.tile(np.arange(70), 77)
    gerr = port.relerr_mm_mct(x, w, rows, cols, got.reshape(-1, 2))
    rerr = port.relerr_mm_mct(x, w, rows, cols, ref.reshape(-1, 2))
    _check_within_4x(gerr, rerr, "ragged mm")
    # odd n: the int8 path pads the columns; same bar
    w3 = wp(rng, (130, 3), 32)
    got3 = gr.run("mm_mcn", x, w3, plan=mcf.FAST)
    r3, c3 = np.repeat(np.arange(77), 3), np.tile(np.arange(3), 77)
    _check_within_4x(port.relerr_mm_mct(x, w3, r3, c3, got3.reshape(-1, 2)),
                     port.relerr_mm_mct(x, w3, r3, c3, port.mm_mcn(x, w3).reshape(-1, 2)), "ragged mm, n = 3")
    # no fast instantiation (binary64 components, nc = 4) -> reference order, bit-identical
    x64 = random_mc(rng, 9 * 20, 4, np.float64, -2, 2).reshape(9, 20, 4)
    w64 = wp(rng, (20, 5), 64)
    assert_bits(gr.run("mm_mcn", x64, w64, plan=mcf.FAST), port.mm_mcn(x64, w64), "fallback")


def test_host_pipelined_fast_mm_equals_device_path(gr, port):
    """mcf_h_bmm_mcn's row-chunked pipeline (copies overlapping the mm, two
    compute streams, per-chunk exactness flags) returns the device entry
    point's bits; a chunk whose operands need the err-carrying kernel still
    meets the tolerance."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(21)
    m, k, n = 2000, 300, 96  # 4 chunks of 512 rows, the last one ragged
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    dev = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    hst = mcf.host.mm_mcn(x, w, strategy=mcf.FAST)
    assert_bits(hst, dev, "host pipeline vs device")
    # components spanning > 53 bits in one chunk only: (sum, err) pairs there
    x2 = x.copy()
    x2[1500, :, 1] = (x2[1500, :, 0] * np.float32(2.0 ** -40)).astype(np.float32)
    hst2 = mcf.host.mm_mcn(x2, w, strategy=mcf.FAST)
    rows = np.repeat(np.array([0, 1499, 1500, 1999]), n)
    cols = np.tile(np.arange(n), 4)
    got = hst2[rows, cols]
    ref = port.mm_mcn_sampled(x2, w, rows, cols)
    gerr = port.relerr_mm_mct(x2, w, rows, cols, got.reshape(-1, 2))
    rerr = port.relerr_mm_mct(x2, w, rows, cols, ref)
    _check_within_4x(gerr, rerr, "host pipeline, inexact chunk")


@pytest.mark.parametrize("nc", [1, 2, 3])
def test_fast_mm_mcmc_fp16_int8_path_within_recipe_b_error(gr, port, nc):
    """Binary16 MC x MC on the int8 tensor cores (five digits per pre-summed
    element, shapes >= 64): within 4x of recipe B's error, both operands with
    rows / columns of very different scales."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(70 + nc)
    m, k, n = 96, 2048, 80
    xs = rng.uniform(-1, 1, (m, k)) / 64 * np.exp2(rng.integers(-3, 4, (m, 1)))
    ys = rng.uniform(-1, 1, (k, n)) / 64 * np.exp2(rng.integers(-3, 4, (1, n)))
    x = split(xs.reshape(-1), nc, np.float16).reshape(m, k, nc)
    y = split(ys.reshape(-1), nc, np.float16).reshape(k, n, nc)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows = np.repeat(np.arange(m), n)
    cols = np.tile(np.arange(n), m)
    ref = port.mm_mcmc_sampled(x, y, rows, cols)
    gerr = port.relerr_mm_mcmc(x, y, rows, cols, got.reshape(-1, nc))
    rerr = port.relerr_mm_mcmc(x, y, rows, cols, ref)
    _check_within_4x(gerr, rerr, f"mm MC x MC fp16 nc={nc}, int8 path")


def test_fast_mm_mcmc_fp16_int8_path_nonfinite_rows_and_columns(gr):
    """A row of A or a column of B holding Inf / NaN makes exactly that row /
    column of the binary16 int8-path product non-finite; the rest is finite."""
    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(99)
    m, k, n = 80, 256, 72
    x = split(rng.uniform(-1, 1, m * k) / 64, 3, np.float16).reshape(m, k, 3)
    y = split(rng.uniform(-1, 1, k * n) / 64, 3, np.float16).reshape(k, n, 3)
    x[7, 3, 0] = np.inf
    y[5, 11, 0] = np.nan
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST).astype(np.float64).sum(axis=-1)
    bad = np.zeros((m, n), bool)
    bad[7, :] = True
    bad[:, 11] = True
    assert np.all(~np.isfinite(got[bad]))
    assert np.all(np.isfinite(got[~bad]))


@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 2), (64, 2), (32, 1)])
def test_mm4d_addmm_matmul_transpose_bitwise(gr, port, bits, nc):
    """The rest of linalg.hpp's surface: mm4d_mcn (two batch axes, :218-231),
    addmm_mcn (alpha / beta through ScalingN, bias broadcast over rows,
    :233-253) against the reference's own composition of the oracle's
    operators, the matmul_mcn dispatcher bitwise equal to the specialised
    operator of every rank pair (T/test_linalg.cpp:220-257), and
    mc_transpose2d (:301-315)."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(bits + nc)
    x4 = random_mc(rng, 2 * 3 * 5 * 6, nc, DT[bits], -3, 3).reshape(2, 3, 5, 6, nc)
    w4 = wp(rng, (2, 3, 6, 4), bits)
    want4 = port.bmm_mcn(x4.reshape(6, 5, 6, nc), w4.reshape(6, 6, 4)).reshape(2, 3, 5, 4, nc)
    assert_bits(gr.run("mm4d_mcn", x4, w4), want4, "mm4d_mcn")
    assert_bits(gr.run("matmul_mcn", x4, w4), want4, "matmul 4/4 == mm4d")
    w2 = wp(rng, (6, 4), bits)
    assert_bits(gr.run("matmul_mcn", x4, w2), port.bmm_mcn(x4.reshape(6, 5, 6, nc), w2).reshape(2, 3, 5, 4, nc),
                "matmul 4/2")
    a = random_mc(rng, 19 * 6, nc, DT[bits], -3, 3).reshape(19, 6, nc)
    x1 = random_mc(rng, 6, nc, DT[bits], -3, 3).reshape(6, nc)
    w1 = wp(rng, (6,), bits)
    assert_bits(gr.run("matmul_mcn", a, w2), gr.run("mm_mcn", a, w2), "matmul 2/2 == mm")
    assert_bits(gr.run("matmul_mcn", a, w1), port.mv_mcn(a, w1), "matmul 2/1 == mv")
    assert_bits(gr.run("matmul_mcn", x1, w1), port.dot_mcn(x1, w1), "matmul 1/1 == dot")
    assert_bits(gr.run("matmul_mcn", x1, w2), port.mm_mcn(x1[None], w2)[0], "matmul 1/2 == row mm")
    # addmm: full bias, and a row bias broadcast with alpha / beta
    bias = random_mc(rng, 19 * 4, nc, DT[bits], -2, 2).reshape(19, 4, nc)
    row = random_mc(rng, 4, nc, DT[bits], -2, 2).reshape(4, nc)
    prod = port.mm_mcn(a, w2)
    assert_bits(gr.run("addmm_mcn", bias, a, w2), port.add_mcn(bias, prod), "addmm_mcn")
    alpha, beta = np.array([0.75], DT[bits]), np.array([-1.5], DT[bits])
    want = port.add_mcn(np.broadcast_to(port.scaling_n(row, beta), (19, 4, nc)).copy(), port.scaling_n(prod, alpha))
    assert_bits(gr.run("addmm_mcn", row, a, w2, alpha=0.75, beta=-1.5), want, "addmm_mcn alpha beta broadcast")
    with pytest.raises(ValueError, match=r"\(3,5,6\)"):
        mcf.matmul_mcn(torch.zeros((3, 5, 6, nc), dtype=torch.float32, device="cuda"),
                       torch.zeros((5, 2), device="cuda"))
    # transpose: component-preserving bit copy
    t = random_mc(rng, 37 * 45, nc, DT[bits], -3, 3).reshape(37, 45, nc)
    assert_bits(gr.run("mc_transpose2d", t), np.ascontiguousarray(t.transpose(1, 0, 2)), "mc_transpose2d")
