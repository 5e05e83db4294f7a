"""MCF_FAST on the INT8 tensor cores (mm_ozaki.cu) against the oracle.

The tensor-core path turns the row/column-scaled operands into pa / pb-bit
integers, multiplies their residues modulo 16-22 coprime moduli exactly in
int8 x int8 -> int32 GEMMs and rebuilds every output by Chinese remaindering;
outputs too small for the rounding's error bound (cancellation) and rows /
columns holding Inf or NaN are recomputed by the fallback kernel.  Bar
(BASELINE.json north star): median and max relative error each <= 4x the
reference's own error on the same outputs.

Every test here drives the int8 path itself: A has at least 64 rows (shorter
A goes to the FP64 pipe, mm_fast.cu), at the BASELINE shapes -- config 2 in
full (4096^3, the bench's own inputs), config 4's K = 16384 for MC x MC in
binary32 nc=2 and binary16 nc=3 -- and at the awkward cases (cancellation,
extreme scales, non-finite lines, K up to 65536 where the residue reduction
takes its two-step form).
"""
import ctypes as C

import numpy as np
import pytest

from mcgen import assert_bits, split

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _within_4x(port, x, w, rows, cols, got, what, mcmc=False):
    if mcmc:
        ref = port.mm_mcmc_sampled(x, w, rows, cols)
        gerr = port.relerr_mm_mcmc(x, w, rows, cols, got)
        rerr = port.relerr_mm_mcmc(x, w, rows, cols, ref)
    else:
        ref = port.mm_mcn_sampled(x, w, rows, cols)
        gerr = port.relerr_mm_mct(x, w, rows, cols, got)
        rerr = port.relerr_mm_mct(x, w, rows, cols, ref)
    gerr, rerr = np.asarray(gerr), np.asarray(rerr)
    gm, gx = np.median(gerr), gerr.max()
    rm, rx = np.median(rerr), rerr.max()
    msg = (f"{what}: GPU median 2^{np.log2(max(gm, 1e-300)):.1f} max 2^{np.log2(max(gx, 1e-300)):.1f}; "
           f"reference median 2^{np.log2(max(rm, 1e-300)):.1f} max 2^{np.log2(max(rx, 1e-300)):.1f}")
    print(msg)
    assert gm <= 4 * rm and gx <= 4 * rx, msg
    return gerr, rerr


def _sample(seed, m, n, count):
    rng = np.random.default_rng(seed)
    return rng.integers(0, m, count), rng.integers(0, n, count)


def _phases(x, w):
    """mcf_fast_mm_phases on device copies: (product, phase ms, fallback count)."""
    import torch

    import paper_2207_08867_b200 as mcf

    m, k, _ = x.shape
    n = w.shape[1]
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    out = torch.empty((m, n, 2), dtype=torch.float32, device="cuda")
    ph = (C.c_double * 4)()
    fb = C.c_int64(0)
    rc = mcf.lib().mcf_fast_mm_phases(xd.data_ptr(), wd.data_ptr(), m, k, n, out.data_ptr(), ph, C.byref(fb), None)
    assert rc == 0, mcf.lib().mcf_last_error().decode()
    torch.cuda.synchronize()
    return out.cpu().numpy(), list(ph), fb.value


def test_config2_full_size(gr, port):
    """Config 2 exactly as the bench runs it (4096^3, data.config2): 4096 sampled
    outputs against the reference, the instrumented entry point bit-identical
    to the one-call product, and the fallback list small."""
    import paper_2207_08867_b200 as mcf
    from paper_2207_08867_b200 import data

    x, w = data.config2(4096, 4096, 4096)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows, cols = _sample(41, 4096, 4096, 4096)
    _within_4x(port, x, w, rows, cols, got[rows, cols], "config 2 (4096^3)")
    prod, ph, fb = _phases(x, w)
    assert_bits(prod, got, "phases entry point")
    print(f"config 2 phases (ms): {ph}, fallback outputs {fb}")
    assert fb < 4096 * 4096 * 1e-4


def test_config2_agrees_with_fp64_pipe_everywhere(gr):
    """All 16.7 M outputs of config 2: the int8 path (binary64 value before the
    greedy split, relative error <= 2^-52 + the bound) and the FP64-pipe path
    (~2^-100 x cond before the split) agree to the two components'
    resolution everywhere; most outputs are bit-identical (the others differ
    in the second component's last bit, where the split of the two nearly
    exact values rounds differently)."""
    import paper_2207_08867_b200 as mcf
    from paper_2207_08867_b200 import data

    x, w = data.config2(4096, 4096, 4096)
    a = gr.run("mm_mcn", x, w, plan=mcf.FAST).astype(np.float64)
    b = gr.run("mm_mcn", x, w, plan=mcf.FAST_FP64).astype(np.float64)
    va, vb = a[..., 0] + a[..., 1], b[..., 0] + b[..., 1]
    rel = np.abs(va - vb) / np.maximum(np.abs(vb), 1e-300)
    same = np.mean((a == b).all(-1))
    print(f"identical outputs {same:.6f}, max rel diff 2^{np.log2(max(rel.max(), 1e-300)):.1f}")
    assert rel.max() <= 2.0 ** -47
    assert same >= 0.85


def test_cancelling_outputs_take_the_fallback(gr, port):
    """Columns built so that some dot products cancel to ~2^-20 .. 2^-40 of
    their terms: the integer rounding alone would lose those outputs'
    relative accuracy; the fallback keeps them within the reference's error."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(32)
    m, k, n = 64, 1500, 64
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    xv = x[..., 0].astype(np.float64) + x[..., 1].astype(np.float64)
    for j in range(0, n, 2):
        i = j % m
        d = xv[i, :-1] @ w[:-1, j].astype(np.float64)
        w[-1, j] = np.float32(-d / xv[i, -1])
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows = np.array([j % m for j in range(0, n, 2)] + list(range(m)))
    cols = np.array(list(range(0, n, 2)) + [1] * m)
    _within_4x(port, x, w, rows, cols, got[rows, cols], "cancelling outputs")
    _, _, fb = _phases(x, w)
    assert fb >= 1, "the cancelling outputs must be listed for the fallback"


def test_extreme_scales_and_zero_lines(gr, port):
    """Rows and columns at 2^+-60, rows whose elements span 2^-80 of their
    maximum, an all-zero row and column: scaling is per row / column, so the
    relative accuracy must not depend on magnitude."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(33)
    m, k, n = 64, 700, 64
    v = rng.uniform(-1, 1, m * k).reshape(m, k)
    v[1] *= 2.0**60
    v[2] *= 2.0**-60
    v[3] *= np.exp2(rng.uniform(-80, 0, k))
    v[4] = 0.0
    x = split(v.ravel(), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n))
    w[:, 1] *= 2.0**-60
    w[:, 2] *= 2.0**50
    w[:, 3] = 0.0
    w[:, 4] *= np.exp2(rng.uniform(-60, 0, k))  # elements far below the column max (inexact in 48 bits)
    w = w.astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    assert np.all(got[4] == 0) and np.all(got[:, 3] == 0)
    rows, cols = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    keep = (rows != 4) & (cols != 3)
    rows, cols = rows[keep], cols[keep]
    _within_4x(port, x, w, rows, cols, got[rows, cols], "extreme scales")


@pytest.mark.parametrize("dist", ["config0", "cauchy", "lognormal2"])
def test_wide_dynamic_range_operands(gr, port, dist):
    """Operands whose elements span many binades below their row / column maxima
    (config 0's U(-1,1) 2^U(-8,8) magnitudes, Cauchy and log-normal tails): the
    binary32 B elements that do not fit the column's 48-bit fixed point are
    listed per column and their dropped parts added back in the reconstruction,
    and the fallback thresholds use the operands' magnitude sums -- so these
    products stay on the tensor-core path (few fallback outputs) and within the
    reference's error.  One column is given more inexact elements than the list
    holds (it must fall back whole and still be right)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng({"config0": 51, "cauchy": 52, "lognormal2": 53}[dist])
    m, k, n = 128, 2048, 256

    def draw(shape):
        if dist == "config0":
            return rng.uniform(-1, 1, shape) * np.exp2(rng.uniform(-8, 8, shape))
        if dist == "cauchy":
            return rng.standard_cauchy(shape)
        return rng.lognormal(0, 2, shape) * rng.choice([-1.0, 1.0], shape)

    xv, wv = draw((m, k)), draw((k, n))
    wv[:, 7] *= np.exp2(rng.uniform(-40, 0, k))  # hundreds of elements below the 48-bit window
    x = split(xv.ravel(), 2, np.float32).reshape(m, k, 2)
    w = wv.astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows, cols = np.meshgrid(np.arange(0, m, 3), np.arange(n), indexing="ij")
    rows, cols = rows.ravel(), cols.ravel()
    _within_4x(port, x, w, rows, cols, got[rows, cols], f"wide range ({dist})")
    prod, _, fb = _phases(x, w)
    assert_bits(prod, got, "phases entry point")
    # how many columns list inexact elements at all (scaled below 2^-24 of twice the column maximum)
    cmax = np.abs(w).max(0)
    listed = int(((np.abs(w) < cmax * 2.0**-22) & (w != 0)).any(0).sum())
    print(f"{dist}: fallback outputs {fb} of {m * n}; columns with elements 2^-22 below their maximum: {listed}")
    assert fb >= m, "column 7 must fall back whole"
    assert fb <= m * n * 0.05, "wide-range operands must stay on the tensor-core path"
    if dist != "lognormal2":
        assert listed > n // 4, "the case must exercise the inexact-element lists"


def test_nonfinite_rows_and_columns(gr, port):
    """Inf / NaN operands propagate to exactly their row / column; every other
    output is unaffected (same bits as without the non-finite values)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(34)
    m, k, n = 64, 300, 72
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    clean = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    x2, w2 = x.copy(), w.copy()
    x2[3, 17, 0] = np.inf
    w2[5, 6] = np.nan
    got = gr.run("mm_mcn", x2, w2, plan=mcf.FAST)
    assert not np.isfinite(got[3, :, 0]).any()
    assert not np.isfinite(got[:, 6, 0]).any()
    mask = np.ones((m, n), bool)
    mask[3, :] = False
    mask[:, 6] = False
    assert_bits(got[mask], clean[mask], "untouched outputs")


@pytest.mark.parametrize("k", [20000, 65536])
def test_long_k(gr, port, k):
    """K beyond 16384: more moduli (the bound grows with K) and the two-step
    residue reduction of the int32 sums."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(37)
    m, n = 64, 64
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows, cols = _sample(k, m, n, 256)
    _within_4x(port, x, w, rows, cols, got[rows, cols], f"K = {k}")


def test_mcmc_fp32_nc2_config4_depth(gr, port):
    """MC x MC binary32 nc=2 at config 4's depth K = 16384 (config 4's
    distribution; 256 x 256 outputs, 1024 sampled against recipe B)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(35)
    m, k, n = 256, 16384, 256
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    y = split(rng.uniform(-1, 1, k * n), 2, np.float32).reshape(k, n, 2)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows, cols = _sample(36, m, n, 1024)
    _within_4x(port, x, y, rows, cols, got[rows, cols], "MC x MC fp32 nc=2, K = 16384", mcmc=True)


def test_mcmc_fp16_nc3_config4_depth(gr, port):
    """Config 4's binary16 variant (nc=3, values U[-1,1]/64) at K = 16384."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(38)
    m, k, n = 256, 16384, 256
    x = split(rng.uniform(-1, 1, m * k) / 64, 3, np.float16).reshape(m, k, 3)
    y = split(rng.uniform(-1, 1, k * n) / 64, 3, np.float16).reshape(k, n, 3)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows, cols = _sample(39, m, n, 1024)
    _within_4x(port, x, y, rows, cols, got[rows, cols], "MC x MC fp16 nc=3, K = 16384", mcmc=True)


def test_mcmc_fp32_nc2_mixed_scales(gr, port):
    """MC x MC with rows / columns of very different scales and a cancelling
    column: the per-line scaling and the fallback on both operands."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(40)
    m, k, n = 96, 2048, 80
    v = rng.uniform(-1, 1, (m, k))
    v[5] *= 2.0**40
    v[6] *= np.exp2(rng.uniform(-70, 0, k))
    u = rng.uniform(-1, 1, (k, n))
    u[:, 7] *= 2.0**-45
    xv = v
    d = xv[9, :-1] @ u[:-1, 11]
    u[-1, 11] = -d / xv[9, -1]
    x = split(v.ravel(), 2, np.float32).reshape(m, k, 2)
    y = split(u.ravel(), 2, np.float32).reshape(k, n, 2)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows, cols = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    sel = np.random.default_rng(1).choice(m * n, 1500, replace=False)
    rows, cols = np.concatenate([rows.ravel()[sel], [9]]), np.concatenate([cols.ravel()[sel], [11]])
    _within_4x(port, x, y, rows, cols, got[rows, cols], "MC x MC mixed scales", mcmc=True)


def test_deterministic_and_chunking_invariant(gr):
    """Same bits on repeated calls, for a sub-block of rows computed alone,
    and through the host entry point's chunked pipeline."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(36)
    m, k, n = 2100, 512, 64
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    a = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    b = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    assert_bits(a, b, "repeat")
    sub = gr.run("mm_mcn", np.ascontiguousarray(x[1000:1100]), w, plan=mcf.FAST)
    assert_bits(sub, a[1000:1100], "row block alone")
    h = mcf.host.mm_mcn(x, w, strategy=mcf.FAST)
    assert_bits(h, a, "host pipeline")


@pytest.mark.parametrize("m,k,n", [(64, 33, 17), (65, 4097, 129), (300, 1, 31), (64, 4096, 4096)])
def test_ragged_shapes(gr, port, m, k, n):
    """Shapes off every alignment (K padding to 32, N padding to 16, K = 1)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(m * 7 + k + n)
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows, cols = _sample(m + n, m, n, min(m * n, 512))
    _within_4x(port, x, w, rows, cols, got[rows, cols], f"ragged {m}x{k}x{n}")


def test_short_a_uses_fp64_pipe_within_4x(gr, port):
    """m < 64 runs on the FP64 pipe (mm_fast.cu); same bar."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(31)
    m, k, n = 40, 4096, 48
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    for plan in (mcf.FAST, mcf.FAST_FP64):
        got = gr.run("mm_mcn", x, w, plan=plan)
        rows, cols = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
        _within_4x(port, x, w, rows, cols, got.reshape(-1, 2), f"short A, plan {plan}")
