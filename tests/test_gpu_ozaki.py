"""MCF_FAST on the INT8 tensor cores (mm_ozaki.cu) against the oracle.

The tensor-core path splits the row/column-scaled operands into nine balanced
base-256 digits, multiplies digit planes exactly in int32 and recombines in
double-double; outputs too small for the split's error bound (cancellation)
and rows / columns holding Inf or NaN are recomputed by the fallback kernel.
Bar (BASELINE.json north star): median and max relative error each <= 4x the
reference's own error on the same outputs; plus the cases the splitting is
most sensitive to.
"""
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


@pytest.mark.parametrize("plan_name", ["FAST", "FAST_FP64"])
def test_config2_distribution_both_fast_paths(gr, port, plan_name):
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(31)
    m, k, n = 40, 4096, 48
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    got = gr.run("mm_mcn", x, w, plan=getattr(mcf, plan_name))
    rows, cols = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    _within_4x(port, x, w, rows, cols, got.reshape(-1, 2), f"mm config-2 data, {plan_name}")


def test_cancelling_outputs_take_the_fallback(gr, port):
    """Columns built so that some dot products cancel to ~2^-20 .. 2^-40 of
    their terms: the digit splitting alone would lose those outputs' relative
    accuracy; the fallback keeps them within the reference's error."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(32)
    m, k, n = 24, 1500, 40
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, k * n).astype(np.float32).reshape(k, n)
    xv = x[..., 0].astype(np.float64) + x[..., 1].astype(np.float64)
    for j in range(0, n, 2):
        i = j % m
        # choose w[-1, j] so that row i . column j nearly vanishes
        d = xv[i, :-1] @ w[:-1, j].astype(np.float64)
        w[-1, j] = np.float32(-d / xv[i, -1])
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows = np.array([j % m for j in range(0, n, 2)] + list(range(m)))
    cols = np.array(list(range(0, n, 2)) + [1] * m)
    _within_4x(port, x, w, rows, cols, got[rows, cols], "cancelling outputs")


def test_extreme_scales_and_zero_lines(gr, port):
    """Rows and columns at 2^+-60, rows whose elements span 2^-80 of their
    maximum, an all-zero row and column: scaling is per row / column, so the
    relative accuracy must not depend on magnitude."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(33)
    m, k, n = 12, 700, 10
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
    w[:, 4] *= np.exp2(rng.uniform(-60, 0, k))
    w = w.astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    assert np.all(got[4] == 0) and np.all(got[:, 3] == 0)
    rows, cols = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    keep = (rows != 4) & (cols != 3)
    rows, cols = rows[keep], cols[keep]
    _within_4x(port, x, w, rows, cols, got[rows, cols], "extreme scales")


def test_nonfinite_rows_and_columns(gr, port):
    """Inf / NaN operands propagate to exactly their row / column; every other
    output is unaffected (same bits as without the non-finite values)."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(34)
    m, k, n = 9, 300, 11
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


def test_mcmc_fp32_nc2_tensor_core(gr, port):
    """MC x MC (config 4 distribution) through the digit splitting of both
    operands."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(35)
    m, k, n = 20, 4096, 28
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    y = split(rng.uniform(-1, 1, k * n), 2, np.float32).reshape(k, n, 2)
    got = gr.run("mm_mcmc", x, y, plan=mcf.FAST)
    rows, cols = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    _within_4x(port, x, y, rows, cols, got.reshape(-1, 2), "MC x MC tensor core", mcmc=True)


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


def test_long_k_is_cut_into_int32_safe_chunks(gr, port):
    """K beyond one int8 GEMM's int32 headroom (9 digits x kc x 2^14 < 2^31,
    kc <= 14400): the digit planes are cut into K chunks whose partial
    products are summed in int64 before the recombination."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(37)
    m, k, n = 6, 20000, 20
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    rows, cols = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    _within_4x(port, x, w, rows, cols, got.reshape(-1, 2), "K = 20000 (two chunks)")
