"""The short-A FP64-pipe kernel (csrc/mm_skinny.cu: MC(nc=2, binary32) x Tensor
for m <= 16 rows, e.g. the MC-MLP's class layer) against the binary128 truth,
beside the reference's own outputs: median and max relative error within 4x of
the reference's (linalg.hpp:138-157 on the same samples).  Shapes cover one and
sixteen rows, odd row counts (the two row groups uneven), K below, at and
across the 512-row chunk and the 32-row ring stage, ragged column tiles, rows
and columns scaled 2^+-30 apart, the config-3 class layer itself, and
non-finite rows / columns."""
import numpy as np
import pytest

from mcgen import split

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


def _errs(port, x, w, got, samples, rng):
    m, n = x.shape[0], w.shape[1]
    if m * n <= samples:
        rows, cols = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    else:
        rows, cols = rng.integers(0, m, samples), rng.integers(0, n, samples)
    ref = port.mm_mcn_sampled(x, w, rows, cols)
    return port.relerr_mm_mct(x, w, rows, cols, got[rows, cols]), port.relerr_mm_mct(x, w, rows, cols, ref)


@pytest.mark.parametrize("m,k,n", [(1, 7, 4), (2, 33, 64), (5, 100, 68), (9, 512, 132), (10, 1024, 1024),
                                   (13, 545, 60), (16, 3000, 200), (10, 1500, 8)])
def test_short_a_product_within_reference_error(gr, port, m, k, n):
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(7000 + m * 131 + k)
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    ge, re_ = _errs(port, x, w, got, 2048, rng)
    gm, gx, rm, rx = np.median(ge), ge.max(), np.median(re_), re_.max()
    print(f"m={m} k={k} n={n}: GPU median 2^{np.log2(max(gm, 1e-300)):.1f} max 2^{np.log2(max(gx, 1e-300)):.1f}; "
          f"reference 2^{np.log2(max(rm, 1e-300)):.1f} / 2^{np.log2(max(rx, 1e-300)):.1f}")
    assert gm <= 4 * rm and gx <= 4 * rx


def test_short_a_rows_and_columns_far_apart_in_scale(gr, port):
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(7100)
    m, k, n = 10, 700, 96
    rs = np.exp2(rng.integers(-30, 31, m).astype(np.float64))[:, None]
    cs = np.exp2(rng.integers(-30, 31, n).astype(np.float64))[None, :]
    x = split((rng.uniform(-1, 1, (m, k)) * rs).ravel(), 2, np.float32).reshape(m, k, 2)
    w = (rng.uniform(-1, 1, (k, n)) * cs).astype(np.float32)
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    ge, re_ = _errs(port, x, w, got, 2048, rng)
    assert np.median(ge) <= 4 * np.median(re_) and ge.max() <= 4 * re_.max()


def test_short_a_nonfinite_rows_and_columns_propagate(gr):
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(7200)
    m, k, n = 6, 200, 72
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    x[2, 17, 0] = np.inf
    x[4, 3, 0] = np.nan
    w[50, 9] = np.nan
    w[120, 40] = -np.inf
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    v = got[..., 0].astype(np.float64) + got[..., 1]
    assert not np.isfinite(v[2]).any() and np.isnan(v[4]).all()
    assert np.isnan(v[:, 9]).all() and not np.isfinite(v[:, 40]).any()
    clean = np.ones((m, n), bool)
    clean[[2, 4], :] = False
    clean[:, [9, 40]] = False
    assert np.isfinite(v[clean]).all()


def test_config3_class_layer_within_reference_error(gr, port):
    """W (10 x 1024) . A (1024 x 512): the short-A kernel within 4x of the
    reference's error, like the general FP64-pipe path it replaces here."""
    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(7300)
    m, k, n = 10, 1024, 512
    bound = 1.0 / np.sqrt(k)
    x = split(rng.uniform(-bound, bound, m * k), 2, np.float32).reshape(m, k, 2)
    w = np.maximum(rng.normal(0, 1, (k, n)), 0).astype(np.float32)  # ReLU activations: many zeros
    got = gr.run("mm_mcn", x, w, plan=mcf.FAST)
    ge, re_ = _errs(port, x, w, got, 2048, rng)
    assert np.median(ge) <= 4 * np.median(re_) and ge.max() <= 4 * re_.max()
