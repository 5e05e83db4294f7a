"""Out-of-bounds write checks for the int8 digit paths (compute-sanitizer is
not available on the GPU pool): outputs are written into larger buffers whose
guard regions hold a sentinel pattern, with ragged shapes that exercise the
padding of k, n (multiples of 16 / 32 in the digit planes) and the row
chunking; the guards must be untouched and the interior correct."""
import numpy as np
import pytest

from mcgen import split

pytestmark = pytest.mark.gpu

SENTINEL = np.float32(-12345.678)


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 1)])
def test_gemm_f32_int8_writes_stay_inside(ta, tb):
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(5 + ta)
    m, n, k = 97, 83, 141
    ldc = n + 9
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    a_st = np.ascontiguousarray(A.T if ta else A)
    b_st = np.ascontiguousarray(B.T if tb else B)
    da, db = torch.from_numpy(a_st).cuda(), torch.from_numpy(b_st).cuda()
    buf = torch.full((m + 3, ldc), float(SENTINEL), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_gemm_f32_fast(ta, tb, da.data_ptr(), a_st.shape[1], db.data_ptr(), b_st.shape[1], buf.data_ptr(),
                                 ldc, m, n, k, None, None) == 0, lib.mcf_last_error()
    got = buf.cpu().numpy()
    assert np.all(got[:m, n:] == SENTINEL), "row padding written"
    assert np.all(got[m:] == SENTINEL), "rows past m written"
    want = A.astype(np.float64) @ B.astype(np.float64)
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    assert np.all(np.abs(got[:m, :n] - want) <= 1e-5 * scale)


@pytest.mark.parametrize("nc", [2, 3])
def test_mm_mcmc_fp16_int8_writes_stay_inside(nc):
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(11 + nc)
    m, k, n = 70, 99, 66
    x = split(rng.uniform(-1, 1, m * k) / 64, nc, np.float16).reshape(m, k, nc)
    y = split(rng.uniform(-1, 1, k * n) / 64, nc, np.float16).reshape(k, n, nc)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    total = m * n * nc
    buf = torch.full((total + 4096,), -7.5, dtype=torch.float16, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_mm_mcmc(mcf.B16, dx.data_ptr(), dy.data_ptr(), nc, m, k, n, buf.data_ptr(), mcf.FAST, None) == 0, \
        lib.mcf_last_error()
    got = buf.cpu().numpy()
    assert np.all(got[total:] == np.float16(-7.5)), "written past the output"
    want = x.astype(np.float64).sum(-1) @ y.astype(np.float64).sum(-1)
    res = got[:total].reshape(m, n, nc).astype(np.float64).sum(-1)
    assert np.allclose(res, want, rtol=1e-3, atol=1e-6)


def test_mm_mct_tensorcore_ragged_writes_stay_inside():
    """MC x T (binary32 nc=2) on the tensor-core path with ragged n and k."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(21)
    m, k, n = 130, 77, 45
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    dx, dw = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    total = m * n * 2
    buf = torch.full((total + 4096,), float(SENTINEL), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_bmm_mcn(mcf.B32, dx.data_ptr(), 2, dw.data_ptr(), 1, m, k, n, 0, buf.data_ptr(), mcf.FAST, 1,
                           None) == 0, lib.mcf_last_error()
    got = buf.cpu().numpy()
    assert np.all(got[total:] == SENTINEL), "written past the output"
    want = x.astype(np.float64).sum(-1) @ w.astype(np.float64)
    res = got[:total].reshape(m, n, 2).astype(np.float64).sum(-1)
    assert np.allclose(res, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("numel", [1, 1023, 3 * 1024 + 13, 200003])
def test_elementwise_certified_ops_write_stay_inside(numel):
    """The binary32 nc=2 operators (TMA ring + ragged grid-stride tail, the
    certified tier and its fallbacks) write exactly numel x 2 components."""
    import torch

    import paper_2207_08867_b200 as mcf
    from mcgen import config_values

    rng = np.random.default_rng(numel)
    x = torch.from_numpy(split(config_values(rng, numel), 2, np.float32)).cuda()
    yv = config_values(rng, numel)
    y = torch.from_numpy(split(yv + np.sign(yv) * 0.5, 2, np.float32)).cuda()
    v = torch.from_numpy(config_values(rng, numel).astype(np.float32)).cuda()
    xe = torch.from_numpy(split(np.clip(config_values(rng, numel), -10, 10), 2, np.float32)).cuda()
    lib = mcf.lib()
    calls = {
        "grow": lambda o: lib.mcf_grow_expn(mcf.B32, x.data_ptr(), 2, v.data_ptr(), numel, o, numel, None),
        "scale": lambda o: lib.mcf_scaling_n(mcf.B32, x.data_ptr(), 2, v.data_ptr(), numel, 0, o, numel, None),
        "div_n": lambda o: lib.mcf_div_n(mcf.B32, v.data_ptr(), numel, y.data_ptr(), 2, o, numel, None),
        "add": lambda o: lib.mcf_add_mcn(mcf.B32, x.data_ptr(), 2, y.data_ptr(), 2, o, numel, None),
        "div": lambda o: lib.mcf_div_mcn(mcf.B32, x.data_ptr(), 2, y.data_ptr(), 2, o, numel, None),
        "mul": lambda o: lib.mcf_mul_mcn(mcf.B32, x.data_ptr(), 2, y.data_ptr(), 2, o, numel, None),
        "square": lambda o: lib.mcf_square_mcn(mcf.B32, x.data_ptr(), 2, o, numel, None),
        "exp": lambda o: lib.mcf_exp_mcn(mcf.B32, xe.data_ptr(), 2, o, numel, None),
    }
    for name, f in calls.items():
        buf = torch.full((2 * numel + 1024,), float(SENTINEL), dtype=torch.float32, device="cuda")
        assert f(buf.data_ptr()) == 0, (name, lib.mcf_last_error())
        got = buf.cpu().numpy()
        assert np.all(got[2 * numel:] == SENTINEL), f"{name}: written past the output"
        assert np.all(np.isfinite(got[: 2 * numel])), f"{name}: interior not fully written"


@pytest.mark.parametrize("m,k,n", [(10, 77, 68), (3, 513, 4), (16, 40, 132)])
def test_short_a_kernel_writes_stay_inside(m, k, n):
    """mm_skinny.cu (MC x T for m <= 16): ragged column tiles, K tails of the
    ring stage and the chunk; the words after the m x n x 2 outputs stay."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(31 + m)
    x = split(rng.uniform(-1, 1, m * k), 2, np.float32).reshape(m, k, 2)
    w = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    dx, dw = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    total = m * n * 2
    buf = torch.full((total + 4096,), float(SENTINEL), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_bmm_mcn(mcf.B32, dx.data_ptr(), 2, dw.data_ptr(), 1, m, k, n, 0, buf.data_ptr(), mcf.FAST, 1,
                           None) == 0, lib.mcf_last_error()
    got = buf.cpu().numpy()
    assert np.all(got[total:] == SENTINEL), "written past the output"
    want = x.astype(np.float64).sum(-1) @ w.astype(np.float64)
    res = got[:total].reshape(m, n, 2).astype(np.float64).sum(-1)
    assert np.allclose(res, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def test_small_k_gemm_writes_stay_inside():
    """k_gemm_smallk (mlp_fast.cu): a padded C (ldc > n) and rows past m keep the sentinel."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(41)
    m, n, k = 70, 260, 10
    ldc = n + 12
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    da, db = torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), torch.from_numpy(B).cuda()
    mask = torch.ones((m + 3, ldc), dtype=torch.float32, device="cuda")
    buf = torch.full((m + 3, ldc), float(SENTINEL), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_gemm_f32_fast(1, 0, da.data_ptr(), m, db.data_ptr(), n, buf.data_ptr(), ldc, m, n, k,
                                 mask.data_ptr(), None) == 0, lib.mcf_last_error()
    got = buf.cpu().numpy()
    assert np.all(got[:m, n:] == SENTINEL) and np.all(got[m:] == SENTINEL)
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert np.allclose(got[:m, :n], want, rtol=1e-5, atol=1e-5)
