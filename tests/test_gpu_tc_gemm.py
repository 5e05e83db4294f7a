"""The hand-written tcgen05 int8 GEMM (tc_gemm.cu) against independent products.

int32 mode: every entry of C_b = A_b . B_b^T compared with cuBLASLt's
torch._int_mm (and numpy at small sizes); residue mode: the int8 outputs are
the exact symmetric residues of those products modulo the CRT scheme's moduli.
Shapes cover partial tiles in every dimension (M, N not multiples of 128 /
256; K not a multiple of the 128-byte stage) and the int32 extremes.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tc(a, b, moduli=None, ldo=None):
    import torch

    import paper_2207_08867_b200 as mcf

    batch, m, kp = a.shape
    n = b.shape[1]
    ldo = ldo or (n + 15) // 16 * 16
    out = torch.zeros((batch, m, ldo), dtype=torch.int8 if moduli is not None else torch.int32, device="cuda")
    mods = None
    if moduli is not None:
        mods = (C.c_int * batch)(*moduli)
    rc = mcf.lib().mcf_tc_gemm_s8(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, kp, batch, ldo, mods, None)
    assert rc == 0, mcf.lib().mcf_last_error().decode()
    torch.cuda.synchronize()
    return out


def _ref(a, b):
    import torch

    return torch.stack([torch._int_mm(a[i], b[i].t()) for i in range(a.shape[0])])


@pytest.mark.parametrize("batch,m,n,kp", [(1, 128, 256, 128), (3, 300, 520, 4096), (2, 100, 72, 32),
                                          (1, 129, 257, 160), (2, 256, 16, 16384), (17, 512, 512, 1024)])
def test_int32_products_match(batch, m, n, kp):
    import torch

    g = torch.Generator(device="cuda").manual_seed(batch * 1000 + m + n + kp)
    a = torch.randint(-128, 128, (batch, m, kp), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-128, 128, (batch, n, kp), dtype=torch.int8, device="cuda", generator=g)
    got = _tc(a, b)[:, :, :n]
    if m % 8 == 0 and n % 8 == 0 and kp % 8 == 0 and m > 16:
        want = _ref(a, b)
    else:
        an, bn = a.cpu().numpy().astype(np.float64), b.cpu().numpy().astype(np.float64)
        want = torch.from_numpy(np.einsum("bmk,bnk->bmn", an, bn).astype(np.int32)).cuda()
    assert torch.equal(got, want)


def test_int32_extremes():
    """All -128: every product 2^14, |C| = K 2^14 at K = 65536 - 16 (just
    below 2^30); mixed signs cancel exactly."""
    import torch

    kp = 65536 - 16
    a = torch.full((1, 128, kp), -128, dtype=torch.int8, device="cuda")
    b = torch.full((1, 256, kp), -128, dtype=torch.int8, device="cuda")
    b[0, 1::2, :] = 127
    got = _tc(a, b).cpu().numpy()[:, :, :256]
    assert np.all(got[0, :, 0::2] == kp * 16384)
    assert np.all(got[0, :, 1::2] == -kp * 128 * 127)


@pytest.mark.parametrize("kp", [4096, 20000 // 32 * 32])
def test_residue_mode(kp):
    import torch

    import paper_2207_08867_b200 as mcf

    n_mod = 17
    mods = (C.c_int * 22)()
    assert mcf.lib().mcf_fast_tc_crt_table(22, mods, None, None, None, None) > 0
    moduli = list(mods)[:n_mod]
    g = torch.Generator(device="cuda").manual_seed(kp)
    m, n = 200, 300
    a = torch.randint(-128, 128, (n_mod, m, kp), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-128, 128, (n_mod, n, kp), dtype=torch.int8, device="cuda", generator=g)
    a[:, 0, :] = -128
    b[:, 0, :] = -128  # C[0, 0] = kp 2^14, the largest sum
    got = _tc(a, b, moduli, ldo=304).cpu().numpy()[:, :, :n].astype(np.int64)
    c = np.einsum("bmk,bnk->bmn", a.cpu().numpy().astype(np.float64), b.cpu().numpy().astype(np.float64)).astype(np.int64)
    for t, mm in enumerate(moduli):
        r = c[t] % mm
        r = np.where(r > mm // 2, r - mm, r)
        if mm == 256:  # 128 and -128 are the same residue; the int8 output holds -128
            r = np.where(r == 128, -128, r)
        assert np.array_equal(got[t], r), mm


def test_rate_vs_library():
    """Timing printout (not a bar): the CRT product's 17 batched 4096^3 GEMMs
    on this kernel and on cuBLASLt."""
    import torch

    import paper_2207_08867_b200 as mcf

    batch, m, n, kp = 17, 4096, 4096, 4096
    a = torch.randint(-128, 128, (batch, m, kp), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (batch, n, kp), dtype=torch.int8, device="cuda")
    out = torch.empty((batch, m, n), dtype=torch.int8, device="cuda")
    mods = (C.c_int * 22)()
    mcf.lib().mcf_fast_tc_crt_table(22, mods, None, None, None, None)

    def ours():
        assert mcf.lib().mcf_tc_gemm_s8(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, kp, batch, n, mods,
                                        torch.cuda.current_stream().cuda_stream) == 0

    def lib_():
        for i in range(batch):
            torch._int_mm(a[i], b[i].t())

    res = {}
    for name, f in (("tcgen05", ours), ("cuBLASLt", lib_)):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = (ms, 2.0 * batch * m * n * kp / ms / 1e9)
    print("17 x 4096^3 int8:", {k: f"{v[0]:.3f} ms, {v[1]:.0f} TOPS" for k, v in res.items()})
