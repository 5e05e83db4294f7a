"""MC-MLP training step (config 3) on the GPU against the reference's own
training loop (golden trajectory from oracle/_ref: MCSequential, MCLinear,
ReLU, cross_entropy_loss, Tape, MCSGD compiled unmodified).

* reference-order plan, one process: losses and final MC parameters
  bit-identical to the reference's at every step;
* FAST plan: per-step loss within 1e-6 relative of the reference (the forward
  products differ from the reference's only in the last bit of some outputs);
* data-parallel semantics emulated on one GPU: two half-batch shards whose
  gradients are summed equal the full-batch step within binary32 rounding.
"""
import os

import numpy as np
import pytest

from mcgen import assert_bits

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_mlp.npz"))


def _setup(plan):
    import torch

    import paper_2207_08867_b200 as mcf
    from paper_2207_08867_b200 import mlp

    dims = [int(d) for d in G["dims"]]
    L = len(dims) - 1
    params = [(G[f"w{l}"], G[f"b{l}"]) for l in range(L)]
    model = mlp.MCMLP(dims, params, lr=float(G["lr"][0]), plan=plan)
    xt = torch.from_numpy(np.ascontiguousarray(G["x"].T)).cuda()
    y = torch.from_numpy(G["y"]).cuda()
    return model, xt, y, dims, L, mcf


def test_reference_order_training_is_bitwise():
    import paper_2207_08867_b200 as mcf

    model, xt, y, dims, L, _ = _setup(mcf.SEQUENTIAL)
    n = xt.shape[1]
    losses = [model.loss_value(model.step(xt, y, n), n) for _ in range(len(G["losses"]))]
    assert np.array_equal(np.array(losses, np.float32).view(np.uint32), G["losses"].view(np.uint32)), (losses, G["losses"])
    for l, (w, b) in enumerate(model.params_numpy()):
        assert_bits(w, G[f"w{l}_final"], f"W{l}")
        assert_bits(b, G[f"b{l}_final"], f"b{l}")


def test_fast_plan_training_tracks_reference():
    import paper_2207_08867_b200 as mcf

    model, xt, y, dims, L, _ = _setup(mcf.FAST)
    n = xt.shape[1]
    losses = np.array([model.loss_value(model.step(xt, y, n), n) for _ in range(len(G["losses"]))])
    rel = np.abs(losses - G["losses"]) / np.abs(G["losses"])
    print("FAST vs reference loss rel diff per step:", rel)
    assert rel.max() <= 1e-6


def test_data_parallel_shards_sum_to_full_batch():
    import torch

    import paper_2207_08867_b200 as mcf

    model_a, xt, y, dims, L, _ = _setup(mcf.SEQUENTIAL)
    model_b, _, _, _, _, _ = _setup(mcf.SEQUENTIAL)
    n = xt.shape[1]
    h = n // 2
    # full batch on model_a
    la = model_a.loss_value(model_a.step(xt, y, n), n)
    # two shards on model_b: run the forward/backward of each half, sum grads by hand
    grads = []
    loss_sum = 0.0
    for sl in (slice(0, h), slice(h, n)):
        m, _, _, _, _, _ = _setup(mcf.SEQUENTIAL)
        m.lr = 0.0  # gradient only: the update is the identity
        loss = m.loss_value(m.step(xt[:, sl].contiguous(), y[sl].contiguous(), n), n)
        loss_sum += loss
        grads.append(m.grads.flat.clone())
    total = grads[0] + grads[1]
    full, _, _, _, _, _ = _setup(mcf.SEQUENTIAL)
    full.lr = 0.0
    full.step(xt, y, n)
    torch.cuda.synchronize()
    diff = (total - full.grads.flat).abs().max().item()
    scale = full.grads.flat.abs().max().item()
    assert diff <= 1e-5 * scale, (diff, scale)
    assert abs(loss_sum - la) <= 1e-5 * abs(la)


def _ordered_gemm_np(A, B):
    """matmul2d (ndarray.hpp:147-165): fl_mul then fl_add, k increasing, from 0."""
    acc = np.zeros((A.shape[0], B.shape[1]), np.float32)
    for k in range(A.shape[1]):
        acc = (acc + (A[:, k, None] * B[None, k, :]).astype(np.float32)).astype(np.float32)
    return (np.float32(0) + acc).astype(np.float32)


# shapes chosen so each tile configuration of mcf_gemm_f32_ordered runs
# (128x128, 128x64, 64x64, 32x32, 16x16 -- picked by the CTA count) with ragged edges
@pytest.mark.parametrize("m,n,k", [(2000, 1300, 37), (1100, 1100, 40), (700, 800, 21), (300, 500, 70), (10, 1024, 300)])
@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0), (0, 0), (1, 1)])
def test_ordered_gemm_bitwise(m, n, k, ta, tb):
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(m + 7 * n + k + 100 * ta + 10 * tb)
    A = (rng.standard_normal((m, k)) * np.exp2(rng.integers(-6, 6, (m, k)))).astype(np.float32)
    B = (rng.standard_normal((k, n)) * np.exp2(rng.integers(-6, 6, (k, n)))).astype(np.float32)
    mask = rng.standard_normal((m, n)).astype(np.float32)
    want = _ordered_gemm_np(A, B)
    want_masked = np.where(mask > 0, want, np.float32(0)).astype(np.float32)
    a_st = np.ascontiguousarray(A.T if ta else A)
    b_st = np.ascontiguousarray(B.T if tb else B)
    da, db = torch.from_numpy(a_st).cuda(), torch.from_numpy(b_st).cuda()
    dm = torch.from_numpy(mask).cuda()
    lib = mcf.lib()
    for use_mask, ref in ((False, want), (True, want_masked)):
        dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
        rc = lib.mcf_gemm_f32_ordered(ta, tb, da.data_ptr(), a_st.shape[1], db.data_ptr(), b_st.shape[1],
                                      dc.data_ptr(), n, m, n, k, dm.data_ptr() if use_mask else None, None)
        assert rc == 0, lib.mcf_last_error()
        torch.cuda.synchronize()
        assert_bits(dc.cpu().numpy(), ref, f"gemm ta={ta} tb={tb} {m}x{n}x{k} mask={use_mask}")


@pytest.mark.parametrize("rows,n", [(1024, 8192), (37, 300), (10, 129)])
def test_ordered_rowsum_bitwise(rows, n):
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(rows * 3 + n)
    g = (rng.standard_normal((rows, n)) * np.exp2(rng.integers(-10, 10, (rows, n)))).astype(np.float32)
    want = np.zeros(rows, np.float32)
    for j in range(n):
        want = (want + g[:, j]).astype(np.float32)
    dg = torch.from_numpy(g).cuda()
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_rowsum_f32_ordered(dg.data_ptr(), rows, n, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert_bits(out.cpu().numpy(), want, "row sums")


def test_loss_sum_is_left_to_right_over_slabs():
    """The loss's binary32 sum runs left to right from 0 (autodiff.hpp:572)
    across the kernel's 2048-term shared-memory slabs."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(5)
    classes, n = 10, 5000
    logits = torch.from_numpy((rng.standard_normal((classes, n)) * 4).astype(np.float32)).cuda()
    labels = torch.from_numpy(rng.integers(0, classes, n).astype(np.int32)).cuda()
    grad = torch.empty((classes, n), dtype=torch.float32, device="cuda")
    terms = torch.empty(n, dtype=torch.float32, device="cuda")
    tsum = torch.empty(1, dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_mlp_cross_entropy(logits.data_ptr(), labels.data_ptr(), classes, n, n, grad.data_ptr(),
                                     terms.data_ptr(), tsum.data_ptr(), None) == 0
    torch.cuda.synchronize()
    t = terms.cpu().numpy()
    acc = np.float32(0)
    for v in t:
        acc = np.float32(acc + v)
    assert_bits(tsum.cpu().numpy(), np.array([acc], np.float32), "loss sum")


@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0)])
def test_fast_plan_backward_gemm_and_rowsum(ta, tb):
    """Plan FAST's backward pieces (FP32 library GEMM + ReLU mask, tree row
    sums) against a binary64 reference: binary32-level relative error."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(9 + ta)
    m, n, k = 300, 500, 700
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    mask = rng.standard_normal((m, n)).astype(np.float32)
    want = np.where(mask > 0, A.astype(np.float64) @ B.astype(np.float64), 0.0)
    a_st = np.ascontiguousarray(A.T if ta else A)
    b_st = np.ascontiguousarray(B.T if tb else B)
    da, db, dm = (torch.from_numpy(v).cuda() for v in (a_st, b_st, mask))
    dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_gemm_f32_fast(ta, tb, da.data_ptr(), a_st.shape[1], db.data_ptr(), b_st.shape[1], dc.data_ptr(),
                                 n, m, n, k, dm.data_ptr(), None) == 0, lib.mcf_last_error()
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    assert lib.mcf_rowsum_f32_fast(dc.data_ptr(), m, n, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    got = dc.cpu().numpy().astype(np.float64)
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    assert np.all(np.abs(got - want) <= 1e-5 * scale), "gemm_f32_fast"
    rs = got.sum(axis=1)
    assert np.allclose(out.cpu().numpy(), rs, rtol=1e-5, atol=1e-5 * np.abs(got).sum(axis=1).max()), "rowsum"


@pytest.mark.parametrize("relu", [0, 1])
def test_fused_linear_forward_equals_product_then_bias_act(relu):
    """Plan FAST's fused layer (bias / approx / ReLU in the tensor-core
    product's epilogue, fallback outputs included) gives the same bits as the
    product written out and mcf_mlp_bias_act applied to it."""
    import torch

    import paper_2207_08867_b200 as mcf
    from mcgen import split

    rng = np.random.default_rng(80 + relu)
    out_dim, in_dim, n = 200, 300, 500
    w = torch.from_numpy(split(rng.uniform(-0.1, 0.1, out_dim * in_dim), 2, np.float32)
                         .reshape(out_dim, in_dim, 2)).cuda()
    a = torch.from_numpy(np.maximum(rng.standard_normal((in_dim, n)), 0).astype(np.float32)).cuda()
    b = torch.from_numpy(split(rng.uniform(-0.1, 0.1, out_dim), 2, np.float32).reshape(out_dim, 2)).cuda()
    lib = mcf.lib()
    f32 = dict(dtype=torch.float32, device="cuda")
    z = torch.empty((out_dim, n, 2), **f32)
    h1, a1 = torch.empty((out_dim, n), **f32), torch.empty((out_dim, n), **f32)
    h2, a2 = torch.empty((out_dim, n), **f32), torch.empty((out_dim, n), **f32)
    assert lib.mcf_mlp_linear_fwd(w.data_ptr(), 2, a.data_ptr(), out_dim, in_dim, n, b.data_ptr(), relu,
                                  z.data_ptr(), h1.data_ptr(), a1.data_ptr(), mcf.FAST, None) == 0
    assert lib.mcf_bmm_mcn(mcf.B32, w.data_ptr(), 2, a.data_ptr(), 1, out_dim, in_dim, n, 0, z.data_ptr(),
                           mcf.FAST, 1, None) == 0
    assert lib.mcf_mlp_bias_act(z.data_ptr(), 2, b.data_ptr(), out_dim, n, relu, h2.data_ptr(), a2.data_ptr(),
                                None) == 0
    torch.cuda.synchronize()
    assert_bits(h1.cpu().numpy(), h2.cpu().numpy(), "h")
    assert_bits(a1.cpu().numpy(), a2.cpu().numpy(), "act")


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(130, 77, 1000), (64, 200, 4100), (257, 96, 65)])
def test_fast_gemm_int8_digits_binary32_accuracy(ta, tb, m, n, k):
    """The binary32 GEMM on the int8 tensor cores (four balanced digits per
    operand, exact int32 diagonal sums) for every operand layout, ragged k and
    n, rows of very different magnitude and an all-zero row: error within the
    binary32 GEMM bound (1e-5 sum |a||b|), ReLU mask applied."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(1000 + 10 * ta + tb + m)
    A = (rng.standard_normal((m, k)) * np.exp2(rng.integers(-20, 20, (m, 1)))).astype(np.float32)
    B = (rng.standard_normal((k, n)) * np.exp2(rng.integers(-20, 20, (1, n)))).astype(np.float32)
    A[3] = 0.0
    mask = rng.standard_normal((m, n)).astype(np.float32)
    want = np.where(mask > 0, A.astype(np.float64) @ B.astype(np.float64), 0.0)
    a_st = np.ascontiguousarray(A.T if ta else A)
    b_st = np.ascontiguousarray(B.T if tb else B)
    da, db, dm = (torch.from_numpy(v).cuda() for v in (a_st, b_st, mask))
    dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_gemm_f32_fast(ta, tb, da.data_ptr(), a_st.shape[1], db.data_ptr(), b_st.shape[1], dc.data_ptr(),
                                 n, m, n, k, dm.data_ptr(), None) == 0, lib.mcf_last_error()
    got = dc.cpu().numpy().astype(np.float64)
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    err = np.abs(got - want)
    assert np.all(err <= 1e-5 * scale + 1e-300), float((err / np.maximum(scale, 1e-300)).max())
    assert np.all(got[3] == 0.0)
    # the products themselves (no mask) stay far below the bound on ordinary data
    dc2 = torch.empty((m, n), dtype=torch.float32, device="cuda")
    assert lib.mcf_gemm_f32_fast(ta, tb, da.data_ptr(), a_st.shape[1], db.data_ptr(), b_st.shape[1], dc2.data_ptr(),
                                 n, m, n, k, None, None) == 0
    g2 = dc2.cpu().numpy().astype(np.float64)
    rel = np.abs(g2 - A.astype(np.float64) @ B.astype(np.float64)) / np.maximum(scale, 1e-300)
    assert rel.max() <= 1e-6, float(rel.max())


def test_fast_gemm_int8_nonfinite_rows_are_nan():
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(77)
    m, n, k = 100, 80, 300
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    A[5, 7] = np.inf
    B[11, 9] = np.nan
    da, db = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dc = torch.empty((m, n), dtype=torch.float32, device="cuda")
    lib = mcf.lib()
    assert lib.mcf_gemm_f32_fast(0, 0, da.data_ptr(), k, db.data_ptr(), n, dc.data_ptr(), n, m, n, k, None, None) == 0
    got = dc.cpu().numpy()
    assert np.all(np.isnan(got[5])) and np.all(np.isnan(got[:, 9]))
    ok = np.ones((m, n), bool)
    ok[5] = False
    ok[:, 9] = False
    want = A.astype(np.float64) @ B.astype(np.float64)
    assert np.allclose(got[ok], want[ok], rtol=0, atol=1e-5 * np.abs(want[ok]).max())


def test_config3_fast_tracks_reference_within_spread():
    """Config 3's network (784-1024-1024-10, nc=2, the bench's init and data
    generators) at a reduced batch of 512 for 6 steps: plan FAST (int8
    tensor-core forward with the fused bias / approx / ReLU epilogue, int8
    digit backward GEMMs) against the reference-order plan, which is
    bit-identical to the reference (test_reference_order_training_is_bitwise).
    Bound per step: 4x the reference's own summation-order spread,
    measured as the same reference-order run on the batch in reversed sample
    order (every binary32 gradient sum over the batch and the loss sum run in
    the other order), running max over the steps so far, floored at 1 ulp of
    the loss."""
    import torch

    import paper_2207_08867_b200 as mcf
    from paper_2207_08867_b200 import mlp

    dims, n, steps = [784, 1024, 1024, 10], 512, 6
    params = mlp.init_params(dims, 2)
    xb, yb = mlp.make_batch(n)

    def run(plan, order):
        model = mlp.MCMLP(dims, params, lr=0.01, plan=plan)
        xt = torch.from_numpy(np.ascontiguousarray(xb[order].T)).cuda()
        yt = torch.from_numpy(np.ascontiguousarray(yb[order])).cuda()
        return np.array([model.loss_value(model.step(xt, yt, n), n) for _ in range(steps)], np.float64)

    fwd = np.arange(n)
    ref = run(mcf.SEQUENTIAL, fwd)
    ref_rev = run(mcf.SEQUENTIAL, fwd[::-1])
    fast = run(mcf.FAST, fwd)
    spread = np.maximum.accumulate(np.abs(ref - ref_rev))
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    bound = 4 * np.maximum(spread, ulp)
    diff = np.abs(fast - ref)
    print("reference losses", ref, "\nreversed-order spread", spread, "\nFAST diff", diff)
    assert np.all(diff <= bound), (diff, bound)
    assert ref[-1] < ref[0]  # it trains


@pytest.mark.parametrize("plan_name", ["SEQUENTIAL", "FAST"])
def test_captured_step_replays_the_bits_of_direct_steps(plan_name):
    """MCMLP.capture: the step as a CUDA graph (three streams, no allocation
    inside) gives the losses and parameters of direct step() calls bit for bit;
    the reference-order plan's graph still reproduces the reference's
    trajectory."""
    import paper_2207_08867_b200 as mcf

    plan = getattr(mcf, plan_name)
    direct, xt, y, dims, L, _ = _setup(plan)
    graphed, xt2, y2, *_ = _setup(plan)
    n = xt.shape[1]
    steps = len(G["losses"])
    want = [direct.loss_value(direct.step(xt, y, n), n) for _ in range(steps)]
    replay = graphed.capture(xt2, y2, n)  # two real steps happen inside
    got = [graphed.loss_value(replay(), n) for _ in range(steps - 2)]
    assert np.array_equal(np.array(got, np.float32).view(np.uint32), np.array(want[2:], np.float32).view(np.uint32))
    for l, ((w, b), (w2, b2)) in enumerate(zip(direct.params_numpy(), graphed.params_numpy())):
        assert_bits(w2, w, f"W{l}")
        assert_bits(b2, b, f"b{l}")
    if plan_name == "SEQUENTIAL":
        assert np.array_equal(np.array(got, np.float32).view(np.uint32), G["losses"][2:].view(np.uint32))


@pytest.mark.parametrize("ta,k,m,n,masked", [(1, 10, 1024, 512, True), (0, 10, 70, 260, True), (1, 16, 33, 128, False),
                                             (0, 1, 5, 4, True), (1, 7, 1000, 1028, True)])
def test_fast_gemm_short_k_is_bitwise_the_ordered_gemm(ta, k, m, n, masked):
    """Plan FAST's small-K kernel (the class layer's dA = approx(W)^T G, K = 10
    classes; csrc/mlp_fast.cu k_gemm_smallk) computes fl_mul then fl_add in k
    order like the reference's matmul2d: every output equals
    mcf_gemm_f32_ordered bit for bit, with and without the ReLU mask."""
    import torch

    import paper_2207_08867_b200 as mcf

    rng = np.random.default_rng(500 + k + m)
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    mask = rng.standard_normal((m, n)).astype(np.float32)
    a_st = np.ascontiguousarray(A.T if ta else A)
    da, db, dm = (torch.from_numpy(v).cuda() for v in (a_st, B, mask))
    lib = mcf.lib()
    outs = []
    for fn in (lib.mcf_gemm_f32_fast, lib.mcf_gemm_f32_ordered):
        dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
        assert fn(ta, 0, da.data_ptr(), a_st.shape[1], db.data_ptr(), n, dc.data_ptr(), n, m, n, k,
                  dm.data_ptr() if masked else None, None) == 0, lib.mcf_last_error()
        torch.cuda.synchronize()
        outs.append(dc.cpu().numpy())
    assert_bits(outs[0], outs[1], "small-K gemm vs ordered gemm")
