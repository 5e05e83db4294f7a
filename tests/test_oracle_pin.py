"""Pin the C restatement (oracle/libmcf_oracle.so) to the reference itself.

The reference's header-only C++ is compiled here unmodified into
oracle/_ref/libmcf_ref.so; every entry point of the restatement must agree
with it bit for bit (NaN payloads aside) on seeded inputs covering every
precision the reference supports, nc 1..8 and the awkward cases.
"""
import numpy as np
import pytest

import oracle
from mcgen import DT, assert_bits, nasty_mc, random_mc

PRECS = [16, 32, 64]


def inputs(seed, n, nc, bits, nasty=False, nonfinite=False):
    rng = np.random.default_rng(seed)
    dt = DT[bits]
    if nasty:
        return nasty_mc(rng, n, nc, dt, allow_nonfinite=nonfinite)
    lo, hi = (-4, 4) if bits == 16 else (-8, 8)
    return random_mc(rng, n, nc, dt, lo, hi)


def wp(seed, n, bits, lo=-8, hi=8):
    rng = np.random.default_rng(seed)
    if bits == 16:
        lo, hi = -4, 4
    return (rng.uniform(-1, 1, n) * np.exp2(rng.uniform(lo, hi, n))).astype(DT[bits])


@pytest.mark.parametrize("bits", PRECS)
def test_eft_arrays(port, ref, bits):
    a, b = wp(1, 4000, bits), wp(2, 4000, bits)
    for f in ("two_sum",):
        assert_bits(port.two_sum(a, b)[0], ref.two_sum(a, b)[0], f)
        assert_bits(port.two_sum(a, b)[1], ref.two_sum(a, b)[1], f)
    for use_fma in (True, False):
        p1, e1 = port.two_prod(a, b, use_fma)
        p2, e2 = ref.two_prod(a, b, use_fma)
        assert_bits(p1, p2, "two_prod p")
        assert_bits(e1, e2, "two_prod e")


@pytest.mark.parametrize("bits", PRECS)
@pytest.mark.parametrize("nasty", [False, True])
def test_renorm_family(port, ref, bits, nasty):
    for nc in range(1, 9):
        h = inputs(10 + nc, 600, nc, bits, nasty=True, nonfinite=nasty)
        for r_nc in sorted({1, max(1, nc - 1), nc, min(8, nc + 1)}):
            assert_bits(port.renormalize(h, r_nc), ref.renormalize(h, r_nc), f"renorm {nc}->{r_nc}")
            assert_bits(port.simple_renorm(h, r_nc), ref.simple_renorm(h, r_nc), f"simple {nc}->{r_nc}")
        assert_bits(port.approx(h), ref.approx(h), "approx")
        assert_bits(port.negate(h), ref.negate(h), "negate")


@pytest.mark.parametrize("bits", PRECS)
@pytest.mark.parametrize("nasty", [False, True])
def test_ops_with_tensor_operand(port, ref, bits, nasty):
    for nc in range(1, 9):
        x = inputs(20 + nc, 500, nc, bits, nasty=nasty, nonfinite=nasty)
        y = inputs(40 + nc, 500, nc, bits, nasty=nasty, nonfinite=nasty)
        y[..., 0] += np.sign(y[..., 0]).astype(y.dtype) * y.dtype.type(0.5)  # keep divisors off 0 mostly
        v = wp(30 + nc, 500, bits)
        for vv in (v, v[:1], v[:0] if False else v[:1]):
            assert_bits(port.grow_expn(x, vv), ref.grow_expn(x, vv), f"grow nc={nc}")
            assert_bits(port.scaling_n(x, vv), ref.scaling_n(x, vv), f"scaling nc={nc}")
            if nc < 8:
                assert_bits(port.scaling_n(x, vv, True), ref.scaling_n(x, vv, True), f"scaling exp nc={nc}")
            assert_bits(port.div_n(vv, y), ref.div_n(vv, y), f"div_n nc={nc}")


@pytest.mark.parametrize("bits", PRECS)
@pytest.mark.parametrize("nasty", [False, True])
def test_binary_ops(port, ref, bits, nasty):
    for nc in range(1, 9):
        x = inputs(50 + nc, 400, nc, bits, nasty=nasty, nonfinite=nasty)
        y = inputs(60 + nc, 400, nc, bits, nasty=nasty, nonfinite=nasty)
        for name in ("add_mcn", "div_mcn", "mul_mcn", "mul_mcn_slow"):
            assert_bits(getattr(port, name)(x, y), getattr(ref, name)(x, y), f"{name} nc={nc}")
        assert_bits(port.square_mcn(x), ref.square_mcn(x), f"square nc={nc}")


@pytest.mark.parametrize("bits", PRECS)
def test_mixed_nc_padding(port, ref, bits):
    x = inputs(70, 300, 2, bits)
    y = inputs(71, 300, 3, bits)
    for name in ("add_mcn", "div_mcn", "mul_mcn", "mul_mcn_slow"):
        assert_bits(getattr(port, name)(x, y), getattr(ref, name)(x, y), name)
        assert_bits(getattr(port, name)(y, x), getattr(ref, name)(y, x), name)


@pytest.mark.parametrize("bits", PRECS)
def test_exp_libm_mode_matches_reference(port, ref, bits):
    for nc in range(1, 9):
        rng = np.random.default_rng(80 + nc)
        lim = 10.0 if bits != 16 else 4.0
        x = random_mc(rng, 500, nc, DT[bits], -6, 3)
        x = np.clip(x.astype(np.float64), -lim, lim).astype(DT[bits])
        assert_bits(port.exp_mcn(x, oracle.EXP_LIBM), ref.exp_mcn(x, oracle.EXP_LIBM), f"exp nc={nc}")


@pytest.mark.parametrize("bits", [16, 32, 64])
@pytest.mark.parametrize("nc", [1, 2, 3, 4])
def test_contractions(port, ref, bits, nc):
    rng = np.random.default_rng(90 + nc + bits)
    x = random_mc(rng, 3 * 5 * 7, nc, DT[bits], -3, 3).reshape(3, 5, 7, nc)
    w = wp(91, 3 * 7 * 4, bits, -3, 3).reshape(3, 7, 4)
    w2 = wp(92, 7 * 4, bits, -3, 3).reshape(7, 4)
    assert_bits(port.bmm_mcn(x, w), ref.bmm_mcn(x, w), "bmm")
    assert_bits(port.bmm_mcn(x, w2), ref.bmm_mcn(x, w2), "matmul 3/2")
    for leaf in (1, 2, 4):
        assert_bits(port.bmm_mcn(x, w, oracle.PAIRWISE_TREE, leaf), ref.bmm_mcn(x, w, oracle.PAIRWISE_TREE, leaf), "tree")
    rows = np.array([0, 2, 1, 2]); cols = np.array([3, 0, 1, 2])
    assert_bits(port.mm_mcn_sampled(x[0], w[0], rows, cols), ref.mm_mcn_sampled(x[0], w[0], rows, cols), "sampled")
    y = random_mc(rng, 4 * 7, nc, DT[bits], -3, 3).reshape(4, 7, nc)
    xx = random_mc(rng, 4 * 7, nc, DT[bits], -3, 3).reshape(4, 7, nc)
    assert_bits(port.dot_mcmc(xx, y), ref.dot_mcmc(xx, y), "dot_mcmc")
    yy = random_mc(rng, 7 * 5, nc, DT[bits], -3, 3).reshape(7, 5, nc)
    assert_bits(port.mm_mcmc_sampled(x[0], yy, rows, cols), ref.mm_mcmc_sampled(x[0], yy, rows, cols), "mm_mcmc")
    a = wp(93, 4 * 6, bits, -3, 3).reshape(4, 6)
    b = wp(94, 6 * 3, bits, -3, 3).reshape(6, 3)
    assert_bits(port.matmul2d(a, b), ref.matmul2d(a, b), "matmul2d")


def test_b16_rounding_matches_reference(port, ref):
    # the restatement's binary64 -> binary16 RN against the reference's
    # round_to_binary16 (precision.hpp:31-79), through fl_add of x + 0 in B16
    rng = np.random.default_rng(5)
    v = np.concatenate([
        rng.uniform(-1, 1, 20000) * np.exp2(rng.uniform(-27, 17, 20000)),
        np.array([65504.0, 65519.99, 65520.0, 2.0**-25, 2.0**-25 * 1.0000001, 2.0**-24 * 1.5, 0.0, -0.0]),
    ])
    got = np.array([port.round_b16(t) for t in v])
    want = v.astype(np.float16).astype(np.float64)  # numpy's direct double->half RN
    assert np.array_equal(np.signbit(got), np.signbit(want))
    assert np.array_equal(got, want)


# ---- MC activations: mc_relu_op, mc_softmax -----------------

@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 2), (64, 2), (32, 1), (64, 4)])
def test_mc_relu_port_equals_reference(port, ref, bits, nc):
    rng = np.random.default_rng(40 + nc + bits)
    x = random_mc(rng, 500, nc, DT[bits], -3, 3)
    x[::7] = 0
    x[5, -1] = -abs(x[5, -1]) if nc > 1 else x[5, -1]
    assert_bits(port.mc_relu(x), ref.mc_relu(x), f"mc_relu b{bits} nc{nc}")


@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 2), (64, 2), (32, 1)])
@pytest.mark.parametrize("shape,axis", [((37,), -1), ((9, 23), -1), ((23, 9), 0)])
def test_mc_softmax_port_equals_reference(port, ref, bits, nc, shape, axis):
    rng = np.random.default_rng(50 + nc + bits + len(shape))
    n = int(np.prod(shape))
    x = random_mc(rng, n, nc, DT[bits], -2, 2).reshape(*shape, nc)
    got = port.mc_softmax(x, axis, oracle.EXP_LIBM)
    want = ref.mc_softmax(x, axis, oracle.EXP_LIBM)
    assert_bits(got, want, f"mc_softmax b{bits} nc{nc} {shape} axis {axis}")


# ---- mct blobs: serialize.hpp ------------------------------

@pytest.mark.parametrize("bits,nc,shape", [(32, 2, (3, 4)), (16, 3, (5,)), (64, 1, (2, 2, 2)), (32, 8, (1,))])
def test_mct_json_matches_reference(ref, bits, nc, shape):
    import ctypes as C
    import json

    import torch

    from paper_2207_08867_b200 import serialize

    rng = np.random.default_rng(bits + nc)
    x = random_mc(rng, int(np.prod(shape)), nc, DT[bits], -8, 8).reshape(*shape, nc)
    x.reshape(-1)[:3] = [0.0, -0.0, np.inf]
    f = ref.lib.mcfref_mct_to_json
    f.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_char_p, C.c_int64]
    f.restype = C.c_int64
    shp = np.array(shape, np.int64)
    buf = C.create_string_buffer(1 << 20)
    n = f(oracle.prec_of(x), x.ctypes.data, nc, shp.ctypes.data, len(shape), buf, len(buf))
    assert n > 0
    want = json.loads(buf.value.decode())
    got = serialize.mct_to_json(torch.from_numpy(x))
    assert got == want
    back = serialize.mct_from_json(want, f"b{bits}").numpy()
    assert_bits(back, x, "round trip")
    with pytest.raises(ValueError, match="does not match requested"):
        serialize.mct_from_json(want, "b64" if bits != 64 else "b32")


# ---- hyperbolic distance pipeline: hyperbolic.hpp ---------------

@pytest.mark.parametrize("bits,nc,dim", [(32, 2, 3), (16, 2, 4), (64, 3, 2), (32, 1, 5), (64, 2, 6)])
def test_halfspace_arg_port_equals_reference(port, ref, bits, nc, dim):
    rng = np.random.default_rng(bits * 10 + nc + dim)
    n = 40
    tab = random_mc(rng, n * dim, nc, DT[bits], -2, 1).reshape(n, dim, nc)
    tab[:, -1, 0] = np.abs(tab[:, -1, 0]) + DT[bits](0.05)  # positive heights
    tab[3] = tab[4]  # coincident rows
    u = rng.integers(0, n, 300)
    v = rng.integers(0, n, 300)
    u[:2], v[:2] = [3, 7], [4, 7]
    got = port.halfspace_arg(tab, u, v)
    want = ref.halfspace_arg(tab, u, v)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_mlp_checkpoint_equals_reference(ref):
    """The MC-MLP checkpoint (nn.hpp:207-229): paper_2207_08867_b200.mlp
    writes the reference's checkpoint_to_json text byte for byte (keys sorted,
    dump(2)) for the same parameters, reads it back bit-exact, and raises the
    reference's errors on a foreign blob or a topology mismatch."""
    import ctypes as C
    import json

    from paper_2207_08867_b200 import mlp, serialize

    dims = [7, 5, 3]
    params = mlp.init_params(dims, 2, seed=44)
    params[0][0].reshape(-1)[:2] = [-0.0, np.float32(1e-40)]  # sign of zero and a subnormal survive
    flat = np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in params]).astype(np.float32)
    f = ref.lib.mcfref_mlp_checkpoint
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_int64]
    f.restype = C.c_int64
    d = np.array(dims, np.int32)
    buf = C.create_string_buffer(1 << 20)
    n = f(d.ctypes.data, len(dims) - 1, 2, flat.ctypes.data, buf, len(buf))
    assert n > 0
    want = buf.value.decode()
    got = mlp.checkpoint_to_json(dims, params)
    assert serialize.dumps(got) == want
    back = mlp.load_checkpoint(dims, json.loads(want))
    for (w, b), (w2, b2) in zip(params, back):
        assert_bits(w2, w, "W")
        assert_bits(b2, b, "b")
    with pytest.raises(ValueError, match="not a checkpoint blob"):
        mlp.load_checkpoint(dims, {"format": "mct"})
    with pytest.raises(ValueError, match="topology mismatch"):
        mlp.load_checkpoint([7, 6, 3], got)
