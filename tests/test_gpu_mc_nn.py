"""MC activations on the GPU against the oracle:
mc_relu_op forward and mc_softmax (autodiff.hpp:340-413), every component
bit-identical (softmax: with the correctly rounded exp of exp_mcn; the
oracle port is pinned to the reference with libm exp in test_oracle_pin)."""
import numpy as np
import pytest

import oracle
from mcgen import DT, assert_bits, random_mc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gr():
    import gpu_util

    return gpu_util


@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 2), (64, 2), (32, 1), (64, 4), (16, 3)])
def test_mc_relu_bitwise(gr, port, bits, nc):
    rng = np.random.default_rng(60 + nc + bits)
    x = random_mc(rng, 3000, nc, DT[bits], -4, 4)
    x[::11] = 0
    assert_bits(gr.run("mc_relu", x), port.mc_relu(x), f"mc_relu b{bits} nc{nc}")


@pytest.mark.parametrize("bits,nc", [(32, 2), (32, 3), (16, 2), (64, 2), (32, 1)])
@pytest.mark.parametrize("shape,axis", [((131,), -1), ((64, 10), -1), ((10, 64), 0), ((300, 33), 1)])
def test_mc_softmax_bitwise(gr, port, bits, nc, shape, axis):
    rng = np.random.default_rng(70 + nc + bits + shape[0])
    n = int(np.prod(shape))
    x = random_mc(rng, n, nc, DT[bits], -2, 3).reshape(*shape, nc)
    got = gr.run("mc_softmax", x, axis=axis)
    want = port.mc_softmax(x, axis, oracle.EXP_CR)
    assert_bits(got, want, f"mc_softmax b{bits} nc{nc} {shape} axis {axis}")


def test_mc_softmax_rejects_rank3(gr):
    import torch

    import paper_2207_08867_b200 as mcf

    x = torch.zeros((2, 3, 4, 2), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError, match="rank 1/2"):
        mcf.mc_softmax(x)


def _arcosh_guarded(a, dt):
    """hyperbolic.hpp:160-170 on the host (libm log / log1p), rounded to P."""
    a = np.clip(a, 1.0, float(np.finfo(dt).max))
    small = a <= 1.0 + 1e-12
    with np.errstate(invalid="ignore"):
        inv = 1.0 / a
        big = np.log(a) + np.log1p(np.sqrt((1.0 - inv) * (1.0 + inv)))
    return np.where(small, np.sqrt(2.0 * (a - 1.0)), big).astype(dt).astype(np.float64)


@pytest.mark.parametrize("bits,nc,dim", [(32, 2, 3), (16, 2, 4), (64, 3, 2), (32, 1, 5), (64, 2, 6)])
def test_halfspace_distance(gr, port, bits, nc, dim):
    """Half-space model distances (hyperbolic.hpp:183-226):
    the MC arcosh argument bit-identical to the oracle (pinned to the
    reference), symmetric bitwise, the distance within four units of P's
    last place of the host arcosh (two libm calls and a sum on each side)."""
    import torch

    import paper_2207_08867_b200 as mcf

    dt = DT[bits]
    rng = np.random.default_rng(bits * 10 + nc + dim)
    n = 64
    tab = random_mc(rng, n * dim, nc, dt, -2, 1).reshape(n, dim, nc)
    tab[:, -1, 0] = np.abs(tab[:, -1, 0]) + dt(0.05)
    tab[3] = tab[4]
    u = rng.integers(0, n, 2000)
    v = rng.integers(0, n, 2000)
    u[:2], v[:2] = [3, 7], [4, 7]
    dist, arg = mcf.halfspace_distance(torch.from_numpy(tab).cuda(), u, v, return_arg=True)
    arg = arg.cpu().numpy()
    want = port.halfspace_arg(tab, u, v)
    assert np.array_equal(arg.view(np.uint64), want.view(np.uint64))
    d2, _ = mcf.halfspace_distance(torch.from_numpy(tab).cuda(), v, u, return_arg=True)
    assert np.array_equal(dist.cpu().numpy().view(np.uint64), d2.cpu().numpy().view(np.uint64)), "symmetry"
    dh = _arcosh_guarded(want, dt)
    dg = dist.cpu().numpy()
    ulp = np.spacing(np.abs(dh).astype(dt)).astype(np.float64)
    assert np.all(np.abs(dg - dh) <= 4 * ulp), "distance vs host arcosh"
    assert dg[0] == 0.0 and dg[1] == 0.0  # coincident rows, same row


@pytest.mark.parametrize("bits", [32, 16])
def test_halfspace_distance_domain(gr, bits):
    """halfspace_distance throws std::domain_error for a non-positive height
    (hyperbolic.hpp:219-224): the GPU entry raises ValueError with the
    reference's message; the argument alone (halfspace_arg) has no domain."""
    import torch

    import paper_2207_08867_b200 as mcf

    dt = DT[bits]
    rng = np.random.default_rng(bits)
    n, dim, nc = 16, 3, 2
    tab = random_mc(rng, n * dim, nc, dt, -2, 1).reshape(n, dim, nc)
    tab[:, -1, 0] = np.abs(tab[:, -1, 0]) + dt(0.05)
    mcf.halfspace_distance(torch.from_numpy(tab).cuda(), [0, 1], [2, 3])  # fine
    for bad in (0.0, -0.25):
        t2 = tab.copy()
        t2[5, -1, :] = 0
        t2[5, -1, 0] = dt(bad)
        with pytest.raises(ValueError, match="nonpositive height"):
            mcf.halfspace_distance(torch.from_numpy(t2).cuda(), [0, 5], [1, 2])
        with pytest.raises(ValueError, match="nonpositive height"):
            mcf.halfspace_distance(torch.from_numpy(t2).cuda(), [2], [5])
