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
