"""The reference's invariant audit (T/test_mct.cpp:449-473, Invariants.
HoldOnAllOperatorOutputs): every operator's output is ordered, nonoverlapping
(|c_i| <= ulp(c_{i-1})), zero-padded only at the end and above the format's
subnormal quantum, for nc 1..4 and B16 / B32 / B64.  The predicate is
host.satisfies_invariants (mc_ops.hpp:537-554); its CPU tests pin it on
hand-made cases, the GPU test applies it to device outputs."""
import numpy as np
import pytest

from mcgen import DT, random_mc
from paper_2207_08867_b200 import host


def test_predicate_known_cases():
    f32 = np.float32
    assert host.satisfies_invariants(np.array([[1.0, 2.0**-30, 0.0]], f32))
    assert not host.satisfies_invariants(np.array([[1.0, 0.0, 2.0**-30]], f32))  # interleaved zero
    assert not host.satisfies_invariants(np.array([[2.0**-40, 1.0]], f32))  # wrong order
    assert not host.satisfies_invariants(np.array([[1.0, 2.0**-20]], f32))  # overlap: > ulp(1) = 2^-23
    assert host.satisfies_invariants(np.array([[1.0, 2.0**-23]], f32))  # exactly one ulp
    assert not host.satisfies_invariants(np.array([[np.inf, 0.0]], f32))
    # the subnormal-floor clause cannot fire on stored binary16 / binary32 values
    # (the reference stores doubles); on binary64 storage it is the 2^-1074 quantum
    assert host.satisfies_invariants(np.array([[2.0**-24, 0.0]], np.float16))
    assert host.ulp(1.0, np.float32) == 2.0**-23 and host.ulp(0.0, np.float32) == 2.0**-149
    assert host.ulp(1.5, np.float64) == 2.0**-52 and host.ulp(2.0**-150, np.float32) == 2.0**-149
    assert host.ulp(-3.0, np.float16) == 2.0**-9


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [16, 32, 64])
@pytest.mark.parametrize("nc", [1, 2, 3, 4])
def test_invariants_hold_on_all_operator_outputs(bits, nc):
    import gpu_util as gr

    rng = np.random.default_rng(33 + 10 * nc + bits)
    dt = DT[bits]
    n = 4000
    lo, hi = (-4, 4) if bits == 16 else (-8, 8)
    x = random_mc(rng, n, nc, dt, lo, hi)
    y = random_mc(rng, n, nc, dt, lo, hi)
    # divisors kept away from zero (config 0's rule; Mul-MCN divides by 1 / y):
    # a quotient beyond the format's range (binary16: 65504) is a legitimate
    # non-finite result, which the audit rejects
    yd = y.copy()
    yd[..., 0] = (yd[..., 0].astype(np.float64) + np.sign(yd[..., 0]) * 0.5).astype(dt)
    v = np.asarray(rng.uniform(-8.0, 8.0), dt)  # a scalar operand, as in the reference test
    for name, out in (("grow_expn", gr.run("grow_expn", x, v)), ("scaling_n", gr.run("scaling_n", x, v)),
                      ("add_mcn", gr.run("add_mcn", x, y)), ("div_mcn", gr.run("div_mcn", x, yd)),
                      ("mul_mcn", gr.run("mul_mcn", x, yd)), ("mul_mcn_slow", gr.run("mul_mcn_slow", x, y)),
                      ("square_mcn", gr.run("square_mcn", x))):
        assert host.satisfies_invariants(out), (name, bits, nc)
    xe = x[np.abs(x[:, 0].astype(np.float64)) < 5.0]
    assert host.satisfies_invariants(gr.run("exp_mcn", xe)), ("exp_mcn", bits, nc)
