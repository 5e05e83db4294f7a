"""Generate golden fixtures from the reference itself (run in the container
that has /root/reference).

Inputs are seeded; outputs come from oracle/_ref/libmcf_ref.so, i.e. the
reference's header-only C++ compiled unmodified.  The fixtures travel with
the repository, so GPU tests on a box without /root/reference still compare
against the reference's own bits.  Exp-MCN fixtures hold the reference's libm
result AND the correctly rounded variant from the oracle port, plus a mask of
the elements where they differ.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from mcgen import DT, nasty_mc, random_mc  # noqa: E402


def main():
    ref = oracle.Oracle("ref")
    port = oracle.Oracle("port")
    out = {}
    for bits, nc, n in ((32, 2, 4096), (32, 3, 2048), (16, 3, 2048), (64, 2, 1024), (32, 1, 1024)):
        rng = np.random.default_rng(1000 * bits + nc)
        dt = DT[bits]
        lo, hi = (-4, 4) if bits == 16 else (-8, 8)
        x = np.concatenate([random_mc(rng, n, nc, dt, lo, hi), nasty_mc(rng, n // 4, nc, dt)])
        y = np.concatenate([random_mc(rng, n, nc, dt, lo, hi), nasty_mc(rng, n // 4, nc, dt)])
        yd = y.copy()
        yd[..., 0] = (yd[..., 0].astype(np.float64) + np.sign(yd[..., 0]) * 0.5).astype(dt)
        v = (rng.uniform(-1, 1, x.shape[0]) * np.exp2(rng.uniform(lo, hi, x.shape[0]))).astype(dt)
        xe = np.clip(x.astype(np.float64), -10 if bits != 16 else -4, 10 if bits != 16 else 4).astype(dt)
        key = f"b{bits}_nc{nc}"
        out[f"{key}_x"], out[f"{key}_y"], out[f"{key}_yd"], out[f"{key}_v"], out[f"{key}_xe"] = x, y, yd, v, xe
        out[f"{key}_grow_expn"] = ref.grow_expn(x, v)
        out[f"{key}_scaling_n"] = ref.scaling_n(x, v)
        if nc < 8:
            out[f"{key}_scaling_n_x"] = ref.scaling_n(x, v, True)
        out[f"{key}_div_n"] = ref.div_n(v, yd)
        out[f"{key}_add_mcn"] = ref.add_mcn(x, y)
        out[f"{key}_div_mcn"] = ref.div_mcn(x, yd)
        out[f"{key}_mul_mcn"] = ref.mul_mcn(x, y)
        out[f"{key}_mul_mcn_slow"] = ref.mul_mcn_slow(x, y)
        out[f"{key}_square_mcn"] = ref.square_mcn(x)
        out[f"{key}_negate"] = ref.negate(x)
        out[f"{key}_approx"] = ref.approx(x)
        out[f"{key}_renormalize"] = ref.renormalize(x, nc)
        out[f"{key}_simple_renorm"] = ref.simple_renorm(x, nc)
        out[f"{key}_exp_mcn"] = ref.exp_mcn(xe)
        out[f"{key}_exp_mcn_cr"] = port.exp_mcn(xe, oracle.EXP_CR)
        a = (rng.uniform(-1, 1, 2048) * np.exp2(rng.uniform(lo, hi, 2048))).astype(dt)
        b = (rng.uniform(-1, 1, 2048) * np.exp2(rng.uniform(lo, hi, 2048))).astype(dt)
        out[f"{key}_a"], out[f"{key}_b"] = a, b
        out[f"{key}_two_sum"] = np.stack(ref.two_sum(a, b))
        out[f"{key}_two_prod"] = np.stack(ref.two_prod(a, b))
        # contractions: small mm / bmm / dot, reference order (bitwise pins)
        if nc < 8:
            xm = random_mc(rng, 24 * 64, nc, dt, -3, 3).reshape(24, 64, nc)
            wm = (rng.uniform(-1, 1, 64 * 16) * np.exp2(rng.uniform(-3, 3, 64 * 16))).astype(dt).reshape(64, 16)
            out[f"{key}_mm_x"], out[f"{key}_mm_w"] = xm, wm
            out[f"{key}_mm"] = ref.mm_mcn(xm, wm)
            out[f"{key}_mm_tree"] = ref.bmm_mcn(xm, wm, oracle.PAIRWISE_TREE, 2)
            ym = random_mc(rng, 64 * 16, nc, dt, -3, 3).reshape(64, 16, nc)
            out[f"{key}_mm_y"] = ym
            rows = np.repeat(np.arange(24), 16)
            cols = np.tile(np.arange(16), 24)
            out[f"{key}_mmmc"] = ref.mm_mcmc_sampled(xm, ym, rows, cols).reshape(24, 16, nc)
    path = os.path.join(HERE, "golden_elementwise.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
