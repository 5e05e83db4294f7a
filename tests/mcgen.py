"""Seeded input generators and bitwise comparison helpers for the tests.

MC tensors are numpy arrays with the component axis last.  Values are built
the way the reference builds them (greedy round-and-residual split of a
binary64 value, ``detail::expansion_of_double``, mc_ops.hpp:286-297), plus
deliberately awkward cases: zeros, subnormals, equal magnitudes, unsorted and
overlapping components, and non-finite values.
"""
from __future__ import annotations

import numpy as np

DT = {16: np.float16, 32: np.float32, 64: np.float64}
UINT = {np.dtype(np.float16): np.uint16, np.dtype(np.float32): np.uint32, np.dtype(np.float64): np.uint64}


def split(v: np.ndarray, nc: int, dtype) -> np.ndarray:
    """expansion_of_double: out[i] = round_P(rem); rem -= out[i] (exact)."""
    v = np.asarray(v, np.float64)
    out = np.zeros(v.shape + (nc,), dtype)
    rem = v.copy()
    with np.errstate(all="ignore"):
        for i in range(nc):
            c = rem.astype(dtype)
            out[..., i] = c
            rem = np.where(np.isfinite(c), rem - c.astype(np.float64), 0.0)
    return out


def split_ld(hi: np.ndarray, lo: np.ndarray, nc: int, dtype) -> np.ndarray:
    """Split hi+lo (two float64 with |lo| <= ulp(hi)/2) greedily into nc comps of dtype."""
    out = np.zeros(hi.shape + (nc,), dtype)
    h, l = hi.astype(np.float64).copy(), lo.astype(np.float64).copy()
    with np.errstate(all="ignore"):
        for i in range(nc):
            c = (h + l).astype(dtype)  # nearly greedy; residual stays exact below
            out[..., i] = c
            cd = c.astype(np.float64)
            # (h + l) - c computed exactly with two-sum in float64
            s = h - cd
            t = s + l
            e = (s - t) + l
            h, l = t, e
    return out


def config_values(rng: np.random.Generator, n: int, lo_exp=-8, hi_exp=8) -> np.ndarray:
    """v = U(-1,1) * 2^U(lo_exp, hi_exp) in binary64 (BASELINE config 0)."""
    return rng.uniform(-1.0, 1.0, n) * np.exp2(rng.uniform(lo_exp, hi_exp, n))


def random_mc(rng, n, nc, dtype, lo_exp=-8, hi_exp=8, extra_bits=True):
    """Valid (ordered, nonoverlapping) MC values with about nc*p bits."""
    if extra_bits:
        hi = config_values(rng, n, lo_exp, hi_exp)
        lo = hi * rng.uniform(-1, 1, n) * 2.0**-53
        return split_ld(hi, lo, nc, dtype)
    return split(config_values(rng, n, lo_exp, hi_exp), nc, dtype)


def nasty_mc(rng, n, nc, dtype, allow_nonfinite=True):
    """Arbitrary component soup: unordered, overlapping, zeros, ties, subnormals."""
    dt = np.dtype(dtype)
    finfo = np.finfo(dt)
    kinds = rng.integers(0, 9, size=(n, nc))
    base = rng.uniform(-1, 1, (n, nc)) * np.exp2(rng.integers(-6, 7, size=(n, nc)))
    out = base.astype(dt)
    tiny = (rng.integers(1, 8, size=(n, nc)) * float(finfo.smallest_subnormal)).astype(dt)
    out = np.where(kinds == 0, dt.type(0), out)
    out = np.where(kinds == 1, tiny, out)
    lead = np.repeat(out[:, :1], nc, axis=1)
    out = np.where(kinds == 2, -lead, out)  # equal magnitude, opposite sign
    out = np.where(kinds == 3, lead, out)  # exact tie
    out = np.where(kinds == 4, (lead.astype(np.float64) * 2.0**-int(finfo.nmant + 1)).astype(dt), out)
    if allow_nonfinite:
        special = rng.random((n, nc)) < 0.002
        vals = np.array([np.inf, -np.inf, np.nan], np.float64).astype(dt)
        out = np.where(special, vals[rng.integers(0, 3, size=(n, nc))], out)
    out = np.where(rng.random((n, nc)) < 0.02, dt.type(-0.0), out)
    return out


def same_bits(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Elementwise bit equality, with every NaN equal to every NaN."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    u = UINT[a.dtype]
    eq = a.view(u) == b.view(u)
    return eq | (np.isnan(a) & np.isnan(b))


def assert_bits(got, want, what="", max_report=5):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    ok = same_bits(got, want)
    if not ok.all():
        bad = np.argwhere(~ok)
        rows = sorted({tuple(i[:-1]) if got.ndim > 1 else tuple(i) for i in bad})[:max_report]
        msg = [f"{what}: {int((~ok).sum())} mismatching components"]
        for r in rows:
            msg.append(f"  at {r}: got {got[r]!r} want {want[r]!r}")
        raise AssertionError("\n".join(msg))
