"""CPU pins of the MCF_FAST tensor-core scheme's integer arithmetic (mm_ozaki.cu).

The binary32 nc=2 MC contractions are exact integer products by Chinese
remaindering: operands rounded to pa / pb-bit integers, one int8 GEMM per
modulus, reconstruction from binary32 slice sums.  These tests need no GPU:
they read the library's own constants (mcf_fast_tc_plan / _crt_table, host
code) and replay the device arithmetic step by step in numpy (binary32 /
binary64 operations with the same roundings), checking every intermediate
against exact Python integers.
"""
import ctypes as C
import math
from fractions import Fraction

import numpy as np
import pytest

import paper_2207_08867_b200 as mcf

S = 8  # slices
SB = 12  # slice bits
MAGIC = np.float32(12582912.0)


def plan(k, ncb):
    n, pa, pb = C.c_int(), C.c_int(), C.c_int()
    r = mcf.lib().mcf_fast_tc_plan(k, ncb, C.byref(n), C.byref(pa), C.byref(pb))
    assert r == n.value
    return n.value, pa.value, pb.value


def table(n):
    mods = (C.c_int * n)()
    w = (C.c_float * (n * S))()
    mh = (C.c_float * S)()
    cq = C.c_float()
    L = C.c_int()
    assert mcf.lib().mcf_fast_tc_crt_table(n, mods, w, mh, C.byref(cq), C.byref(L)) == S
    return (list(mods), np.array(w, np.float32).reshape(n, S), np.array(mh, np.float32), np.float32(cq.value),
            L.value)


def test_plans_at_the_baseline_shapes():
    assert plan(4096, 1) == (17, 72, 48)      # config 2: 17 int8 GEMMs
    n, pa, pb = plan(16384, 2)                # config 4 MC x MC
    assert n == 20 and pa == pb == 70
    assert plan(784, 1)[0] == plan(1024, 1)[0] == 16  # MLP layers
    for k in (1, 64, 1000, 4096, 20000, 65536):
        for ncb in (1, 2):
            n, pa, pb = plan(k, ncb)
            _, _, _, _, L = table(n)
            M = math.prod(table(n)[0])
            lk = math.ceil(math.log2(k)) if k > 1 else 0
            # |C'| <= K 2^(pa-1) 2^(pb-1) <= M / 4, and the bound target
            assert (1 << lk) * 2 ** (pa + pb - 2) * 4 <= M
            assert pa >= lk + 56 and pa <= 73
            assert pb == (48 if ncb == 1 else pa)


@pytest.mark.parametrize("n", range(16, 23))
def test_crt_tables_are_exact_slices(n):
    mods, w, mh, cq, L = table(n)
    assert len(set(mods)) == n and all(math.gcd(a, b) == 1 for i, a in enumerate(mods) for b in mods[i + 1:])
    M = math.prod(mods)
    assert M.bit_length() == L
    tail = 2 ** (L - SB * S - 1)
    rec = lambda d: sum(int(v) * 2 ** (L - SB * (j + 1)) for j, v in enumerate(d))
    assert abs(rec(mh) - M) <= tail
    assert np.all(np.abs(w) <= 2048) and np.all(np.abs(mh[1:]) <= 2048) and mh[0] <= 4096
    for t, m in enumerate(mods):
        Mt = M // m
        wt = Mt * pow(Mt, -1, m) % M
        if 2 * wt > M:
            wt -= M
        assert abs(rec(w[t]) - wt) <= tail
        for s, ms in enumerate(mods):
            assert wt % ms == (1 if s == t else 0)
    assert abs(float(cq) - 2.0 ** (L - SB) / M) <= 2.0 ** (L - SB) / M * 2 ** -24


def sym(v, m):
    r = v % m
    return r - m if r > m // 2 else r


def emulate_mod_c(c, m, big):
    """mm_ozaki.cu mod_c<BIG> in numpy binary32 (all steps exact or single-rounded)."""
    c = np.asarray(c, np.int64)
    cl = ((c + 8192) & 16383) - 8192
    ch = (c - cl) >> 14
    c14 = np.float32(sym(1 << 14, m))
    inv = np.float32(1.0) / np.float32(m)
    s = (ch.astype(np.float64) * np.float64(c14) + cl).astype(np.float32)  # exact
    if big:
        q0 = (s.astype(np.float64) * np.float64(inv) + np.float64(MAGIC)).astype(np.float32) - MAGIC
        s = (s.astype(np.float64) - q0.astype(np.float64) * m).astype(np.float32)
    q = (s.astype(np.float64) * np.float64(inv) + np.float64(MAGIC)).astype(np.float32) - MAGIC
    return (s.astype(np.float64) - q.astype(np.float64) * m).astype(np.float32)


@pytest.mark.parametrize("k,big", [(4096, False), (16384, False), (65536, True)])
def test_gemm_residue_reduction_is_exact(k, big):
    rng = np.random.default_rng(k)
    lim = k * 2 ** 14
    c = np.concatenate([rng.integers(-lim, lim + 1, 200000), [lim, -lim, 0, 1, -1, 8191, -8192, 8192]])
    mods, *_ = table(22)
    for m in mods[1:]:
        r = emulate_mod_c(c, m, big)
        want = np.array([sym(int(v), m) for v in c[:2000]] + [sym(int(v), m) for v in c[-8:]])
        got = np.concatenate([r[:2000], r[-8:]])
        assert np.array_equal(got.astype(np.int64), want), m
        assert np.all(np.abs(r) <= (m - 1) // 2)
        # the rest by congruence and range
        assert np.all(((c - r.astype(np.int64)) % m) == 0)


def emulate_reconstruct(res, n):
    """k_crt's slice sums, quotient and Horner pass for one output."""
    mods, w, mh, cq, L = table(n)
    T = np.zeros(S, np.float32)
    for t in range(n):
        T = (T.astype(np.float64) + np.float64(res[t]) * w[t].astype(np.float64)).astype(np.float32)  # exact
    u0 = np.float32(np.float64(T[1]) * 2.0 ** -SB + np.float64(T[0]))
    q = np.float32(np.float64(u0) * np.float64(cq) + np.float64(MAGIC)) - MAGIC
    D = (T.astype(np.float64) - np.float64(q) * mh.astype(np.float64)).astype(np.float32)
    assert np.all(D.astype(np.float64) == T.astype(np.float64) - np.float64(q) * mh)  # exact
    y = np.float64(D[0])
    for j in range(1, S):
        y = np.float64(y * 4096.0 + np.float64(D[j]))  # fma: y * 4096 is exact
    return float(y), L


@pytest.mark.parametrize("n", [16, 17, 20, 22])
def test_reconstruction_recovers_the_integer(n):
    rng = np.random.default_rng(n)
    mods, _, _, _, L = table(n)
    M = math.prod(mods)
    vals = [int(rng.integers(-2**62, 2**62)) * (M // 4 >> 62) // 3 for _ in range(300)]
    vals += [M // 4, -(M // 4), 0, 1, -1, 2 ** 70 + 12345, -(2 ** 100) - 7]
    for v in vals:
        res = [sym(v, m) for m in mods]
        y, L = emulate_reconstruct(res, n)
        got = Fraction(y) * 2 ** (L - SB * S)
        err = abs(got - v)
        # slice tail (<= 2^12 units of 2^(L-96)) + binary64 Horner rounding
        assert err <= 2 ** (L - SB * S + 12) + abs(Fraction(v)) * 2 ** -50, (v, float(err))


def emulate_limbs2(x, s):
    """mm_ozaki.cu limbs2() for one binary32 value: scale by 2^s as two exact
    binary32 products, then six magic-constant roundings from the top (the
    FFMA's single rounding replayed exactly with Fractions)."""
    s1 = min(s, 127)
    r = np.float32(np.float32(x) * np.float32(2.0 ** s1))
    r = np.float32(r * np.float32(2.0 ** (s - s1)))
    xs = r
    limbs = [0] * 6
    for j in range(5, -1, -1):
        t = round(Fraction(float(r)) / 2 ** (12 * j))  # RN-even of the exact quotient (magic rounding)
        rem = Fraction(float(r)) - t * 2 ** (12 * j)
        assert rem == Fraction(float(np.float32(float(rem))))  # the remainder is exact in binary32
        r = np.float32(float(rem))
        limbs[j] = t
    return limbs, r, xs


def test_operand_residues_are_exact():
    """A' = round(c0 2^s) + round(c1 2^s) cut into six balanced 12-bit limbs
    per component by binary32 magic-constant rounding; the limb sums' residues,
    reduced by one rounded quotient, equal the exact symmetric residues; the
    error is <= 1/2 per rounded component."""
    rng = np.random.default_rng(5)
    mods, *_ = table(22)
    for p, e in ((72, 1), (73, -3), (48, 0), (67, 5), (72, -140), (48, 100)):
        v = rng.uniform(-1, 1, 1500) * np.exp2(rng.uniform(-60, 0, 1500)) * 2.0 ** (e - 1)
        c0 = v.astype(np.float32)
        c1 = (v - c0.astype(np.float64)).astype(np.float32)
        for a, b in zip(c0, c1):
            la, ra, _ = emulate_limbs2(a, p - e)
            lb, rb, _ = emulate_limbs2(b, p - e)
            limbs = [x + y for x, y in zip(la, lb)]
            X = sum(l * 2 ** (12 * j) for j, l in enumerate(limbs))
            exact = (Fraction(float(a)) + Fraction(float(b))) * Fraction(2) ** (p - e)
            assert abs(X - exact) <= Fraction(1) and abs(X - exact) == abs(Fraction(float(ra)) + Fraction(float(rb)))
            assert abs(limbs[5]) <= 2 ** 13 and all(abs(l) <= 2 ** 12 for l in limbs[:5])
            for m in mods[1:]:
                cw = [np.float32(sym(2 ** (12 * j), m)) for j in range(6)]
                sacc = Fraction(0)
                for l, c in zip(limbs, cw):
                    sacc += l * int(c)
                assert abs(sacc) < 2 ** 22  # exact binary32 sums, s + kMagic exact
                inv = np.float32(1.0) / np.float32(m)
                q = round(sacc * Fraction(float(inv)))  # FFMA(s, RN(1/m), kMagic): one rounding to an integer
                r = int(sacc - q * m)
                assert r == sym(X, m), (m, X)
            assert (limbs[0] & 0xFF) == X % 256
