"""Seeded synthetic inputs for the BASELINE.json configurations.

Draws come from the reference's own generator mappings (mcf::Rng,
rng.hpp:13-65: std::mt19937_64, 53-bit uniform) through mcf_rng_uniform, and
binary64 values are split into components by the reference's greedy
round-and-residual rule (detail::expansion_of_double, mc_ops.hpp:286-297).
Seeds follow SURVEY 8d: Rng(1000 * config + operand_index).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import lib


def uniform(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().mcf_rng_uniform(seed, n, out.ctypes.data_as(C.c_void_p))
    return out


def normal(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().mcf_rng_normal(seed, n, out.ctypes.data_as(C.c_void_p))
    return out


def below(seed: int, bound: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().mcf_rng_below(seed, bound, n, out.ctypes.data_as(C.c_void_p))
    return out


def split(v: np.ndarray, nc: int, dtype=np.float32) -> np.ndarray:
    """expansion_of_double: out[i] = round_P(rest); rest -= out[i]."""
    v = np.asarray(v, np.float64)
    out = np.zeros(v.shape + (nc,), dtype)
    rest = v.copy()
    with np.errstate(all="ignore"):
        for i in range(nc):
            c = rest.astype(dtype)
            out[..., i] = c
            rest = np.where(np.isfinite(c), rest - c.astype(np.float64), 0.0)
    return out


def config0_values(seed: int, n: int) -> np.ndarray:
    """U(-1,1) * 2^U(-8,8) in binary64 (two draws per value, interleaved)."""
    u = uniform(seed, 2 * n)
    return (-1.0 + 2.0 * u[0::2]) * np.exp2(-8.0 + 16.0 * u[1::2])


def config0(n: int = 1 << 24, nc: int = 2, dtype=np.float32):
    """BASELINE config 0 operands: MC x, y (divisor-safe yd), exp input xe, tensor v."""
    x = split(config0_values(1000, n), nc, dtype)
    yv = config0_values(1001, n)
    y = split(yv, nc, dtype)
    yd = split(yv + np.sign(yv) * 0.5, nc, dtype)
    v = config0_values(1002, n).astype(dtype)
    xe = split(np.clip(config0_values(1003, n), -10.0, 10.0), nc, dtype)
    return x, y, yd, v, xe


def config2(m: int = 4096, k: int = 4096, n: int = 4096):
    """BASELINE config 2: A (m,k) nc=2 split from fp64 U[-1,1]; B (k,n) fp32 U[-1,1]."""
    a = split(-1.0 + 2.0 * uniform(2000, m * k), 2, np.float32).reshape(m, k, 2)
    b = (-1.0 + 2.0 * uniform(2001, k * n)).astype(np.float32).reshape(k, n)
    return a, b
