"""Host-array MCF operators: the reference's calling model (host values in,
host values out) over the library's mcf_h_* entry points.

Arrays are numpy with the component axis last; float16/float32/float64 select
B16/B32/B64.  Each call stages through the device workspace (pipelined
H2D / kernel / D2H over three streams) and blocks until the result is in host
memory.  Page-locked inputs (e.g. torch pinned tensors' numpy views) take the
direct DMA path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _check, lib

_PREC = {np.dtype(np.float16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _prec(a):
    if a.dtype not in _PREC:
        raise ValueError(f"unsupported component dtype {a.dtype}")
    return _PREC[a.dtype]


def elementwise(op: str, x=None, y=None, v=None, out=None):
    """Run elementwise operator `op` ("add_mcn", "grow_expn", ...) on host arrays."""
    ref = x if x is not None else y
    ref = np.ascontiguousarray(ref)
    prec = _prec(ref)
    x = None if x is None else np.ascontiguousarray(x, dtype=ref.dtype)
    y = None if y is None else np.ascontiguousarray(y, dtype=ref.dtype)
    if v is not None:
        v = np.ascontiguousarray(np.asarray(v, dtype=ref.dtype).reshape(-1))
    ncx = x.shape[-1] if x is not None else 0
    ncy = y.shape[-1] if y is not None else 0
    numel = ref.size // ref.shape[-1]
    if op == "approx":
        shape = ref.shape[:-1]
    elif op == "scaling_n_expanded":
        shape = ref.shape[:-1] + (ncx + 1,)
    elif op in ("add_mcn", "div_mcn", "mul_mcn", "mul_mcn_slow"):
        shape = ref.shape[:-1] + (max(ncx, ncy),)
    else:
        shape = ref.shape
    if out is None:
        out = np.empty(shape, ref.dtype)
    vn = 1 if v is None else v.size
    _check(lib().mcf_h_elementwise(op.encode(), prec, _p(x), ncx, _p(y), ncy, _p(v), vn, _p(out), numel))
    return out


def grow_expn(x, v):
    return elementwise("grow_expn", x=x, v=v)


def scaling_n(x, v, expanded=False):
    return elementwise("scaling_n_expanded" if expanded else "scaling_n", x=x, v=v)


def div_n(v, y):
    return elementwise("div_n", y=y, v=v)


def add_mcn(x, y):
    return elementwise("add_mcn", x=x, y=y)


def div_mcn(x, y):
    return elementwise("div_mcn", x=x, y=y)


def mul_mcn(x, y):
    return elementwise("mul_mcn", x=x, y=y)


def mul_mcn_slow(x, y):
    return elementwise("mul_mcn_slow", x=x, y=y)


def square_mcn(x):
    return elementwise("square_mcn", x=x)


def exp_mcn(x):
    return elementwise("exp_mcn", x=x)


def negate(x):
    return elementwise("negate", x=x)


def approx(x):
    return elementwise("approx", x=x)


def mm_mcn(x, w, strategy=0, out=None):
    """MC (m,k,nc) x working (k,n); strategy 0 = reference order (bitwise),
    2 = FAST (compensated binary64)."""
    x = np.ascontiguousarray(x)
    w = np.ascontiguousarray(w, dtype=x.dtype)
    m, k, nc = x.shape
    n = w.shape[1]
    if out is None:
        out = np.empty((m, n, nc), x.dtype)
    _check(lib().mcf_h_bmm_mcn(_prec(x), _p(x), nc, _p(w), 1, m, k, n, 0, _p(out), strategy))
    return out


def mm_mcmc(x, y, strategy=0, out=None):
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    m, k, nc = x.shape
    n = y.shape[1]
    if out is None:
        out = np.empty((m, n, nc), x.dtype)
    _check(lib().mcf_h_mm_mcmc(_prec(x), _p(x), _p(y), nc, m, k, n, _p(out), strategy))
    return out


# ---- the reference's test predicates (value checks on host arrays) -----------

_SIG = {np.dtype(np.float16): 11, np.dtype(np.float32): 24, np.dtype(np.float64): 53}
_MIN_POS = {np.dtype(np.float16): 2.0**-24, np.dtype(np.float32): 2.0**-149, np.dtype(np.float64): 2.0**-1074}


def ulp(x, dtype):
    """ulp<P>(x) (precision.hpp:200-206): the spacing of P at |x|, clamped to the
    subnormal quantum; min_pos for zero and non-finite x.  Elementwise, binary64."""
    dt = np.dtype(dtype)
    x = np.asarray(x, np.float64)
    with np.errstate(all="ignore"):
        e = np.floor(np.log2(np.abs(np.where(np.isfinite(x) & (x != 0), x, 1.0))))
        # log2 can round at the top of a binade: correct with exact comparisons
        e = np.where(np.exp2(e) > np.abs(x), e - 1, e)
        e = np.where(np.exp2(e + 1) <= np.abs(x), e + 1, e)
        sp = np.exp2(e - (_SIG[dt] - 1))
    sp = np.maximum(sp, _MIN_POS[dt])
    return np.where((x == 0) | ~np.isfinite(x), _MIN_POS[dt], sp)


def satisfies_invariants(x) -> bool:
    """satisfies_invariants<P> (mc_ops.hpp:537-554) on an MC array (..., nc):
    every component finite, zeros only as a trailing suffix, no nonzero
    component below P's subnormal quantum, and |c_i| <= ulp(c_{i-1})."""
    x = np.asarray(x)
    dt = x.dtype
    c = x.reshape(-1, x.shape[-1]).astype(np.float64)
    if not np.all(np.isfinite(c)):
        return False
    nz = c != 0
    # a zero followed by a nonzero component
    seen_zero = np.logical_or.accumulate(~nz, axis=1)
    if np.any(nz[:, 1:] & seen_zero[:, :-1]):
        return False
    if np.any(nz & (np.abs(c) < _MIN_POS[dt])):
        return False
    if c.shape[1] > 1:
        bad = nz[:, 1:] & (np.abs(c[:, 1:]) > ulp(c[:, :-1], dt))
        if np.any(bad):
            return False
    return True
