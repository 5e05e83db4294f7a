"""CPU oracle for the MCF hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker.  The product path (``paper_2207_08867_b200``) never touches it.

Two back ends share one C interface (``oracle/mcf_oracle.h``):

* ``Oracle("port")`` -- ``oracle/libmcf_oracle.so``: plain-C restatement of the
  reference algorithms (``oracle/mcf_oracle_body.inc`` cites the reference
  file:line of every function).
* ``Oracle("ref")``  -- ``oracle/_ref/libmcf_ref.so``: the reference's own
  header-only C++ (``/root/reference/proj/include/mcfloat``) compiled
  unmodified behind ``oracle/ref_shim.cpp``.

Arrays are numpy: MC tensors have shape ``(..., nc)`` with the component axis
last; B16/B32/B64 map to float16/float32/float64 (IEEE bit patterns, exactly
the device storage of ``include/mcf_gpu.h``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libmcf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmcf_ref.so")

B16, B32, B64 = 0, 1, 2
DTYPES = {B16: np.float16, B32: np.float32, B64: np.float64}
PREC_OF = {np.dtype(np.float16): B16, np.dtype(np.float32): B32, np.dtype(np.float64): B64}
EXP_LIBM, EXP_CR = 0, 1
SEQUENTIAL, PAIRWISE_TREE = 0, 1

_p = C.c_void_p
_i64 = C.c_int64
_int = C.c_int


def build(force: bool = False) -> None:
    """Build the port (and, when /root/reference exists, the reference shim
    and the C++ drop-in check); make skips whatever is up to date."""
    if force or not os.path.exists(PORT_SO) or os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_p)


def prec_of(a: np.ndarray) -> int:
    return PREC_OF[a.dtype]


class OracleError(RuntimeError):
    pass


class Oracle:
    """ctypes view of one oracle back end ("port" or "ref")."""

    def __init__(self, which: str = "port"):
        self.which = which
        path, self.pfx = (PORT_SO, "mcfo_") if which == "port" else (REF_SO, "mcfref_")
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise OracleError(f"oracle back end {which!r} not built: {path}")
        self.lib = C.CDLL(path)
        self._sig()

    def _f(self, name):
        return getattr(self.lib, self.pfx + name)

    def _sig(self):
        for name, args in {
            "two_sum": [_int, _p, _p, _p, _p, _i64],
            "two_prod": [_int, _p, _p, _p, _p, _i64, _int],
            "renormalize": [_int, _p, _int, _p, _int, _i64],
            "simple_renorm": [_int, _p, _int, _p, _int, _i64],
            "approx": [_int, _p, _int, _p, _i64],
            "negate": [_int, _p, _int, _p, _i64],
            "grow_expn": [_int, _p, _int, _p, _i64, _p, _i64],
            "scaling_n": [_int, _p, _int, _p, _i64, _int, _p, _i64],
            "div_n": [_int, _p, _i64, _p, _int, _p, _i64],
            "add_mcn": [_int, _p, _int, _p, _int, _p, _i64],
            "div_mcn": [_int, _p, _int, _p, _int, _p, _i64],
            "mul_mcn": [_int, _p, _int, _p, _int, _p, _i64],
            "mul_mcn_slow": [_int, _p, _int, _p, _int, _p, _i64],
            "square_mcn": [_int, _p, _int, _p, _i64],
            "exp_mcn": [_int, _p, _int, _p, _i64, _int],
            "bmm_mcn": [_int, _p, _int, _p, _i64, _i64, _i64, _i64, _int, _p, _int, _int],
            "mm_mcn_sampled": [_int, _p, _int, _p, _i64, _i64, _i64, _p, _p, _i64, _p],
            "dot_mcmc": [_int, _p, _p, _int, _i64, _i64, _p],
            "mm_mcmc_sampled": [_int, _p, _p, _int, _i64, _i64, _i64, _p, _p, _i64, _p],
            "matmul2d": [_int, _p, _p, _i64, _i64, _i64, _p],
            "mc_relu": [_int, _p, _int, _p, _i64],
            "mc_softmax": [_int, _p, _int, _i64, _i64, _i64, _p, _int],
            "halfspace_arg": [_int, _p, _int, _i64, _i64, _p, _p, _i64, _p],
        }.items():
            f = self._f(name)
            f.argtypes = args
            f.restype = _int
        if self.which == "port":
            L = self.lib
            L.mcfo_cr_exp.argtypes = [C.c_double, C.POINTER(C.c_int)]
            L.mcfo_cr_exp.restype = C.c_double
            L.mcfo_libm_exp.argtypes = [C.c_double]
            L.mcfo_libm_exp.restype = C.c_double
            L.mcfo_round_b16.argtypes = [C.c_double]
            L.mcfo_round_b16.restype = C.c_double
            for n in ("mcfo_relerr_mm_mct",):
                getattr(L, n).argtypes = [_int, _p, _int, _p, _i64, _i64, _i64, _p, _p, _i64, _p, _int, _p]
                getattr(L, n).restype = _int
            L.mcfo_relerr_mm_mcmc.argtypes = [_int, _p, _p, _int, _i64, _i64, _i64, _p, _p, _i64, _p, _int, _p]
            L.mcfo_relerr_mm_mcmc.restype = _int
        else:
            L = self.lib
            L.mcfref_time_elementwise.argtypes = [C.c_char_p, _int, _p, _int, _p, _p, _i64, _int, _int, _p]
            L.mcfref_time_elementwise.restype = C.c_double
            L.mcfref_time_mm_rows.argtypes = [_int, _p, _int, _p, _i64, _i64, _i64, _int, _p]
            L.mcfref_time_mm_rows.restype = C.c_double
            L.mcfref_time_dot_mcmc.argtypes = [_int, _p, _p, _int, _i64, _i64, _int, _p]
            L.mcfref_time_dot_mcmc.restype = C.c_double
            L.mcfref_mlp_train.argtypes = [_p, _int, _int, _p, _p, _p, _i64, _int, C.c_double, _p, _p]
            L.mcfref_mlp_train.restype = _int
            L.mcfref_rng_uniform.argtypes = [C.c_uint64, _i64, _p]
            L.mcfref_rng_uniform.restype = None
            L.mcfref_rng_normal.argtypes = [C.c_uint64, _i64, _p]
            L.mcfref_rng_normal.restype = None
            L.mcfref_rng_below.argtypes = [C.c_uint64, C.c_uint64, _i64, _p]
            L.mcfref_rng_below.restype = None

    # ---- the reference's own Rng (rng.hpp:13-65), ref back end only ----------
    def rng_uniform(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.mcfref_rng_uniform(seed, n, _ptr(out))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.mcfref_rng_normal(seed, n, _ptr(out))
        return out

    def rng_below(self, seed, bound, n):
        out = np.empty(n, np.uint64)
        self.lib.mcfref_rng_below(seed, bound, n, _ptr(out))
        return out

    @staticmethod
    def _check(rc, what):
        if rc != 0:
            raise OracleError(f"{what}: oracle returned {rc}")

    # ---- EFT arrays ---------------------------------------------------------
    def two_sum(self, a, b):
        a = np.ascontiguousarray(a); b = np.ascontiguousarray(b, dtype=a.dtype)
        s = np.empty_like(a); e = np.empty_like(a)
        self._check(self._f("two_sum")(prec_of(a), _ptr(a), _ptr(b), _ptr(s), _ptr(e), a.size), "two_sum")
        return s, e

    def two_prod(self, a, b, use_fma=True):
        a = np.ascontiguousarray(a); b = np.ascontiguousarray(b, dtype=a.dtype)
        p = np.empty_like(a); e = np.empty_like(a)
        self._check(self._f("two_prod")(prec_of(a), _ptr(a), _ptr(b), _ptr(p), _ptr(e), a.size, int(use_fma)), "two_prod")
        return p, e

    # ---- MC ops ------------------------------------------------------------------
    def _renorm(self, name, h, r_nc):
        h = np.ascontiguousarray(h); nc = h.shape[-1]
        out = np.empty(h.shape[:-1] + (r_nc,), h.dtype)
        self._check(self._f(name)(prec_of(h), _ptr(h), nc, _ptr(out), r_nc, h.size // nc), name)
        return out

    def renormalize(self, h, r_nc):
        return self._renorm("renormalize", h, r_nc)

    def simple_renorm(self, h, r_nc):
        return self._renorm("simple_renorm", h, r_nc)

    def approx(self, x):
        x = np.ascontiguousarray(x); nc = x.shape[-1]
        out = np.empty(x.shape[:-1], x.dtype)
        self._check(self._f("approx")(prec_of(x), _ptr(x), nc, _ptr(out), x.size // nc), "approx")
        return out

    def negate(self, x):
        x = np.ascontiguousarray(x); nc = x.shape[-1]
        out = np.empty_like(x)
        self._check(self._f("negate")(prec_of(x), _ptr(x), nc, _ptr(out), x.size // nc), "negate")
        return out

    def grow_expn(self, x, v):
        x = np.ascontiguousarray(x); v = np.ascontiguousarray(v, dtype=x.dtype).reshape(-1)
        nc = x.shape[-1]; out = np.empty_like(x)
        self._check(self._f("grow_expn")(prec_of(x), _ptr(x), nc, _ptr(v), v.size, _ptr(out), x.size // nc), "grow_expn")
        return out

    def scaling_n(self, x, v, expanded=False):
        x = np.ascontiguousarray(x); v = np.ascontiguousarray(v, dtype=x.dtype).reshape(-1)
        nc = x.shape[-1]; onc = nc + 1 if expanded else nc
        out = np.empty(x.shape[:-1] + (onc,), x.dtype)
        self._check(self._f("scaling_n")(prec_of(x), _ptr(x), nc, _ptr(v), v.size, int(expanded), _ptr(out), x.size // nc), "scaling_n")
        return out

    def div_n(self, v, y):
        y = np.ascontiguousarray(y); v = np.ascontiguousarray(v, dtype=y.dtype).reshape(-1)
        nc = y.shape[-1]; out = np.empty_like(y)
        self._check(self._f("div_n")(prec_of(y), _ptr(v), v.size, _ptr(y), nc, _ptr(out), y.size // nc), "div_n")
        return out

    def _binary(self, name, x, y):
        x = np.ascontiguousarray(x); y = np.ascontiguousarray(y, dtype=x.dtype)
        ncx, ncy = x.shape[-1], y.shape[-1]
        out = np.empty(x.shape[:-1] + (max(ncx, ncy),), x.dtype)
        self._check(self._f(name)(prec_of(x), _ptr(x), ncx, _ptr(y), ncy, _ptr(out), x.size // ncx), name)
        return out

    def add_mcn(self, x, y):
        return self._binary("add_mcn", x, y)

    def div_mcn(self, x, y):
        return self._binary("div_mcn", x, y)

    def mul_mcn(self, x, y):
        return self._binary("mul_mcn", x, y)

    def mul_mcn_slow(self, x, y):
        return self._binary("mul_mcn_slow", x, y)

    def square_mcn(self, x):
        x = np.ascontiguousarray(x); nc = x.shape[-1]; out = np.empty_like(x)
        self._check(self._f("square_mcn")(prec_of(x), _ptr(x), nc, _ptr(out), x.size // nc), "square_mcn")
        return out

    def exp_mcn(self, x, exp_mode=EXP_LIBM):
        x = np.ascontiguousarray(x); nc = x.shape[-1]; out = np.empty_like(x)
        self._check(self._f("exp_mcn")(prec_of(x), _ptr(x), nc, _ptr(out), x.size // nc, exp_mode), "exp_mcn")
        return out

    # ---- contractions ----------------------------------------------------------
    def bmm_mcn(self, x, w, strategy=SEQUENTIAL, leaf_arity=1):
        """x (B,M,K,nc) or (M,K,nc); w (B,K,N) batched or (K,N) broadcast."""
        x = np.ascontiguousarray(x); w = np.ascontiguousarray(w, dtype=x.dtype)
        squeeze = x.ndim == 3
        if squeeze:
            x = x[None]
        B, M, K, nc = x.shape
        w_batched = w.ndim == 3
        N = w.shape[-1]
        out = np.empty((B, M, N, nc), x.dtype)
        self._check(self._f("bmm_mcn")(prec_of(x), _ptr(x), nc, _ptr(w), B, M, K, N, int(w_batched), _ptr(out), strategy, leaf_arity), "bmm_mcn")
        return out[0] if squeeze else out

    def mm_mcn(self, x, w, strategy=SEQUENTIAL, leaf_arity=1):
        return self.bmm_mcn(x, w, strategy, leaf_arity)

    def mv_mcn(self, x, v, strategy=SEQUENTIAL, leaf_arity=1):
        return self.bmm_mcn(x, np.asarray(v).reshape(-1, 1), strategy, leaf_arity)[:, 0, :]

    def dot_mcn(self, x, v, strategy=SEQUENTIAL, leaf_arity=1):
        return self.mv_mcn(x[None], v, strategy, leaf_arity)[0]

    def mm_mcn_sampled(self, x, w, rows, cols):
        x = np.ascontiguousarray(x); w = np.ascontiguousarray(w, dtype=x.dtype)
        M, K, nc = x.shape; N = w.shape[1]
        rows = np.ascontiguousarray(rows, np.int64); cols = np.ascontiguousarray(cols, np.int64)
        out = np.empty((rows.size, nc), x.dtype)
        self._check(self._f("mm_mcn_sampled")(prec_of(x), _ptr(x), nc, _ptr(w), M, K, N, _ptr(rows), _ptr(cols), rows.size, _ptr(out)), "mm_mcn_sampled")
        return out

    def dot_mcmc(self, x, y):
        """x, y (B, K, nc): B independent MC x MC dots (recipe B)."""
        x = np.ascontiguousarray(x); y = np.ascontiguousarray(y, dtype=x.dtype)
        B, K, nc = x.shape
        out = np.empty((B, nc), x.dtype)
        self._check(self._f("dot_mcmc")(prec_of(x), _ptr(x), _ptr(y), nc, B, K, _ptr(out)), "dot_mcmc")
        return out

    def mm_mcmc_sampled(self, x, y, rows, cols):
        x = np.ascontiguousarray(x); y = np.ascontiguousarray(y, dtype=x.dtype)
        M, K, nc = x.shape; N = y.shape[1]
        rows = np.ascontiguousarray(rows, np.int64); cols = np.ascontiguousarray(cols, np.int64)
        out = np.empty((rows.size, nc), x.dtype)
        self._check(self._f("mm_mcmc_sampled")(prec_of(x), _ptr(x), _ptr(y), nc, M, K, N, _ptr(rows), _ptr(cols), rows.size, _ptr(out)), "mm_mcmc_sampled")
        return out

    def matmul2d(self, a, b):
        a = np.ascontiguousarray(a); b = np.ascontiguousarray(b, dtype=a.dtype)
        M, K = a.shape; N = b.shape[1]
        out = np.empty((M, N), a.dtype)
        self._check(self._f("matmul2d")(prec_of(a), _ptr(a), _ptr(b), M, K, N, _ptr(out)), "matmul2d")
        return out

    # ---- MC activations (autodiff.hpp:340-413) ------------------------------------
    def mc_relu(self, x):
        x = np.ascontiguousarray(x); nc = x.shape[-1]; out = np.empty_like(x)
        self._check(self._f("mc_relu")(prec_of(x), _ptr(x), nc, _ptr(out), x.size // nc), "mc_relu")
        return out

    def mc_softmax(self, x, axis=-1, exp_mode=EXP_LIBM):
        """x: (n, nc) or (rows, cols, nc); softmax over `axis` of the value shape."""
        x = np.ascontiguousarray(x); nc = x.shape[-1]; shp = x.shape[:-1]
        if len(shp) == 1:
            outer, n, inner = 1, shp[0], 1
        else:
            ax = axis % 2
            outer, n, inner = (shp[0], shp[1], 1) if ax == 1 else (1, shp[0], shp[1])
        out = np.empty_like(x)
        self._check(self._f("mc_softmax")(prec_of(x), _ptr(x), nc, outer, n, inner, _ptr(out), exp_mode), "mc_softmax")
        return out

    def halfspace_arg(self, table, u, v):
        """table (n, dim, nc); u, v pair indices -> float64 arcosh arguments."""
        table = np.ascontiguousarray(table); n, dim, nc = table.shape
        u = np.ascontiguousarray(u, np.int64); v = np.ascontiguousarray(v, np.int64)
        out = np.empty(u.size, np.float64)
        self._check(self._f("halfspace_arg")(prec_of(table), _ptr(table), nc, n, dim, _ptr(u), _ptr(v), u.size,
                                             _ptr(out)), "halfspace_arg")
        return out

    # ---- port-only helpers -------------------------------------------------------
    def cr_exp(self, x: float):
        amb = C.c_int(0)
        y = self.lib.mcfo_cr_exp(float(x), C.byref(amb))
        return y, bool(amb.value)

    def libm_exp(self, x: float) -> float:
        return self.lib.mcfo_libm_exp(float(x))

    def round_b16(self, x: float) -> float:
        return self.lib.mcfo_round_b16(float(x))

    def relerr_mm_mct(self, x, w, rows, cols, cand):
        x = np.ascontiguousarray(x); w = np.ascontiguousarray(w, dtype=x.dtype)
        cand = np.ascontiguousarray(cand, dtype=x.dtype)
        M, K, nc = x.shape; N = w.shape[1]
        rows = np.ascontiguousarray(rows, np.int64); cols = np.ascontiguousarray(cols, np.int64)
        out = np.empty(rows.size, np.float64)
        self._check(self.lib.mcfo_relerr_mm_mct(prec_of(x), _ptr(x), nc, _ptr(w), M, K, N, _ptr(rows), _ptr(cols), rows.size, _ptr(cand), cand.shape[-1], _ptr(out)), "relerr")
        return out

    def relerr_mm_mcmc(self, x, y, rows, cols, cand):
        x = np.ascontiguousarray(x); y = np.ascontiguousarray(y, dtype=x.dtype)
        cand = np.ascontiguousarray(cand, dtype=x.dtype)
        M, K, nc = x.shape; N = y.shape[1]
        rows = np.ascontiguousarray(rows, np.int64); cols = np.ascontiguousarray(cols, np.int64)
        out = np.empty(rows.size, np.float64)
        self._check(self.lib.mcfo_relerr_mm_mcmc(prec_of(x), _ptr(x), _ptr(y), nc, M, K, N, _ptr(rows), _ptr(cols), rows.size, _ptr(cand), cand.shape[-1], _ptr(out)), "relerr")
        return out

    # ---- ref-only timing -----------------------------------------------------
    def time_elementwise(self, op, x=None, y=None, v=None, threads=1, reps=1):
        ref = next(a for a in (x, y, v) if a is not None)
        prec = prec_of(ref)
        nc = (x if x is not None else y).shape[-1]
        numel = (x if x is not None else y).size // nc
        onc = nc
        out = np.empty((numel, onc), ref.dtype)
        t = self.lib.mcfref_time_elementwise(op.encode(), prec, _ptr(x), nc, _ptr(y), _ptr(v), numel, threads, reps, _ptr(out))
        if t < 0:
            raise OracleError(f"time_elementwise({op}) failed")
        return t, out

    def time_mm_rows(self, x, w, rows, threads=1):
        M, K, nc = x.shape; N = w.shape[1]
        out = np.empty((rows, N, nc), x.dtype)
        t = self.lib.mcfref_time_mm_rows(prec_of(x), _ptr(np.ascontiguousarray(x)), nc, _ptr(np.ascontiguousarray(w)), rows, K, N, threads, _ptr(out))
        if t < 0:
            raise OracleError("time_mm_rows failed")
        return t, out

    def time_dot_mcmc(self, x, y, threads=1):
        B, K, nc = x.shape
        out = np.empty((B, nc), x.dtype)
        t = self.lib.mcfref_time_dot_mcmc(prec_of(x), _ptr(np.ascontiguousarray(x)), _ptr(np.ascontiguousarray(y)), nc, B, K, threads, _ptr(out))
        if t < 0:
            raise OracleError("time_dot_mcmc failed")
        return t, out


def mlp_train_reference(dims, nc, params, X, labels, steps, lr):
    """The reference's own MC-MLP training loop (oracle/_ref).  params: list of
    (W (out, in, nc), b (out, nc)) float32 per layer; X (n, dims[0]) float32;
    returns (losses[steps], list of final (W, b))."""
    ref = Oracle("ref")
    flat = np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in params]).astype(np.float32)
    dims_c = np.ascontiguousarray(dims, np.int32)
    X = np.ascontiguousarray(X, np.float32)
    lab = np.ascontiguousarray(labels, np.int32)
    losses = np.empty(steps, np.float32)
    out = np.empty_like(flat)
    rc = ref.lib.mcfref_mlp_train(_ptr(dims_c), len(dims) - 1, nc, _ptr(flat), _ptr(X), _ptr(lab), X.shape[0],
                                  steps, float(lr), _ptr(losses), _ptr(out))
    if rc != 0:
        raise OracleError("mcfref_mlp_train failed")
    res, off = [], 0
    for w, b in params:
        W = out[off:off + w.size].reshape(w.shape)
        off += w.size
        B = out[off:off + b.size].reshape(b.shape)
        off += b.size
        res.append((W, B))
    return losses, res


def ref_available() -> bool:
    return os.path.exists(REF_SO)
