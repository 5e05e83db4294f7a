"""B200-native MCF (multi-component float) operator layer -- Python host side.

The compute lives in ``libmcf_b200.so`` (hand-written sm_100a CUDA behind the
C-ABI of ``include/mcf_gpu.h``).  This module binds that ABI with ctypes and
mirrors the reference's operator API (``mcf::`` in
``/root/reference/proj/include/mcfloat``): same operator names, same argument
meaning, value semantics (every call returns a new tensor), and the same error
behaviour -- ``ValueError`` where the reference throws ``std::invalid_argument``
and :class:`UnsupportedOperation` where it throws ``mcf::unsupported_operation``.

Two calling models:

* device tensors (``torch.Tensor`` on CUDA): MC tensors have the component
  axis last, ``(..., nc)``; B16/B32/B64 = float16/float32/float64.  Calls are
  asynchronous on the current torch stream.
* host arrays (``numpy``): ``mcf.host.<op>`` -- the reference's own calling
  model -- stage through the library's device workspace and block.

There is no CPU fallback: if the library or a CUDA device is missing, every
operator raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCF_LIB") or os.path.join(_PKG, "libmcf_b200.so")  # MCF_LIB: an alternative build (tuning probes)

B16, B32, B64 = 0, 1, 2
SEQUENTIAL, PAIRWISE_TREE, FAST, FAST_FP64 = 0, 1, 2, 3


class UnsupportedOperation(NotImplementedError):
    """mcf::unsupported_operation (linalg.hpp:30-32)."""


class MCFError(RuntimeError):
    pass


_lib = None
_p, _i64, _int = C.c_void_p, C.c_int64, C.c_int

_SIGS = {
    "mcf_two_sum": [_int, _p, _p, _p, _p, _i64, _p],
    "mcf_two_prod": [_int, _p, _p, _p, _p, _i64, _p],
    "mcf_renormalize": [_int, _p, _int, _p, _int, _i64, _p],
    "mcf_simple_renorm": [_int, _p, _int, _p, _int, _i64, _p],
    "mcf_approx": [_int, _p, _int, _p, _i64, _p],
    "mcf_negate": [_int, _p, _int, _p, _i64, _p],
    "mcf_grow_expn": [_int, _p, _int, _p, _i64, _p, _i64, _p],
    "mcf_scaling_n": [_int, _p, _int, _p, _i64, _int, _p, _i64, _p],
    "mcf_div_n": [_int, _p, _i64, _p, _int, _p, _i64, _p],
    "mcf_add_mcn": [_int, _p, _int, _p, _int, _p, _i64, _p],
    "mcf_div_mcn": [_int, _p, _int, _p, _int, _p, _i64, _p],
    "mcf_mul_mcn": [_int, _p, _int, _p, _int, _p, _i64, _p],
    "mcf_mul_mcn_slow": [_int, _p, _int, _p, _int, _p, _i64, _p],
    "mcf_square_mcn": [_int, _p, _int, _p, _i64, _p],
    "mcf_exp_mcn": [_int, _p, _int, _p, _i64, _p],
    "mcf_bmm_mcn": [_int, _p, _int, _p, _i64, _i64, _i64, _i64, _int, _p, _int, _int, _p],
    "mcf_mm_mcmc": [_int, _p, _p, _int, _i64, _i64, _i64, _p, _int, _p],
    "mcf_dot_mcmc": [_int, _p, _p, _int, _i64, _i64, _p, _int, _p],
    "mcf_h_elementwise": [C.c_char_p, _int, _p, _int, _p, _int, _p, _i64, _p, _i64],
    "mcf_h_bmm_mcn": [_int, _p, _int, _p, _i64, _i64, _i64, _i64, _int, _p, _int],
    "mcf_h_mm_mcmc": [_int, _p, _p, _int, _i64, _i64, _i64, _p, _int],
    "mcf_fast_ops_per_mad": [_int, _int, _int],
    "mcf_fast_tc_digits": [],
    "mcf_fast_tc_gemm_equivalents": [_int, _i64],
    "mcf_fast_mm_phases": [_p, _p, _i64, _i64, _i64, _p, _p, _p, _p],
    "mcf_fast_mm_reserve": [_i64, _i64, _i64, C.c_int, _p],
    "mcf_fast_tc_plan": [_i64, _int, _p, _p, _p],
    "mcf_fast_tc_crt_table": [_int, _p, _p, _p, _p, _p],
    "mcf_tc_gemm_s8": [_p, _p, _p, _i64, _i64, _i64, _int, _i64, _p, _p],
    "mcf_mc_transpose2d": [_int, _p, _int, _i64, _i64, _p, _p],
    "mcf_halfspace_distance": [_int, _p, _int, _i64, _i64, _p, _p, _i64, _p, _p, _p],
    "mcf_h_renorm": [_int, _int, _p, _int, _p, _int, _i64],
    "mcf_h_eft": [_int, _int, _p, _p, _p, _p, _i64],
    "mcf_h_mc_transpose2d": [_int, _p, _int, _i64, _i64, _p],
    "mcf_probe_pipe_rates": [_p, _p],
    "mcf_mlp_bias_act": [_p, _int, _p, _i64, _i64, _int, _p, _p, _p],
    "mcf_mlp_cross_entropy": [_p, _p, _i64, _i64, _i64, _p, _p, _p, _p],
    "mcf_mlp_loss_sum": [_p, _i64, _p, _p],
    "mcf_gemm_f32_ordered": [_int, _int, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _p],
    "mcf_rowsum_f32_ordered": [_p, _i64, _i64, _p, _p],
    "mcf_gemm_f32_fast": [_int, _int, _p, _i64, _p, _i64, _p, _i64, _i64, _i64, _i64, _p, _p],
    "mcf_rowsum_f32_fast": [_p, _i64, _i64, _p, _p],
    "mcf_mc_relu": [_int, _p, _int, _p, _i64, _p],
    "mcf_halfspace_arg": [_int, _p, _int, _i64, _i64, _p, _p, _i64, _p, _p, _p],
    "mcf_mlp_linear_fwd": [_p, _int, _p, _i64, _i64, _i64, _p, _int, _p, _p, _p, _int, _p],
    "mcf_mc_softmax": [_int, _p, _int, _i64, _i64, _i64, _p, _p],
    "mcf_sgd_grow": [_p, _int, _p, _i64, C.c_float, _p],
}


def lib():
    """Load libmcf_b200.so (raises if it is not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MCFError(f"{LIB_PATH} is not built; run paper_2207_08867_b200/build.py")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _int
        L.mcf_last_error.restype = C.c_char_p
        L.mcf_abi_version.restype = _int
        L.mcf_launch_count.restype = _i64
        L.mcf_rng_uniform.argtypes = [C.c_uint64, _i64, _p]
        L.mcf_rng_uniform.restype = None
        L.mcf_rng_normal.argtypes = [C.c_uint64, _i64, _p]
        L.mcf_rng_normal.restype = None
        L.mcf_rng_below.argtypes = [C.c_uint64, C.c_uint64, _i64, _p]
        L.mcf_rng_below.restype = None
        L.mcf_mm_mcn_mcmc_refusal.restype = _int
        _lib = L
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().mcf_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise UnsupportedOperation(msg)
    if rc == 5:  # std::domain_error in the reference
        raise ValueError(msg)
    raise MCFError(f"[{rc}] {msg}")


def launch_count() -> int:
    return lib().mcf_launch_count()


def reset_launch_count() -> None:
    lib().mcf_reset_launch_count()


from . import ops  # noqa: E402  (device-tensor operators)
from . import host  # noqa: E402  (host-buffer operators)
from .ops import *  # noqa: E402,F401,F403
