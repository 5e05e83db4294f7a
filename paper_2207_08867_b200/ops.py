"""Device-tensor MCF operators (torch CUDA tensors) over the C-ABI.

Names and argument meaning follow the reference (mc_ops.hpp / linalg.hpp /
eft.hpp); each docstring cites the reference entry point it replaces.  MC
tensors are ``(..., nc)`` with the component axis last; the working-precision
operand ``v`` is a tensor of the same dtype, a scalar, or a trailing suffix of
the MC tensor's shape (mc_ops.hpp:14-15, 317-329).
"""
from __future__ import annotations

import torch

from . import B16, B32, B64, FAST, FAST_FP64, PAIRWISE_TREE, SEQUENTIAL, UnsupportedOperation, _check, lib  # noqa: F401

__all__ = [
    "two_sum", "two_prod", "renormalize", "simple_renorm", "approx", "negate", "grow_expn",
    "scaling_n", "div_n", "add_mcn", "div_mcn", "mul_mcn", "mul_mcn_slow", "square_mcn",
    "exp_mcn", "dot_mcn", "mv_mcn", "mm_mcn", "bmm_mcn", "mm4d_mcn", "matmul_mcn", "addmm_mcn",
    "mc_transpose2d", "mm_mcmc", "dot_mcmc", "mc_relu", "mc_softmax", "halfspace_distance", "from_float",
    "PREC",
]

PREC = {torch.float16: B16, torch.float32: B32, torch.float64: B64}


def _prec(t: torch.Tensor) -> int:
    if t.dtype not in PREC:
        raise ValueError(f"unsupported component dtype {t.dtype}")
    if not t.is_cuda:
        raise ValueError("device operators need CUDA tensors (use mcf.host for host arrays)")
    return PREC[t.dtype]


def _c(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_contiguous() else t.contiguous()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _nc(x: torch.Tensor) -> int:
    if x.dim() < 1:
        raise ValueError("an MC tensor needs a trailing component axis")
    return x.shape[-1]


def _shape_str(s) -> str:
    return "(" + ",".join(str(d) for d in s) + ")"


def _operand(x: torch.Tensor, v, op: str) -> torch.Tensor:
    """Working-precision operand: scalar or trailing suffix (mc_ops.hpp:317-329)."""
    if not torch.is_tensor(v):
        v = torch.tensor([v], dtype=x.dtype, device=x.device)
    v = _c(v.to(dtype=x.dtype, device=x.device))
    xs = tuple(x.shape[:-1])
    if v.numel() != 1:
        vs = tuple(v.shape)
        if len(vs) > len(xs):
            raise ValueError(f"{op}: operand shape {_shape_str(vs)} does not broadcast over {_shape_str(xs)}")
        if xs[len(xs) - len(vs):] != vs:
            raise ValueError(f"{op}: operand shape {_shape_str(vs)} is not a trailing suffix of {_shape_str(xs)}")
    return v


def _ptr(t):
    return None if t is None else t.data_ptr()


# ---- EFT arrays (eft.hpp:89-111) ------------------------------------------------

def two_sum(a: torch.Tensor, b: torch.Tensor):
    """(s, e) with s = fl(a+b), s + e == a + b  [eft.hpp:31-38, array form :89-99]."""
    a, b = _c(a), _c(b.to(a.dtype))
    s, e = torch.empty_like(a), torch.empty_like(a)
    _check(lib().mcf_two_sum(_prec(a), _ptr(a), _ptr(b), _ptr(s), _ptr(e), a.numel(), _stream()))
    return s, e


def two_prod(a: torch.Tensor, b: torch.Tensor):
    """(p, e) with p = fl(ab), p + e == ab  [eft.hpp:75-86, array form :101-111]."""
    a, b = _c(a), _c(b.to(a.dtype))
    p, e = torch.empty_like(a), torch.empty_like(a)
    _check(lib().mcf_two_prod(_prec(a), _ptr(a), _ptr(b), _ptr(p), _ptr(e), a.numel(), _stream()))
    return p, e


# ---- renormalization -----------------------------------------------------------

def renormalize(h: torch.Tensor, r_nc: int) -> torch.Tensor:
    """Priest renormalization to r_nc components  [mc_ops.hpp:339-348]."""
    h = _c(h)
    nc = _nc(h)
    out = torch.empty(h.shape[:-1] + (r_nc,), dtype=h.dtype, device=h.device)
    _check(lib().mcf_renormalize(_prec(h), _ptr(h), nc, _ptr(out), r_nc, h.numel() // max(nc, 1), _stream()))
    return out


def simple_renorm(h: torch.Tensor, r_nc: int) -> torch.Tensor:
    """Zero compaction keeping order  [mc_ops.hpp:350-359]."""
    h = _c(h)
    nc = _nc(h)
    out = torch.empty(h.shape[:-1] + (r_nc,), dtype=h.dtype, device=h.device)
    _check(lib().mcf_simple_renorm(_prec(h), _ptr(h), nc, _ptr(out), r_nc, h.numel() // max(nc, 1), _stream()))
    return out


def approx(x: torch.Tensor) -> torch.Tensor:
    """Smallest-first working-precision sum  [mctensor.hpp:56-65]."""
    x = _c(x)
    nc = _nc(x)
    out = torch.empty(x.shape[:-1], dtype=x.dtype, device=x.device)
    _check(lib().mcf_approx(_prec(x), _ptr(x), nc, _ptr(out), x.numel() // nc, _stream()))
    return out


def negate(x: torch.Tensor) -> torch.Tensor:
    """[mc_ops.hpp:376-381]"""
    x = _c(x)
    nc = _nc(x)
    out = torch.empty_like(x)
    _check(lib().mcf_negate(_prec(x), _ptr(x), nc, _ptr(out), x.numel() // nc, _stream()))
    return out


def from_float(t: torch.Tensor, nc: int) -> torch.Tensor:
    """Embed a working-precision tensor: component 0 = t  [mctensor.hpp:35-41]."""
    out = torch.zeros(tuple(t.shape) + (nc,), dtype=t.dtype, device=t.device)
    out[..., 0] = t
    return out


# ---- elementwise MCF operators -----------------------------------------------------

def grow_expn(x: torch.Tensor, v) -> torch.Tensor:
    """x + v for a working-precision v (Grow-ExpN)  [mc_ops.hpp:384-394]."""
    x = _c(x)
    nc = _nc(x)
    v = _operand(x, v, "grow_expn")
    out = torch.empty_like(x)
    _check(lib().mcf_grow_expn(_prec(x), _ptr(x), nc, _ptr(v), v.numel(), _ptr(out), x.numel() // nc, _stream()))
    return out


def scaling_n(x: torch.Tensor, v, expanded: bool = False) -> torch.Tensor:
    """x * v for a working-precision v (ScalingN); nc+1 comps if expanded  [mc_ops.hpp:398-410]."""
    x = _c(x)
    nc = _nc(x)
    v = _operand(x, v, "scaling_n")
    onc = nc + 1 if expanded else nc
    out = torch.empty(x.shape[:-1] + (onc,), dtype=x.dtype, device=x.device)
    _check(lib().mcf_scaling_n(_prec(x), _ptr(x), nc, _ptr(v), v.numel(), int(expanded), _ptr(out), x.numel() // nc, _stream()))
    return out


def div_n(v, y: torch.Tensor) -> torch.Tensor:
    """v / y for a working-precision v (DivN)  [mc_ops.hpp:494-507]."""
    y = _c(y)
    nc = _nc(y)
    v = _operand(y, v, "div_n")
    out = torch.empty_like(y)
    _check(lib().mcf_div_n(_prec(y), _ptr(v), v.numel(), _ptr(y), nc, _ptr(out), y.numel() // nc, _stream()))
    return out


def _binary(fn, name, x, y):
    x, y = _c(x), _c(y)
    if x.shape[:-1] != y.shape[:-1]:
        raise ValueError(f"{name}: shape mismatch {_shape_str(x.shape[:-1])} vs {_shape_str(y.shape[:-1])}")
    if y.dtype != x.dtype:
        raise ValueError(f"{name}: component dtypes differ")
    ncx, ncy = _nc(x), _nc(y)
    out = torch.empty(x.shape[:-1] + (max(ncx, ncy),), dtype=x.dtype, device=x.device)
    _check(fn(_prec(x), _ptr(x), ncx, _ptr(y), ncy, _ptr(out), x.numel() // ncx, _stream()))
    return out


def add_mcn(x, y):
    """Add-MCN; mixed nc padded to max  [mc_ops.hpp:440-446]."""
    return _binary(lib().mcf_add_mcn, "add_mcn", x, y)


def div_mcn(x, y):
    """Div-MCN (long division)  [mc_ops.hpp:448-454]."""
    return _binary(lib().mcf_div_mcn, "div_mcn", x, y)


def mul_mcn(x, y):
    """Mul-MCN fast: x / (1/y) with zero short-circuit  [mc_ops.hpp:456-462]."""
    return _binary(lib().mcf_mul_mcn, "mul_mcn", x, y)


def mul_mcn_slow(x, y):
    """Mul-MCN slow (direct partial products)  [mc_ops.hpp:464-470]."""
    return _binary(lib().mcf_mul_mcn_slow, "mul_mcn_slow", x, y)


def square_mcn(x):
    """Square-MCN  [mc_ops.hpp:472-480]."""
    x = _c(x)
    nc = _nc(x)
    out = torch.empty_like(x)
    _check(lib().mcf_square_mcn(_prec(x), _ptr(x), nc, _ptr(out), x.numel() // nc, _stream()))
    return out


def exp_mcn(x):
    """Exp-MCN (correctly rounded binary64 lead factor)  [mc_ops.hpp:482-490]."""
    x = _c(x)
    nc = _nc(x)
    out = torch.empty_like(x)
    _check(lib().mcf_exp_mcn(_prec(x), _ptr(x), nc, _ptr(out), x.numel() // nc, _stream()))
    return out


# ---- MC activations (autodiff.hpp:340-413) -------------------------------------------

def mc_relu(x):
    """mc_relu_op forward: zero every component where approx() <= 0  [autodiff.hpp:340-350]."""
    x = _c(x)
    nc = _nc(x)
    out = torch.empty_like(x)
    _check(lib().mcf_mc_relu(_prec(x), _ptr(x), nc, _ptr(out), x.numel() // nc, _stream()))
    return out


def mc_softmax(x, axis=-1):
    """Softmax over `axis` in MC arithmetic: max shift via grow_expn, exp_mcn,
    add_mcn row sum, div_mcn  [autodiff.hpp:383-413].  Rank 1 / 2 values only."""
    x = _c(x)
    nc = _nc(x)
    shp = tuple(x.shape[:-1])
    rank = len(shp)
    ax = axis + rank if axis < 0 else axis
    if rank < 1 or rank > 2 or ax < 0 or ax >= rank:
        raise ValueError("mc_softmax: supported on rank 1/2 tensors")
    if rank == 1:
        outer, n, inner = 1, shp[0], 1
    elif ax == 1:
        outer, n, inner = shp[0], shp[1], 1
    else:
        outer, n, inner = 1, shp[0], shp[1]
    out = torch.empty_like(x)
    _check(lib().mcf_mc_softmax(_prec(x), _ptr(x), nc, outer, n, inner, _ptr(out), _stream()))
    return out


def halfspace_distance(table, u, v, return_arg=False):
    """Half-space model distances between rows u[p] and v[p] of an (n, dim, nc)
    MC embedding table  [hyperbolic.hpp:160-226]: the arcosh argument in MC
    arithmetic (bit-identical), then arcosh_guarded in binary64."""
    table = _c(table)
    nc = _nc(table)
    if table.dim() != 3:
        raise ValueError("halfspace_distance: table rank")
    n, dim = table.shape[0], table.shape[1]
    u = torch.as_tensor(u, dtype=torch.int64, device=table.device).contiguous()
    v = torch.as_tensor(v, dtype=torch.int64, device=table.device).contiguous()
    arg = torch.empty(u.shape, dtype=torch.float64, device=table.device)
    dist = torch.empty(u.shape, dtype=torch.float64, device=table.device)
    # synchronous, with the reference's domain check (non-positive height -> ValueError)
    _check(lib().mcf_halfspace_distance(_prec(table), _ptr(table), nc, n, dim, _ptr(u), _ptr(v), u.numel(),
                                        _ptr(arg), _ptr(dist), _stream()))
    return (dist, arg) if return_arg else dist


# ---- contractions (linalg.hpp) ------------------------------------------------------

def _plan(plan):
    if plan is None:
        return SEQUENTIAL, 1
    if isinstance(plan, tuple):
        return int(plan[0]), int(plan[1])
    return int(plan), 1


def _bmm(x, w, batch, m, k, n, w_batched, out_shape, plan):
    x, w = _c(x), _c(w.to(x.dtype))
    nc = _nc(x)
    strategy, leaf = _plan(plan)
    out = torch.empty(tuple(out_shape) + (nc,), dtype=x.dtype, device=x.device)
    _check(lib().mcf_bmm_mcn(_prec(x), _ptr(x), nc, _ptr(w), batch, m, k, n, int(w_batched), _ptr(out), strategy, leaf, _stream()))
    return out


def _rank(x):
    return x.dim() - 1


def dot_mcn(x, v, plan=None):
    """MC vector . working vector  [linalg.hpp:103-116]."""
    if _rank(x) != 1:
        raise ValueError(f"dot_mcn: expected rank 1, got {_shape_str(x.shape[:-1])}")
    if v.dim() != 1:
        raise ValueError(f"dot_mcn: expected rank 1, got {_shape_str(v.shape)}")
    if x.shape[0] != v.shape[0]:
        raise ValueError(f"dot_mcn: length mismatch {_shape_str(x.shape[:-1])} vs {_shape_str(v.shape)}")
    return _bmm(x, v, 1, 1, x.shape[0], 1, False, (), plan)


def mv_mcn(x, v, plan=None):
    """MC matrix x working vector  [linalg.hpp:119-135]."""
    if _rank(x) != 2:
        raise ValueError(f"mv_mcn: expected rank 2, got {_shape_str(x.shape[:-1])}")
    if v.dim() != 1:
        raise ValueError(f"mv_mcn: expected rank 1, got {_shape_str(v.shape)}")
    if x.shape[1] != v.shape[0]:
        raise ValueError(f"mv_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(v.shape)}")
    return _bmm(x, v, 1, x.shape[0], x.shape[1], 1, False, (x.shape[0],), plan)


def mm_mcn(x, w, plan=None):
    """MC matrix x working matrix  [linalg.hpp:138-157].  MC x MC raises like linalg.hpp:159-166."""
    if w.dim() == 3 and _rank(x) == 2:  # an MC matrix operand: the reference's MC x MC overload
        _check(lib().mcf_mm_mcn_mcmc_refusal())
    if _rank(x) != 2:
        raise ValueError(f"mm_mcn: expected rank 2, got {_shape_str(x.shape[:-1])}")
    if w.dim() != 2:
        raise ValueError(f"mm_mcn: expected rank 2, got {_shape_str(w.shape)}")
    if x.shape[1] != w.shape[0]:
        raise ValueError(f"mm_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
    m, k = x.shape[0], x.shape[1]
    n = w.shape[1]
    return _bmm(x, w, 1, m, k, n, False, (m, n), plan)


def bmm_mcn(x, w, plan=None):
    """Batched mm over one leading axis  [linalg.hpp:205-216]."""
    if _rank(x) != 3 or w.dim() != 3:
        raise ValueError(f"bmm_mcn: expected rank 3, got {_shape_str(x.shape[:-1])} and {_shape_str(w.shape)}")
    if x.shape[0] != w.shape[0] or x.shape[2] != w.shape[1]:
        raise ValueError(f"bmm_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
    b, m, k = x.shape[:3]
    n = w.shape[2]
    return _bmm(x, w, b, m, k, n, True, (b, m, n), plan)


def mm4d_mcn(x, w, plan=None):
    """Batched mm over two leading axes  [linalg.hpp:220-231]."""
    if _rank(x) != 4 or w.dim() != 4:
        raise ValueError(f"mm4d_mcn: expected rank 4, got {_shape_str(x.shape[:-1])} and {_shape_str(w.shape)}")
    if x.shape[0] != w.shape[0] or x.shape[1] != w.shape[1] or x.shape[3] != w.shape[2]:
        raise ValueError(f"mm4d_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
    b0, b1, m, k = x.shape[:4]
    n = w.shape[3]
    return _bmm(x, w, b0 * b1, m, k, n, True, (b0, b1, m, n), plan)


def matmul_mcn(x, w, plan=None):
    """Rank dispatcher  [linalg.hpp:258-299]."""
    rx, rw = _rank(x), w.dim()
    if rx == 1 and rw == 1:
        return dot_mcn(x, w, plan)
    if rx == 2 and rw == 1:
        return mv_mcn(x, w, plan)
    if rx == 1 and rw == 2:
        if x.shape[0] != w.shape[0]:
            raise ValueError(f"matmul_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
        return mm_mcn(x.unsqueeze(0), w, plan)[0]
    if rx == 2 and rw == 2:
        if x.shape[1] != w.shape[0]:
            raise ValueError(f"matmul_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
        return mm_mcn(x, w, plan)
    if rx == 3 and rw == 3:
        return bmm_mcn(x, w, plan)
    if rx == 3 and rw == 2:
        if x.shape[2] != w.shape[0]:
            raise ValueError(f"matmul_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
        b, m, k = x.shape[:3]
        return _bmm(x, w, b, m, k, w.shape[1], False, (b, m, w.shape[1]), plan)
    if rx == 4 and rw == 4:
        return mm4d_mcn(x, w, plan)
    if rx == 4 and rw == 2:
        if x.shape[3] != w.shape[0]:
            raise ValueError(f"matmul_mcn: incompatible shapes {_shape_str(x.shape[:-1])} vs {_shape_str(w.shape)}")
        b0, b1, m, k = x.shape[:4]
        return _bmm(x, w, b0 * b1, m, k, w.shape[1], False, (b0, b1, m, w.shape[1]), plan)
    raise ValueError(f"matmul_mcn: unsupported rank pair for shapes {_shape_str(x.shape[:-1])} and {_shape_str(w.shape)}")


def addmm_mcn(bias, x, w, alpha=1.0, beta=1.0, plan=None):
    """beta*bias + alpha*(x @ w), factors through ScalingN  [linalg.hpp:234-253]."""
    prod = mm_mcn(x, w, plan)
    if alpha != 1.0:
        prod = scaling_n(prod, torch.tensor([alpha], dtype=x.dtype, device=x.device))
    sb = scaling_n(bias, torch.tensor([beta], dtype=x.dtype, device=x.device)) if beta != 1.0 else bias
    if sb.shape[:-1] != prod.shape[:-1]:
        bs, ps = tuple(sb.shape[:-1]), tuple(prod.shape[:-1])
        if len(bs) > len(ps) or ps[len(ps) - len(bs):] != bs:
            raise ValueError(f"addmm_mcn: operand shape {_shape_str(bs)} is not a trailing suffix of {_shape_str(ps)}")
        sb = sb.expand(ps + (sb.shape[-1],))
    return add_mcn(sb, prod)


def mc_transpose2d(x):
    """Component-preserving 2-D transpose  [linalg.hpp:301-315]: (m, n, nc) -> (n, m, nc)."""
    x = _c(x)
    if _rank(x) != 2:
        raise ValueError(f"mc_transpose2d: expected rank 2, got {_shape_str(x.shape[:-1])}")
    m, n, nc = x.shape
    out = torch.empty((n, m, nc), dtype=x.dtype, device=x.device)
    _check(lib().mcf_mc_transpose2d(_prec(x), _ptr(x), nc, m, n, _ptr(out), _stream()))
    return out


def mm_mcmc(x, y, plan=None):
    """NEW: MC x MC matrix product (the reference refuses it, linalg.hpp:159-166).
    plan SEQUENTIAL = recipe B (bitwise), FAST = compensated binary64."""
    x, y = _c(x), _c(y.to(x.dtype))
    if _rank(x) != 2 or _rank(y) != 2 or x.shape[1] != y.shape[0] or x.shape[-1] != y.shape[-1]:
        raise ValueError(f"mm_mcmc: incompatible shapes {_shape_str(x.shape)} vs {_shape_str(y.shape)}")
    nc = _nc(x)
    m, k, n = x.shape[0], x.shape[1], y.shape[1]
    out = torch.empty((m, n, nc), dtype=x.dtype, device=x.device)
    strategy, _ = _plan(plan)
    _check(lib().mcf_mm_mcmc(_prec(x), _ptr(x), _ptr(y), nc, m, k, n, _ptr(out), strategy, _stream()))
    return out


def dot_mcmc(x, y, plan=None):
    """NEW: batched MC x MC dots, x, y (batch, k, nc)."""
    x, y = _c(x), _c(y.to(x.dtype))
    if x.shape != y.shape or x.dim() != 3:
        raise ValueError(f"dot_mcmc: incompatible shapes {_shape_str(x.shape)} vs {_shape_str(y.shape)}")
    b, k, nc = x.shape
    out = torch.empty((b, nc), dtype=x.dtype, device=x.device)
    strategy, _ = _plan(plan)
    _check(lib().mcf_dot_mcmc(_prec(x), _ptr(x), _ptr(y), nc, b, k, _ptr(out), strategy, _stream()))
    return out
