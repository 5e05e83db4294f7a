"""Helpers for the -m gpu tests: numpy in, CUDA C-ABI in the middle, numpy out."""
import numpy as np
import torch

import paper_2207_08867_b200 as mcf


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run(op, *args, **kw):
    """Call mcf.<op> on device copies of numpy args; return numpy results."""
    conv = [dev(a) if isinstance(a, np.ndarray) else a for a in args]
    r = getattr(mcf, op)(*conv, **kw)
    if isinstance(r, tuple):
        return tuple(host(t) for t in r)
    return host(r)
