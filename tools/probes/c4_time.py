"""Config 4 (MC x MC 16384^3, binary32 nc=2) through the tensor-core path: one
product, device time, fallback count (via the phases API is MC x T only, so
time the whole call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402

N4 = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(1)


def u():
    return torch.rand((N4, N4), generator=g, device="cuda", dtype=torch.float64) * 2 - 1


def split(v):
    c0 = v.float()
    c1 = (v - c0.double()).float()
    return torch.stack([c0, c1], -1).contiguous()


a = split(u())
b = split(u())
out = mcf.mm_mcmc(a, b, plan=mcf.FAST)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = mcf.mm_mcmc(a, b, plan=mcf.FAST)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"config4 fp32 nc=2 {N4}^3: {ms:.1f} ms  {2 * N4**3 / ms / 1e9:.0f} GFLOP/s eff")
