"""Elementwise operators on 2^24 binary64 nc=2 elements: device time and HBM fraction."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402

n = 1 << 24
g = torch.Generator(device="cuda").manual_seed(0)
v = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1)
x = torch.stack([v, v * 2.0**-60], -1).contiguous()
y = torch.stack([v + 0.5 * torch.sign(v), v * 2.0**-61], -1).contiguous()
w = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1)


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, f, byts in (("grow_expn", lambda: mcf.grow_expn(x, w), 40), ("add_mcn", lambda: mcf.add_mcn(x, y), 48),
                      ("mul_mcn", lambda: mcf.mul_mcn(x, y), 48), ("div_mcn", lambda: mcf.div_mcn(x, y), 48),
                      ("square_mcn", lambda: mcf.square_mcn(x), 32), ("exp_mcn", lambda: mcf.exp_mcn(x), 32)):
    ms = t(f)
    print(f"b64 nc=2 {name:12s} {ms * 1e3:8.1f} us  {n * byts / ms / 1e6:7.0f} GB/s")
