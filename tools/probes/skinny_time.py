"""The short-A FP64-pipe kernel on the config-3 class layer's shape (10 x 1024 x 8192)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402

m, k, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (10, 1024, 8192)))
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.rand(m, k, 2, device="cuda", generator=g) * 2 - 1).float()
x[..., 1] *= 2.0**-25
w = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1).float()
for _ in range(3):
    mcf.mm_mcn(x, w, plan=mcf.FAST)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    mcf.mm_mcn(x, w, plan=mcf.FAST)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"mm MC(nc=2) x T {m} x {k} x {n} FAST: {np.median(ts) * 1e3:.1f} us")
