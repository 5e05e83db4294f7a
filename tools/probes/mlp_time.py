"""Time the config-3 MC-MLP step (784-1024-1024-10, nc=2, batch 8192) on one GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import mlp  # noqa: E402

dims = [784, 1024, 1024, 10]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
plan = mcf.FAST if "exact" not in sys.argv else mcf.SEQUENTIAL
params = mlp.init_params(dims, 2)
x, y = mlp.make_batch(N)
model = mlp.MCMLP(dims, params, lr=0.01, plan=plan)
xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
yt = torch.from_numpy(y).cuda()
for _ in range(3):
    model.step(xt, yt, N)
torch.cuda.synchronize()
ts = []
losses = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s = model.step(xt, yt, N)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
    losses.append(model.loss_value(s, N))
ms = float(np.median(ts))
mads_fwd = N * sum(dims[i] * dims[i + 1] for i in range(3))
print(f"MC-MLP step N={N}: {ms:.2f} ms  ({1e3/ms:.1f} steps/s), fwd MC MADs {mads_fwd:.3e}, losses {losses[0]:.6f} -> {losses[-1]:.6f}")
# per-kernel breakdown with a profiler-free approach: time the forward mm alone
W0 = model.W[0]
A0 = xt
Z = torch.empty((1024, N, 2), device="cuda")
lib = mcf.lib()
st = torch.cuda.current_stream().cuda_stream
for name, fn in [
    ("fwd mm L1", lambda: lib.mcf_bmm_mcn(mcf.B32, W0.data_ptr(), 2, A0.data_ptr(), 1, 1024, 784, N, 0, Z.data_ptr(), plan, 1, st)),
]:
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    print(f"  {name}: {a.elapsed_time(b):.2f} ms")
