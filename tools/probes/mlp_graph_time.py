"""Config-3 MC-MLP step: direct calls vs a captured CUDA graph of the same step,
plus the step's launch count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import mlp  # noqa: E402

dims = [784, 1024, 1024, 10]
N = 8192
params = mlp.init_params(dims, 2)
x, y = mlp.make_batch(N)
model = mlp.MCMLP(dims, params, lr=0.01, plan=mcf.FAST)
xt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
yt = torch.from_numpy(y).cuda()


def timeit(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    d = timeit(lambda: model.step(xt, yt, N))
    mcf.reset_launch_count()
    model.step(xt, yt, N)
    torch.cuda.synchronize()
    print("launches per step:", mcf.launch_count())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        model.step(xt, yt, N)
    gr = timeit(g.replay)
print(f"direct {d:.3f} ms, graph replay {gr:.3f} ms")
