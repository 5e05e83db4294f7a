"""Config-3 MC-MLP: 3 warm-up steps + 2 steps (for an ncu launch list of the step's kernels)."""
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
for _ in range(5):
    model.step(xt, yt, N)
torch.cuda.synchronize()
print("ok")
