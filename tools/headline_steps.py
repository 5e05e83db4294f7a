"""The bench's headline step alone (config 2: one MC(4096x4096, nc=2) x T(4096x4096)
product with plan MCF_FAST, data from data.config2), 3 warm-up + 2 steps, for an
ncu launch list whose kernels are exactly the timed step's (bench.py also runs
context measurements: the FP64-pipe path, pipe probes, the elementwise suite)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = K = N = 4096
a_h, b_h = data.config2(M, K, N)
a = torch.from_numpy(a_h).cuda()
b = torch.from_numpy(b_h).cuda()
out = torch.empty((M, N, 2), dtype=torch.float32, device="cuda")
lib = mcf.lib()
for _ in range(5):
    rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, M, K, N, 0, out.data_ptr(), mcf.FAST, 1,
                         torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.mcf_last_error()
torch.cuda.synchronize()
print("ok")
