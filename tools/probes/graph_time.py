"""Config 2 product: direct calls vs a captured CUDA graph of the same call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = K = N = 4096
a_h, b_h = data.config2(M, K, N)
a = torch.from_numpy(a_h).cuda()
b = torch.from_numpy(b_h).cuda()
out = torch.empty((M, N, 2), dtype=torch.float32, device="cuda")
lib = mcf.lib()
s = torch.cuda.Stream()


def step():
    rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, M, K, N, 0, out.data_ptr(), mcf.FAST, 1,
                         torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.mcf_last_error()


def timeit(f, reps=10):
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


with torch.cuda.stream(s):
    d = timeit(step)
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    gr = timeit(g.replay)
    same = torch.equal(out.view(torch.int32), ref.view(torch.int32))
print(f"direct {d:.3f} ms, graph replay {gr:.3f} ms, bitwise same: {same}")
