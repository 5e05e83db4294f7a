"""Device time of one rank's share of the config-2 product under row sharding
(rows = 4096 / G for G = 1, 2, 4, 8): the per-rank step of bench.py --gpus G."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = K = N = 4096
a_h, b_h = data.config2(M, K, N)
b = torch.from_numpy(b_h).cuda()
lib = mcf.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
base = None
for g in (1, 2, 4, 8):
    rows = M // g
    a = torch.from_numpy(a_h[:rows]).cuda()
    out = torch.empty((rows, N, 2), dtype=torch.float32, device="cuda")

    def step():
        rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, rows, K, N, 0, out.data_ptr(), mcf.FAST, 1,
                             torch.cuda.current_stream().cuda_stream)
        assert rc == 0, lib.mcf_last_error()

    for _ in range(3):
        step()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    base = base or ms
    print(f"G={g}: rows {rows}: {ms:.3f} ms per rank step, strong-scaling efficiency {base / (g * ms):.2f}")
