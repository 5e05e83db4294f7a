"""Device time of one rank's share of the config-2 product: the per-rank step of
bench.py --gpus G under a Gr x Gc grid of output blocks (rows / Gr of A, columns
/ Gc of B; Gc = 1 is plain row sharding)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = K = N = 4096
a_h, b_h = data.config2(M, K, N)
lib = mcf.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
base = None
for gr, gc in ((1, 1), (2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2), (2, 4), (1, 8)):
    rows, cols = M // gr, N // gc
    a = torch.from_numpy(a_h[:rows]).cuda()
    b = torch.from_numpy(b_h[:, :cols].copy()).cuda()
    out = torch.empty((rows, cols, 2), dtype=torch.float32, device="cuda")

    def step():
        rc = lib.mcf_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, rows, K, cols, 0, out.data_ptr(), mcf.FAST, 1,
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
    g = gr * gc
    print(f"G={g} ({gr} x {gc}): block {rows} x {cols}: {ms:.3f} ms per rank step, "
          f"strong-scaling efficiency {base / (g * ms):.2f}", flush=True)
