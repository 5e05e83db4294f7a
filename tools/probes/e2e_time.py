"""Time the host-buffer entry point mcf_h_bmm_mcn (config 2, pinned buffers):
the bench's e2e number, alone, plus the raw H2D / D2H copy rates of the box."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = K = N = 4096
a_h, b_h = data.config2(M, K, N)
a = torch.from_numpy(a_h).pin_memory()
b = torch.from_numpy(b_h).pin_memory()
o = torch.empty((M, N, 2), dtype=torch.float32).pin_memory()
lib = mcf.lib()
plan = mcf.FAST_FP64 if "fp64" in sys.argv else mcf.FAST


def run():
    rc = lib.mcf_h_bmm_mcn(mcf.B32, a.data_ptr(), 2, b.data_ptr(), 1, M, K, N, 0, o.data_ptr(), plan)
    assert rc == 0, lib.mcf_last_error()


run()
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    run()
    ts.append(time.perf_counter() - t0)
ts.sort()
ms = ts[len(ts) // 2] * 1e3
tag = f"chunk={os.environ.get('MCF_OZ_CHUNK', '-')} blocks={os.environ.get('MCF_OZ_BLOCKS', '-')}"
print(f"e2e {tag}: {ms:.2f} ms  {2*M*N*K/ms/1e6:.0f} GFLOP/s (min {ts[0]*1e3:.2f})")
if "copies" in sys.argv:
    d = torch.empty(a.shape, dtype=a.dtype, device="cuda")
    for name, f in (("H2D", lambda: d.copy_(a, non_blocking=True)), ("D2H", lambda: a.copy_(d, non_blocking=True))):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"{name}: {a.numel() * 4 / dt / 1e9:.1f} GB/s")
if "duplex" in sys.argv:
    d1 = torch.empty(a.shape, dtype=a.dtype, device="cuda")
    d2 = torch.empty(a.shape, dtype=a.dtype, device="cuda")
    h2 = torch.empty(a.shape, dtype=a.dtype).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        with torch.cuda.stream(s1):
            d1.copy_(a, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d1.copy_(a, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"duplex: {2 * a.numel() * 4 / dt / 1e9:.1f} GB/s total ({a.numel() * 4 / dt / 1e9:.1f} each way)")
