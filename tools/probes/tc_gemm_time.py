"""The tcgen05 residue GEMM alone: [batch][m][kp] x [batch][n][kp]^T -> int8 residues."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402

m, n, kp, batch = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 4096, 4096, 17)))
lib = mcf.lib()
mods = (C.c_int * 32)()
lib.mcf_fast_tc_crt_table(batch, mods, None, None, None, None)
a = torch.randint(-128, 128, (batch, m, kp), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 128, (batch, n, kp), dtype=torch.int8, device="cuda")
out = torch.empty((batch, m, n), dtype=torch.int8, device="cuda")


def run():
    rc = lib.mcf_tc_gemm_s8(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, kp, batch, n, mods,
                            torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.mcf_last_error()


for _ in range(2):
    run()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
print(f"tc gemm {batch} x ({m} x {n} x {kp}): {ms:.3f} ms, {2.0 * m * n * kp * batch / ms / 1e9:.0f} TOPS")
