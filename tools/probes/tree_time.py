"""Reference-order plans on long-K shapes: pairwise tree (warp-parallel split-K)
vs the sequential plan (a thread per output)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g = torch.Generator(device="cuda").manual_seed(0)
for (m, k, n) in ((4096, 4096, 1), (64, 65536, 1), (256, 4096, 64)):
    x = (torch.rand(m, k, 2, device="cuda", generator=g) * 2 - 1).float()
    x[..., 1] *= 2.0**-25
    w = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1).float()
    seq = t(lambda: mcf.mm_mcn(x, w, plan=mcf.SEQUENTIAL))
    tree = t(lambda: mcf.mm_mcn(x, w, plan=(mcf.PAIRWISE_TREE, 1)))
    print(f"m={m} k={k} n={n} nc=2: sequential {seq:.2f} ms, pairwise tree {tree:.2f} ms "
          f"({m * n * k / tree / 1e6:.2f} GMAD/s)")
