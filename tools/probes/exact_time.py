"""Reference-order (bit-identical) MC x T product: 512 x 4096 x 4096, nc=2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402
from paper_2207_08867_b200 import data  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 512
a_h, b_h = data.config2(4096, 4096, 4096)
a = torch.from_numpy(a_h[:M]).cuda()
b = torch.from_numpy(b_h).cuda()
out = mcf.mm_mcn(a, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = mcf.mm_mcn(a, b)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"exact mm {M}x4096x4096 nc=2: {ms:.1f} ms  {2 * M * 4096 * 4096 / ms / 1e6:.1f} GFLOP/s eff")
