"""The tensor-core product on heavy-tailed operands: fallback outputs and time."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2207_08867_b200 as mcf
from paper_2207_08867_b200 import data

lib = mcf.lib()
rng = np.random.default_rng(0)
m = k = n = 2048
cases = {
    "uniform": (rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (k, n))),
    "normal": (rng.normal(0, 1, (m, k)), rng.normal(0, 1, (k, n))),
    "lognormal(0,3) signed": (rng.lognormal(0, 3, (m, k)) * rng.choice([-1, 1], (m, k)), rng.lognormal(0, 3, (k, n)) * rng.choice([-1, 1], (k, n))),
    "cauchy": (rng.standard_cauchy((m, k)), rng.standard_cauchy((k, n))),
    "config0-like 2^U(-8,8)": (rng.uniform(-1, 1, (m, k)) * np.exp2(rng.uniform(-8, 8, (m, k))), rng.uniform(-1, 1, (k, n)) * np.exp2(rng.uniform(-8, 8, (k, n)))),
    "sparse 90% zeros": (rng.normal(0, 1, (m, k)) * (rng.uniform(0, 1, (m, k)) < 0.1), rng.normal(0, 1, (k, n)) * (rng.uniform(0, 1, (k, n)) < 0.1)),
}
for name, (av, bv) in cases.items():
    a = torch.from_numpy(data.split(av.ravel(), 2).reshape(m, k, 2)).cuda()
    b = torch.from_numpy(bv.astype(np.float32)).cuda()
    out = torch.empty((m, n, 2), dtype=torch.float32, device="cuda")
    fb = C.c_int64(0)
    for _ in range(2):
        ph = (C.c_double * 4)()
        rc = lib.mcf_fast_mm_phases(a.data_ptr(), b.data_ptr(), m, k, n, out.data_ptr(), ph, C.byref(fb), torch.cuda.current_stream().cuda_stream)
        assert rc == 0, lib.mcf_last_error()
    print(f"{name:28s} fallback outputs {fb.value:9d} ({100.0 * fb.value / (m * n):6.2f}%)  recon+fallback {ph[3]:8.3f} ms  total {sum(ph) - min(ph[0], ph[1]):8.3f} ms", flush=True)
