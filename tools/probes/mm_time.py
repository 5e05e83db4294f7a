"""Quick device timing of the MC contractions (configs 1, 2, 4 shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_08867_b200 as mcf  # noqa: E402


def timeit(f, reps=5):
    for _ in range(2):
        f()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


sel = sys.argv[1:]
g = torch.Generator(device="cuda").manual_seed(0)
if not sel or "mm" in sel:
    M = K = N = 4096
    x = (torch.rand(M, K, 2, device="cuda", generator=g) * 2 - 1).float()
    x[..., 1] *= 2.0**-25
    w = (torch.rand(K, N, device="cuda", generator=g) * 2 - 1).float()
    ms = timeit(lambda: mcf.mm_mcn(x, w, plan=mcf.FAST))
    print(f"mm MCxT nc=2 4096^3 FAST: {ms:.2f} ms  {2*M*N*K/ms/1e9:.1f} GFLOP/s(eff)  "
          f"{9*M*N*K/ms/1e9/1e3:.2f} T FP64-op/s", flush=True)
    if "exact" in sel:
        ms = timeit(lambda: mcf.mm_mcn(x[:512], w), reps=2)
        print(f"mm MCxT nc=2 512x4096x4096 exact: {ms:.2f} ms  {2*512*N*K/ms/1e9:.1f} GFLOP/s(eff)", flush=True)
if not sel or "mv" in sel:
    M, K = 65536, 4096
    x = (torch.rand(M, K, 3, device="cuda", generator=g) * 2 - 1).float()
    x[..., 1] *= 2.0**-25
    x[..., 2] *= 2.0**-50
    v = (torch.rand(K, device="cuda", generator=g) * 2 - 1).float()
    ms = timeit(lambda: mcf.mv_mcn(x, v, plan=mcf.FAST))
    gb = (M * K * 12 + K * 4 + M * 12) / ms / 1e6
    print(f"mv MCxT nc=3 65536x4096 FAST: {ms:.3f} ms  {gb:.0f} GB/s  {gb/6446.6:.3f} of HBM", flush=True)
    del x
if not sel or "dot" in sel:
    B, K = 65536, 4096
    x = (torch.rand(B, K, 3, device="cuda", generator=g) * 2 - 1).float()
    y = (torch.rand(B, K, 3, device="cuda", generator=g) * 2 - 1).float()
    x[..., 1:] *= 2.0**-25
    y[..., 1:] *= 2.0**-25
    ms = timeit(lambda: mcf.dot_mcmc(x, y, plan=mcf.FAST))
    gb = (B * K * 24 + B * 12) / ms / 1e6
    print(f"dot MCxMC nc=3 65536x4096 FAST: {ms:.3f} ms  {gb:.0f} GB/s  {gb/6446.6:.3f} of HBM", flush=True)
    del x, y
if not sel or "mcmc" in sel:
    M = K = N = 8192
    x = (torch.rand(M, K, 2, device="cuda", generator=g) * 2 - 1).float()
    y = (torch.rand(K, N, 2, device="cuda", generator=g) * 2 - 1).float()
    x[..., 1] *= 2.0**-25
    y[..., 1] *= 2.0**-25
    ms = timeit(lambda: mcf.mm_mcmc(x, y, plan=mcf.FAST), reps=3)
    print(f"mm MCxMC fp32 nc=2 8192^3 FAST: {ms:.2f} ms  {2*M*N*K/ms/1e9:.1f} GFLOP/s(eff)", flush=True)
    del x, y
    xh = ((torch.rand(M, K, 3, device="cuda", generator=g) * 2 - 1) / 64).half()
    yh = ((torch.rand(K, N, 3, device="cuda", generator=g) * 2 - 1) / 64).half()
    xh[..., 1:] = 0
    yh[..., 1:] = 0
    ms = timeit(lambda: mcf.mm_mcmc(xh, yh, plan=mcf.FAST), reps=3)
    print(f"mm MCxMC fp16 nc=3 8192^3 FAST: {ms:.2f} ms  {2*M*N*K/ms/1e9:.1f} GFLOP/s(eff)", flush=True)
