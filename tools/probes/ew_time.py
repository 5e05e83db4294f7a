"""Quick device timing of the elementwise suite (config 0: fp32 nc=2, 2^24)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2207_08867_b200 as mcf

def split2(v):
    c0 = v.astype(np.float32); c1 = (v - c0.astype(np.float64)).astype(np.float32)
    return np.stack([c0, c1], -1)

n = 1 << 24
rng = np.random.default_rng(0)
cv = lambda: rng.uniform(-1, 1, n) * np.exp2(rng.uniform(-8, 8, n))
x = torch.from_numpy(split2(cv())).cuda()
yv = cv(); y = torch.from_numpy(split2(yv)).cuda()
yd = torch.from_numpy(split2(yv + np.sign(yv) * 0.5)).cuda()
v = torch.from_numpy(cv().astype(np.float32)).cuda()
xe = torch.from_numpy(split2(np.clip(cv(), -10, 10))).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ops = {
  "grow_expn": (lambda: mcf.grow_expn(x, v), 20), "scaling_n": (lambda: mcf.scaling_n(x, v), 20),
  "div_n": (lambda: mcf.div_n(v, yd), 20), "add_mcn": (lambda: mcf.add_mcn(x, y), 24),
  "mul_mcn": (lambda: mcf.mul_mcn(x, yd), 24), "div_mcn": (lambda: mcf.div_mcn(x, yd), 24),
  "exp_mcn": (lambda: mcf.exp_mcn(xe), 16), "square_mcn": (lambda: mcf.square_mcn(x), 16),
  "mul_mcn_slow": (lambda: mcf.mul_mcn_slow(x, y), 24),
}
res = {}
sel = sys.argv[1:]
for name, (f, bpe) in ops.items():
    if sel and name not in sel: continue
    for _ in range(3): f()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    res[name] = dict(ms=round(t, 4), GBps=round(bpe * n / t / 1e6, 1), frac=round(bpe * n / t / 1e6 / 6446.6, 3))
    print(f"{name:14s} {t*1e3:9.1f} us  {bpe*n/t/1e6:8.1f} GB/s  {bpe*n/t/1e6/6446.6:6.3f} of HBM", flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/ew_time.json", "w"), indent=1)
