import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2207_08867_b200 as mcf
from paper_2207_08867_b200 import mlp
G = np.load("tests/golden/golden_mlp.npz")
dims = [int(d) for d in G["dims"]]; L = 3
params = [(G[f"w{l}"], G[f"b{l}"]) for l in range(L)]
m = mlp.MCMLP(dims, params, lr=0.0, plan=mcf.SEQUENTIAL)
xt = torch.from_numpy(np.ascontiguousarray(G["x"].T)).cuda(); y = torch.from_numpy(G["y"]).cuda()
n = xt.shape[1]
loss = m.step(xt, y, n); torch.cuda.synchronize()
B = m._bufs
# numpy forward
a = G["x"].astype(np.float64).T
for l in range(L):
    W = params[l][0].astype(np.float64).sum(-1); b = params[l][1].astype(np.float64).sum(-1)
    z = W @ a + b[:, None]
    h = B["H"][l].cpu().numpy()
    print("layer", l, "max |h_gpu - h_np|", np.abs(h - z).max(), "scale", np.abs(z).max())
    a = np.maximum(z, 0) if l < L - 1 else z
lg = a
mx = lg.max(0); e = np.exp(lg - mx); sm = e / e.sum(0)
terms = np.log(e.sum(0)) + mx - lg[G["y"], np.arange(n)]
print("loss np", terms.mean(), "gpu", loss.item(), "terms gpu", B["terms"].cpu().numpy()[:4], "np", terms[:4], "sum", B["loss"].item())
print("ref losses", G["losses"][:2])
