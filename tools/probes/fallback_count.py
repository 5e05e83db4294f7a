"""Outputs the tensor-core product hands to its cancellation fallback, and the
phase times, for an MC-MLP-like layer (W 1024 x 1024 nc=2, activations 1024 x 8192)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2207_08867_b200 as mcf
from paper_2207_08867_b200 import data
split = lambda v, nc, dt: data.split(v, nc)
lib=mcf.lib()
rng=np.random.default_rng(0)
m,k,n=1024,1024,8192
w=split(rng.uniform(-1/32,1/32,m*k),2,np.float32).reshape(m,k,2)
for name,a in (("relu(normal)",np.maximum(rng.normal(0,1,(k,n)),0).astype(np.float32)),("normal",rng.normal(0,1,(k,n)).astype(np.float32)),("uniform",rng.uniform(-1,1,(k,n)).astype(np.float32))):
    x=torch.from_numpy(w).cuda(); b=torch.from_numpy(a).cuda(); out=torch.empty((m,n,2),dtype=torch.float32,device="cuda")
    fb=C.c_int64(0)
    for _ in range(3):
        ph=(C.c_double*4)(); rc=lib.mcf_fast_mm_phases(x.data_ptr(),b.data_ptr(),m,k,n,out.data_ptr(),ph,C.byref(fb),torch.cuda.current_stream().cuda_stream)
    print(name, "phases", [round(v,4) for v in ph], "fallback outputs", fb.value, f"{fb.value/(m*n)*100:.3f}%")
