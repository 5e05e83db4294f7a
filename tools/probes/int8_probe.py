import torch, time
print(torch.cuda.get_device_name())
for K in [4096, 4096*4, 4096*12]:
    a = torch.randint(-127, 128, (4096, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (K, 4096), dtype=torch.int8, device="cuda")
    bt = b.t().contiguous().t()  # column-major
    for name, bb in (("rowmajorB", b), ("colmajorB", bt)):
        try:
            c = torch._int_mm(a, bb); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): c = torch._int_mm(a, bb)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(K, name, f"{ms:.3f} ms", f"{2*4096*4096*K/ms/1e9:.0f} GOPS")
        except Exception as ex:
            print(K, name, "ERR", str(ex)[:200])
# check exactness
a = torch.randint(-127, 128, (256, 4096*12), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (4096*12, 256), dtype=torch.int8, device="cuda")
c = torch._int_mm(a, b.t().contiguous().t())
ref = (a.double() @ b.double())
print("exact:", bool((c.double() == ref).all()))
