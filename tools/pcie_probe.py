import torch, time
x = torch.empty(80_000_000, dtype=torch.float64, device="cuda")
h = torch.empty(80_000_000, dtype=torch.float64, pin_memory=True)
for i in range(4):
    torch.cuda.synchronize(); t=time.perf_counter(); h.copy_(x, non_blocking=True); torch.cuda.synchronize(); t1=time.perf_counter()
    x.copy_(h, non_blocking=True); torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"D2H 640MB {1e3*(t1-t):.2f} ms ({0.64/(t1-t):.1f} GB/s)  H2D {1e3*(t2-t1):.2f} ms ({0.64/(t2-t1):.1f} GB/s)")
