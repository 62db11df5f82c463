import torch, time
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"torch fp64 matmul {n}: {2*n**3/best/1e9:.2f} TFLOP/s")
# small batched
for n, bs in ((64, 4096), (128, 4096), (384, 1024)):
    a = torch.randn(bs, n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ a
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ a; e1.record(); torch.cuda.synchronize()
    print(f"torch fp64 bmm n={n} bs={bs}: {2*bs*n**3/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s")
a = torch.empty(2**28, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
print(f"copy {2*a.numel()*8/e0.elapsed_time(e1)/1e6:.1f} GB/s")
