import torch, time
n = 1 << 28  # 1 GiB of fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
hp = torch.empty(n, dtype=torch.float32)  # pageable
for name, src, dst in [("H2D pinned", h, d), ("D2H pinned", d, h), ("H2D pageable", hp, d), ("D2H pageable", d, hp)]:
    dst.copy_(src); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): dst.copy_(src)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name}: {4*n/dt/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda"); h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print("duplex 1GiB H2D + 256MiB D2H:", round((time.perf_counter()-t0)*1e3, 1), "ms")
import os; print("cpus", os.cpu_count())
