import torch, time, json
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
res = {}
for name, nst in (("one_stream", 1), ("two_streams", 2), ("four_streams", 4)):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    chunk = n // nst
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, st in enumerate(sts):
            with torch.cuda.stream(st):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    res[name] = round(n * 4 / dt / 1e9, 1)
# D2H concurrently with H2D
h2 = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
res["h2d_with_d2h_GBs"] = round(n * 4 / dt / 1e9, 1)
print(json.dumps(res))
