"""align(numpy) wall time at a few large shapes (pageable input: the host staging path)."""
import sys, time, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2409_07704_b200 as m
res = {}
for (B, T, S) in ((32, 1024, 8192), (8, 1024, 4096), (16, 1024, 4096)):
    q = m.generate_device(B, T, S, 0).cpu().numpy()
    m.align(q); m.align(q)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); m.align(q); ts.append(time.perf_counter() - t0)
    res[f"{B}x{T}x{S}"] = round(sorted(ts)[2] * 1e3, 2)
print(json.dumps(res))
