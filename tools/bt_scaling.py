"""K2 (backtrack) time against the speech length at B32 T1024 and against
the text length at S8192: per-column and per-row (exit) costs of the walk.
usage: python tools/bt_scaling.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib

res = {}
shapes = [(1024, S) for S in (1024, 2048, 4096, 8192, 16384)] + [(T, 8192) for T in (128, 256, 512, 2048)]
for T, S in shapes:
    B = 32
    q = m.generate_device(B, T, S, 0)
    out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
    plan = m.Plan(B, T, S)
    plan.enqueue(q, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        plan.enqueue(q, out, parts=_lib.MAS_PART_FORWARD)
        e0.record()
        plan.enqueue(q, out, parts=_lib.MAS_PART_BACKTRACK)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res[f"T{T}_S{S}"] = round(ts[len(ts) // 2], 1)
    plan.close()
    del q, out
print(json.dumps({"bt_us": res}))
