"""Device time of the forward kernel alone and of forward + backtrack at
small shapes (CUDA-graph replay, warm L2), to split fixed from per-column
cost.  usage: python tools/small_parts.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib


def graph_us(fn, reps=200):
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        fn(gs)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        fn(gs)
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return round(float(np.median(ts)), 2)


res = {}
for B, T, S in [(1, 64, 32), (1, 64, 256), (1, 64, 1024), (32, 200, 32), (32, 200, 256), (32, 200, 800),
                (32, 200, 1600)]:
    q = m.generate_device(B, T, S, 0)
    out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
    plan = m.Plan(B, T, S)
    fwd = graph_us(lambda st: plan.enqueue(q, out, stream=st, parts=_lib.MAS_PART_FORWARD))
    both = graph_us(lambda st: plan.enqueue(q, out, stream=st))
    bt = graph_us(lambda st: plan.enqueue(q, out, stream=st, parts=_lib.MAS_PART_BACKTRACK))
    empty = graph_us(lambda st: torch.cuda._sleep(0))
    res[f"{B}x{T}x{S}"] = {"fwd": fwd, "bt": bt, "both": both, "empty_graph": empty}
print(json.dumps(res))
