"""Steady-state step of back-to-back c3 batches: plain plan vs pipelined plan
(batch i's backtrack overlapping batch i+1's forward)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B, T, S = 32, 1024, 8192
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
q = m.generate_device(B, T, S, 0)
outs = [torch.empty((B, T, S), dtype=torch.uint8, device="cuda") for _ in range(2)]
res = {}
for name, pipe in (("plain", False), ("pipelined", True)):
    plan = m.Plan(B, T, S, pipelined=pipe)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(5):
            plan.enqueue(q, outs[k % 2], stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(K):
        plan.enqueue(q, outs[k % 2], stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res[name] = {"ms_per_step": round(ms, 4), "gcells": round(B * T * S / ms / 1e6, 1)}
    res[name]["geometry"] = plan.geometry
    ref = m.align(q)
    assert torch.equal(outs[0], ref) and torch.equal(outs[1], ref), name
print(json.dumps(res))
