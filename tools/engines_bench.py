"""c3 step time of both engines, plain and pipelined plans."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2409_07704_b200 as m
B, T, S = 32, 1024, 8192
q = m.generate_device(B, T, S, 0)
outs = [torch.empty((B, T, S), dtype=torch.uint8, device="cuda") for _ in range(2)]
res = {}
for eng in ("parallel", "reference"):
    for pipe in (False, True):
        plan = m.Plan(B, T, S, engine=eng, pipelined=pipe)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for k in range(4):
                plan.enqueue(q, outs[k % 2], stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(40):
            plan.enqueue(q, outs[k % 2], stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        res[f"{eng}_{'pipelined' if pipe else 'plain'}_ms"] = round(e0.elapsed_time(e1) / 40, 4)
        plan.close()
print(json.dumps(res))
