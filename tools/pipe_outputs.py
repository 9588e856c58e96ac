"""Back-to-back c3 batches writing only durations or only paths (no dense
output): the step without the 1 B/cell output stream."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B, T, S = 32, 1024, 8192
q = m.generate_device(B, T, S, 0)
durs = [torch.empty((B, T), dtype=torch.int32, device="cuda") for _ in range(2)]
paths = [torch.empty((B, S), dtype=torch.int32, device="cuda") for _ in range(2)]
res = {}
for name, kw in (("durations", lambda k: dict(durations=durs[k % 2])), ("paths", lambda k: dict(paths=paths[k % 2]))):
    for pipe in (False, True):
        plan = m.Plan(B, T, S, pipelined=pipe)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for k in range(5):
                plan.enqueue(q, stream=st, **kw(k))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for k in range(50):
            plan.enqueue(q, stream=st, **kw(k))
        e1.record(st)
        torch.cuda.synchronize()
        res[f"{name}_{'pipelined' if pipe else 'plain'}_ms"] = round(e0.elapsed_time(e1) / 50, 4)
        plan.close()
print(json.dumps(res))
