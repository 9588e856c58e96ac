import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib
B,T,S = 32,1024,8192
q = m.generate_device(B,T,S,0)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
paths = torch.empty((B,S), dtype=torch.int32, device='cuda')
dur = torch.empty((B,T), dtype=torch.int32, device='cuda')
plan = m.Plan(B,T,S)
for name, kw in [("out", dict(out=out)), ("paths", dict(paths=paths)), ("durations", dict(durations=dur)), ("all", dict(out=out, paths=paths, durations=dur))]:
    for _ in range(3): plan.enqueue(q, **kw)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(10):
        plan.enqueue(q, parts=_lib.MAS_PART_FORWARD, **kw)
        e[0].record(); plan.enqueue(q, parts=_lib.MAS_PART_BACKTRACK, **kw); e[1].record()
        torch.cuda.synchronize(); ts.append(e[0].elapsed_time(e[1]) * 1e3)
    ts.sort()
    print(f"bt with {name:10s}: min {ts[0]:.1f} med {ts[5]:.1f} us")
