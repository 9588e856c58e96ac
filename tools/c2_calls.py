"""Per-call wall time at BASELINE config 2 (ragged B32 T200 S800), each call
followed by a device synchronise: plan.enqueue, align(check=False),
align(check=True).  usage: python tools/c2_calls.py [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from small_shapes_lengths import c2_lengths

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lens = c2_lengths()
q = m.generate_device(32, 200, 800, 0)
out = torch.empty((32, 200, 800), dtype=torch.uint8, device="cuda")
plan = m.Plan(32, 200, 800, lengths=lens)


def wall(fn):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e6)
    return round(float(np.median(ts)), 1)


res = {"plan_enqueue_sync_us": wall(lambda: plan.enqueue(q, out)),
       "align_nocheck_sync_us": wall(lambda: m.align(q, lengths=lens, check=False)),
       "align_checked_us": wall(lambda: m.align(q, lengths=lens)),
       "launches": plan.launches}
print(json.dumps(res))
