"""Single-batch and back-to-back (pipelined plan) times of BASELINE configs
3-5 on one GPU (device-resident inputs, CUDA events).
usage: python tools/configs_bench.py [K]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
res = {}
for name, (B, T, S) in {"c3": (32, 1024, 8192), "c4": (16, 4096, 16384),
                        "c5": (256, 512, 4096)}.items():
    q = m.generate_device(B, T, S, 0)
    outs = [torch.empty((B, T, S), dtype=torch.uint8, device="cuda") for _ in range(2)]
    row = {"shape": [B, T, S]}
    for mode, pipe in (("single_ms", False), ("pipelined_ms", True)):
        plan = m.Plan(B, T, S, pipelined=pipe)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for k in range(3):
                plan.enqueue(q, outs[k % 2], stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if pipe:
            e0.record(st)
            for k in range(K):
                plan.enqueue(q, outs[k % 2], stream=st)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
        else:
            ts = []
            for k in range(K):
                e0.record(st)
                plan.enqueue(q, outs[0], stream=st)
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
        row[mode] = round(ms, 4)
        row[mode.replace("_ms", "_gcells")] = round(B * T * S / ms / 1e6, 1)
        row["geometry"] = plan.geometry
        plan.close()
    ref = m.align(q)
    assert torch.equal(outs[0], ref)
    res[name] = row
    del q, outs, ref
    torch.cuda.empty_cache()
print(json.dumps(res))
