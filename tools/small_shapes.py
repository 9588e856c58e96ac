"""Latency of the maximum-path call at small shapes (BASELINE configs 1, 2):
device step (plan.enqueue, CUDA events), align(torch cuda) and align(numpy)
wall times.  usage: python tools/small_shapes.py [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def c2_lengths():
    from oracle.oracle import Oracle  # the config's length recipe
    o = Oracle()
    st = o.mix_seed(2, 0)
    t, s = [], []
    M = (1 << 64) - 1
    def sm(x):
        x = (x + 0x9e3779b97f4a7c15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        return x, z ^ (z >> 31)
    for _ in range(32):
        st, r = sm(st); tb = 100 + r % 101
        st, r = sm(st); sb = min(800, 3 * tb + r % (tb + 1))
        t.append(tb); s.append(sb)
    return np.stack([t, s], 1)


res = {}
for name, (B, T, S, lens) in {"c1": (1, 64, 256, None), "c2": (32, 200, 800, c2_lengths())}.items():
    q = m.generate_device(B, T, S, 0)
    out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
    plan = m.Plan(B, T, S, lengths=lens)
    for _ in range(5):
        plan.enqueue(q, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); plan.enqueue(q, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    step = float(np.median(ts))
    # the same enqueue captured in a CUDA graph: device time without host launch cost
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        plan.enqueue(q, out, stream=gs)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=gs):
        plan.enqueue(q, out, stream=gs)
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    graph_us = float(np.median(ts))
    # device time per call: 20 replays back to back between the events, so
    # the host's graph submission (~7 us per replay) overlaps the device work
    ts = []
    for _ in range(max(5, reps // 10)):
        e0.record()
        for _ in range(20):
            graph.replay()
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 20)
    device_us = float(np.median(ts))
    for _ in range(5):
        m.align(q, lengths=lens)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); m.align(q, lengths=lens); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e6)
    torch_us = float(np.median(ts))
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); m.align(q, lengths=lens, check=False); ts.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    nocheck_us = float(np.median(ts))
    qn = q.cpu().numpy()
    for _ in range(3):
        m.align(qn, lengths=lens)
    ts = []
    for _ in range(max(5, reps // 5)):
        t0 = time.perf_counter(); m.align(qn, lengths=lens); ts.append((time.perf_counter() - t0) * 1e6)
    res[name] = {"shape": [B, T, S], "step_us": round(step, 1), "graph_replay_us": round(graph_us, 1), "device_us": round(device_us, 1), "align_torch_us": round(torch_us, 1), "align_torch_nocheck_enqueue_us": round(nocheck_us, 1),
                 "align_numpy_us": round(float(np.median(ts)), 1)}
print(json.dumps(res))
