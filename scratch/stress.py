"""Randomised parity sweep (one-off validation, not part of the suite):
random shapes, ragged lengths, both engines, sentinels, host (numpy,
pageable) and device (torch) entry points, forced bands; every result
checked against the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m
from oracle.oracle import Oracle
o = Oracle()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
deadline = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 240)
n = bad = 0
while time.time() < deadline:
    B = int(rng.integers(1, 9))
    T = int(rng.choice([rng.integers(1, 80), rng.integers(1, 700), rng.integers(500, 2600)]))
    S = T + int(rng.integers(0, 3 * T + 64))
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    if rng.random() < 0.3:
        q = np.round(q)  # many ties
    lens = None
    if rng.random() < 0.6:
        lt = rng.integers(1, T + 1, B)
        ls = np.array([int(rng.integers(a, S + 1)) for a in lt])
        lens = np.stack([lt, ls], 1)
        for b in range(B):
            q[b, lt[b]:, :] = np.nan
            q[b, :, ls[b]:] = np.nan
    eng = "reference" if rng.random() < 0.4 else "parallel"
    exp = o.align(q, lens, engine=eng)[3]
    if rng.random() < 0.5:
        got = m.align(q, lengths=lens, engine=eng)
    else:
        got = m.align(torch.from_numpy(q).cuda(), lengths=lens, engine=eng).cpu().numpy()
    n += 1
    if not np.array_equal(got, exp):
        bad += 1
        print("MISMATCH", B, T, S, eng, lens is not None, int((got != exp).sum()), flush=True)
    d = m.align_durations(q, lengths=lens, engine=eng)
    if not np.array_equal(d, exp.sum(axis=2).astype(np.int32)):
        bad += 1
        print("DUR MISMATCH", B, T, S, eng, flush=True)
print(f"{n} cases, {bad} mismatches")
