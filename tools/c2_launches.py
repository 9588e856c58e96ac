"""Enqueue the c2 plan a few times (for an ncu launch list) and print its
geometry.  usage: python tools/c2_launches.py [c1|c2]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from small_shapes_lengths import c2_lengths

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
B, T, S, lens = (1, 64, 256, None) if which == "c1" else (32, 200, 800, c2_lengths())
q = m.generate_device(B, T, S, 0)
out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
plan = m.Plan(B, T, S, lengths=lens)
for _ in range(6):
    plan.enqueue(q, out)
torch.cuda.synchronize()
print(which, plan.geometry)
