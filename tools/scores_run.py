"""forward_parallel (the K1 score export) on a c3-shaped device tensor, n
times (for ncu captures).  usage: python tools/scores_run.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
q = m.generate_device(32, 1024, 8192, 0)
for _ in range(n):
    m.forward_parallel(q)
torch.cuda.synchronize()
