"""GaussianPlan enqueues at the c3 shape, C channels (for ncu launch lists /
captures).  usage: python tools/gauss_plan_run.py [C] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m

C = int(sys.argv[1]) if len(sys.argv) > 1 else 80
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
B, T, S = 32, 1024, 8192
g = torch.Generator().manual_seed(0)
z = torch.randn(B, C, S, generator=g).cuda()
mean = (torch.randn(B, C, T, generator=g) * 0.8).cuda()
ls = ((torch.rand(B, C, T, generator=g) - 0.5) * 0.6).cuda()
plan = m.GaussianPlan(B, C, T, S)
out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
for _ in range(n):
    plan.enqueue(z, mean, ls, out=out)
torch.cuda.synchronize()
