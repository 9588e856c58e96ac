"""Runs align_gaussian at B32 T1024 S8192 C (argv) a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
C = int(sys.argv[1]) if len(sys.argv) > 1 else 80
B, T, S = 32, 1024, 8192
g = torch.Generator().manual_seed(0)
z = torch.randn(B, C, S, generator=g).cuda()
mean = (torch.randn(B, C, T, generator=g) * 0.8).cuda()
ls = ((torch.rand(B, C, T, generator=g) - 0.5) * 0.6).cuda()
for _ in range(3):
    m.align_gaussian(z, mean, ls)
torch.cuda.synchronize()
