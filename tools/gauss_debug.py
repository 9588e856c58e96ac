import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B, C, T, S = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (1, 16, 128, 64)
g = torch.Generator().manual_seed(0)
z = torch.randn(B, C, S, generator=g).cuda()
mean = torch.randn(B, C, T, generator=g).cuda()
ls = ((torch.rand(B, C, T, generator=g) - 0.5) * 0.6).cuda()
r = m.align_gaussian(z, mean, ls, outputs=("alignment",))
q = m.gaussian_loglik(z, mean, ls)
e = m.align(q)
print("equal", torch.equal(r["alignment"], e))
