import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B,T,S = [int(x) for x in (sys.argv[1:4] if len(sys.argv)>3 else (32,1024,8192))]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
q = m.generate_device(B,T,S,0)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
plan = m.Plan(B,T,S)
for _ in range(reps): plan.enqueue(q, out)
torch.cuda.synchronize()
