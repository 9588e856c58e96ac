import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B,T,S = 32,1024,8192
mode = sys.argv[1] if len(sys.argv)>1 else "out"
q = m.generate_device(B,T,S,0)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda') if mode=="out" else None
paths = torch.empty((B,S), dtype=torch.int32, device='cuda')
plan = m.Plan(B,T,S)
for _ in range(2): plan.enqueue(q, out, paths)
torch.cuda.synchronize()
