import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
cfgs=[(32,64,8192),(128,64,8192),(512,64,8192),(32,256,8192),(32,1024,8192),(64,512,8192)]
for B,T,S in cfgs:
    q = m.generate_device(B,T,S,0)
    out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
    plan = m.Plan(B,T,S)
    for _ in range(2): plan.enqueue(q, out)
    torch.cuda.synchronize()
    del q, out, plan
