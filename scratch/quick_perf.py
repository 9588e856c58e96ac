import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
B,T,S = [int(x) for x in (sys.argv[1:4] if len(sys.argv)>3 else (32,1024,8192))]
q = m.generate_device(B,T,S,0)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
plan = m.Plan(B,T,S)
print("geometry", plan.geometry)
for _ in range(3): plan.enqueue(q, out)
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
K=10
e0.record()
for _ in range(K): plan.enqueue(q, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/K
cells=B*T*S
print(f"{B}x{T}x{S}: {ms:.3f} ms/step  {cells/ms/1e6:.1f} Gcells/s  {cells*5.125/ms/1e6:.1f} GB/s")
plan.finish(q)
