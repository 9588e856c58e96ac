import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib
B,T,S,pad = [int(x) for x in sys.argv[1:5]]
P = S + pad
q = m.generate_device(B,T,S,0,row_pitch=P)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
plan = m.Plan(B,T,S,row_pitch=P)
for _ in range(3): plan.enqueue(q, out)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
K = 10; f = b = 0.0
for _ in range(K):
    ev[0].record(); plan.enqueue(q, out, parts=_lib.MAS_PART_FORWARD); ev[1].record(); plan.enqueue(q, out, parts=_lib.MAS_PART_BACKTRACK); ev[2].record()
    torch.cuda.synchronize(); f += ev[0].elapsed_time(ev[1]); b += ev[1].elapsed_time(ev[2])
cells = B*T*S
print(f"pitch {P} {B}x{T}x{S}: fwd {f/K*1e3:.1f} us ({cells*5.125/(f/K)/1e6:.0f} GB/s), bt {b/K*1e3:.1f} us, step {(f+b)/K*1e3:.1f} us -> {cells/((f+b)/K)/1e6:.0f} Gcells/s")
