import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
for B,T,S in [(32,1024,8192),(64,512,8192)]:
    q = m.generate_device(B,T,S,0)
    out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
    plan = m.Plan(B,T,S)
    for _ in range(3): plan.enqueue(q, out)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): plan.enqueue(q, out)
    e1.record(); torch.cuda.synchronize()
    print(os.environ.get("MAS_LIB_PATH","default")[-12:], B,T,S, "%.1f us/step" % (e0.elapsed_time(e1)/5*1000))
    del q, out, plan
