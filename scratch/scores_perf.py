import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2409_07704_b200 as mas
for (B,T,S) in [(32,1024,8192),(256,512,4096),(1,1024,8192)]:
    x = mas.generate_device(B,T,S,0)
    y = x.clone()
    for _ in range(3): y.copy_(x); mas.forward_parallel(y)
    e0,e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts=[]
    for _ in range(5):
        y.copy_(x); e0.record(); mas.forward_parallel(y); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms=min(ts); print(B,T,S, f"{ms:.3f} ms  {B*T*S/ms/1e6:.1f} Gcells/s  {8*B*T*S/ms/1e6:.0f} GB/s")
