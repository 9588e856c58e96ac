import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_07704_b200 as m
for (B,T,S) in [(1,64,256),(32,200,800),(32,1024,8192)]:
    q = torch.from_numpy(np.random.default_rng(0).uniform(-5,5,(B,T,S)).astype(np.float32)).cuda()
    lens = np.stack([np.full(B, T), np.full(B, S)], 1)
    for _ in range(5): m.align(q, lengths=lens)
    torch.cuda.synchronize()
    ts=[]
    for _ in range(30):
        t0=time.perf_counter(); o = m.align(q, lengths=lens); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    ts.sort()
    print(f"align(torch cuda) {B}x{T}x{S}: median {ts[15]*1e6:.0f} us")
