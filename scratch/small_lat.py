import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_07704_b200 as m
for (B,T,S) in [(1,64,256),(32,200,800),(4,128,512)]:
    q = np.random.default_rng(0).uniform(-5,5,(B,T,S)).astype(np.float32)
    for _ in range(5): m.align(q)
    ts=[]
    for _ in range(50):
        t0=time.perf_counter(); m.align(q); ts.append(time.perf_counter()-t0)
    ts.sort()
    print(f"align(numpy) {B}x{T}x{S}: median {ts[25]*1e6:.0f} us, min {ts[0]*1e6:.0f} us")
