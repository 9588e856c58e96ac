import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_07704_b200 as m
from oracle.oracle import Oracle
o = Oracle()
shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]] or [(2,128,512),(1,64,300),(2,300,2000),(2,1024,8192)]
for B,T,S in shapes:
    q = o.generate(B,T,S,7)
    exp_out, exp_p = o.align(q)[3:5]
    try:
        got = m.align_paths(q)
    except Exception as e:
        print(B,T,S,"ERROR",e); break
    for b in range(B):
        d = np.nonzero(got[b] != exp_p[b])[0]
        print(B,T,S,"item",b,"mismatch cols",len(d), d[:5].tolist(), d[-5:].tolist() if len(d) else "", 
              (got[b][d[:3]].tolist(), exp_p[b][d[:3]].tolist()) if len(d) else "")
