import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Oracle
import paper_2409_07704_b200 as m
o = Oracle()
q = np.array([[1,2,3],[4,5,6]], np.float32)
print("KAT", m.align(q).tolist(), m.align_paths(q).tolist())
print("zeros", m.align_paths(np.zeros((2,3,5),np.float32)))
rng = np.random.default_rng(0)
bad = 0; n = 0
for k in range(60):
    B = int(rng.integers(1, 4)); t = int(rng.integers(1, 300)); s = int(rng.integers(t, 900))
    q = rng.uniform(-5, 5, (B, t, s)).astype(np.float32)
    for eng in ("parallel", "reference"):
        got = m.align(q, engine=eng)
        _, _, _, exp, _ = o.align(q, engine=eng)
        n += 1
        if not np.array_equal(got, exp):
            bad += 1
            print("MISMATCH", B, t, s, eng, np.argwhere(got != exp)[:5])
print("random mismatches", bad, "of", n)
for (B,T,S) in [(4,1024,2048),(2,700,3000),(1,2000,4100)]:
    q = rng.uniform(-5,5,(B,T,S)).astype(np.float32)
    t0=time.time(); got = m.align(q); t1=time.time()
    _,_,_,exp,_ = o.align(q)
    print(B,T,S, "equal", np.array_equal(got,exp), "gpu s", round(t1-t0,3))
