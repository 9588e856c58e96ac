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
# ragged + paths
bad=0
for k in range(30):
    B=int(rng.integers(1,6)); T=int(rng.integers(1,200)); S=int(rng.integers(T,700))
    q = rng.uniform(-5,5,(B,T,S)).astype(np.float32)
    lt = rng.integers(1, T+1, B); ls = np.array([rng.integers(a, S+1) for a in lt])
    lens = np.stack([lt, ls], 1)
    for eng in ("parallel","reference"):
        got = m.align(q, lengths=lens, engine=eng)
        gp = m.align_paths(q, lengths=lens, engine=eng)
        _,_,_,exp,ep = o.align(q, lengths=lens, engine=eng)
        ok = np.array_equal(got, exp) and all(np.array_equal(gp[i], ep[i,:ls[i]]) for i in range(B))
        bad += not ok
print("ragged mismatches", bad)
q = rng.uniform(-5,5,(3,40,100)).astype(np.float32); q[1,5,7]=np.nan; q[2,0,0]=np.inf
try:
    m.align(q); print("NO ERROR?!")
except ValueError as e: print("ValueError:", e)
