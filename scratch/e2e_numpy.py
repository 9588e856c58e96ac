import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_07704_b200 as m
B,T,S = 32,1024,8192
q = m.generate_random_batch(B,T,S,0)   # numpy (pageable)
for _ in range(2): out = m.align(q)
ts=[]
for _ in range(5):
    t0=time.perf_counter(); out = m.align(q); ts.append(time.perf_counter()-t0)
ts.sort()
print("numpy align: med %.1f ms -> %.2f Gcells/s" % (ts[2]*1e3, B*T*S/ts[2]/1e9))
for _ in range(2): d = m.align_durations(q)
ts=[]
for _ in range(5):
    t0=time.perf_counter(); d = m.align_durations(q); ts.append(time.perf_counter()-t0)
ts.sort()
print("numpy align_durations: med %.1f ms -> %.2f Gcells/s" % (ts[2]*1e3, B*T*S/ts[2]/1e9))
