import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib
B,T,S = 32,1024,8192
q = m.generate_device(B,T,S,0)
hq = torch.empty((B,T,S), dtype=torch.float32, pin_memory=True); hq.copy_(q)
hout = torch.empty((B,T,S), dtype=torch.uint8, pin_memory=True)
lib = _lib.load(); cfg = m.api._make_config("parallel", -1e32, 0); err = _lib.MasError()
def call():
    rc = lib.mas_align_host(hq.data_ptr(), B, T, S, None, ctypes.byref(cfg), hout.data_ptr(), None, ctypes.byref(err)); _lib.raise_for(rc, err)
for _ in range(2): call()
ts=[]
for _ in range(8):
    t0=time.perf_counter(); call(); ts.append(time.perf_counter()-t0)
ts.sort()
print(os.environ.get("MAS_HOST_CHUNKS","4"), "e2e min %.2f ms med %.2f ms -> %.2f Gcells/s" % (ts[0]*1e3, ts[4]*1e3, B*T*S/ts[4]/1e9))
