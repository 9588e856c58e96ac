import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib
lib = _lib.load(); cfg = m.api._make_config("parallel", -1e32, 0); err = _lib.MasError()
B,T,S = 32,200,800
qn = np.random.default_rng(0).uniform(-5,5,(B,T,S)).astype(np.float32)
on = np.empty((B,T,S), np.uint8)
qp = torch.from_numpy(qn).pin_memory(); op = torch.empty((B,T,S), dtype=torch.uint8).pin_memory()
def run(qptr, optr, chunks):
    os.environ["MAS_HOST_CHUNKS"] = str(chunks)
    ts=[]
    for _ in range(30):
        t0=time.perf_counter()
        rc = lib.mas_align_host(qptr, B, T, S, None, ctypes.byref(cfg), optr, None, ctypes.byref(err)); _lib.raise_for(rc, err)
        ts.append(time.perf_counter()-t0)
    ts.sort(); return ts[15]*1e6
print("pageable:", run(qn.ctypes.data, on.ctypes.data, 0))
print("pinned  :", run(qp.data_ptr(), op.data_ptr(), 0))
