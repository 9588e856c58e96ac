"""Host-side cost of one align(torch cuda) call at BASELINE config 2 shape:
the Python layer vs the C-ABI call (enqueue only, check=False)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib, api

B, T, S = 32, 200, 800
q = m.generate_device(B, T, S, 0)
lens = np.stack([np.full(B, 150), np.full(B, 700)], 1)
N = 200


def med(fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(N):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    return round(float(np.median(ts)) * 1e6, 1)


res = {"align_check_false_us": med(lambda: m.align(q, lengths=lens, check=False)),
       "align_checked_us": med(lambda: m.align(q, lengths=lens))}
res["prepare_us"] = med(lambda: api._prepare(q, lens, "parallel", -1e32, 0, False))
lib = _lib.load()
values, lns, cfg, was_2d, b, t, s = api._prepare(q, lens, "parallel", -1e32, 0, False)
cfg.flags |= _lib.MAS_FLAG_NO_CHECK
out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
err = _lib.MasError()
st = torch.cuda.current_stream().cuda_stream
lp = lns.ctypes.data


def raw():
    lib.mas_align_device_ex(q.data_ptr(), S, B, T, S, lp, ctypes.byref(cfg), out.data_ptr(), None,
                            None, ctypes.c_void_p(st), ctypes.byref(err))


res["raw_cabi_us"] = med(raw)
res["torch_empty_us"] = med(lambda: torch.empty((B, T, S), dtype=torch.uint8, device="cuda"))
print(json.dumps(res))
