"""Score export (forward_parallel / forward_reference on the device) timing:
K1's export path (aligned layout) vs the general kernel (text_cap % 4 != 0).
usage: python tools/scores_bench.py [B T S]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib

B, T, S = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 1024, 8192)
lib = _lib.load()
res = {"shape": [B, T, S]}
for name, t_cap in (("fwd4_export", T), ("general", T - 1)):
    q = m.generate_device(B, t_cap, S, 0)
    for engine, code in (("parallel", _lib.MAS_ENGINE_PARALLEL), ("reference", _lib.MAS_ENGINE_REFERENCE)):
        err = _lib.MasError()
        st = torch.cuda.current_stream().cuda_stream
        def run():
            rc = lib.mas_forward_scores_ex(q.data_ptr(), S, B, t_cap, S, None, code, -1e32,
                                           ctypes.c_void_p(st), ctypes.byref(err))
            _lib.raise_for(rc, err)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        e0.record()
        for _ in range(K):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        gbs = B * t_cap * S * 8 / ms / 1e6
        res[f"{name}_{engine}"] = {"ms": round(ms, 4), "GB/s": round(gbs, 1)}
print(json.dumps(res))
