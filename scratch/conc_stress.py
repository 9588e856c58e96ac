import sys, os, threading, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_07704_b200 as m
from oracle.oracle import Oracle
o = Oracle()
rng = np.random.default_rng(8)
qs = [rng.uniform(-5, 5, (2, 100 + 50 * k, 700)).astype(np.float32) for k in range(4)]
exps = [o.align(q)[3] for q in qs]
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    res = [None] * 4; errs = [None] * 4
    def work(k):
        try: res[k] = m.align(qs[k])
        except Exception as e: errs[k] = traceback.format_exc()
    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th: t.start()
    for t in th: t.join()
    for k in range(4):
        if errs[k]: print("iter", it, "thread", k, "EXC", errs[k][-300:]); bad += 1
        elif not np.array_equal(res[k], exps[k]):
            d = np.argwhere(res[k] != exps[k]); print("iter", it, "thread", k, "MISMATCH", len(d), d[:3].tolist()); bad += 1
print("bad", bad)
