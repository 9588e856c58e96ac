import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_07704_b200 as m
from oracle.oracle import Oracle
o = Oracle()
i = np.arange(32)[:, None]; j = np.arange(2048)[None, :]
q = np.where(i > j, np.float32(1e8), np.float32(-1e8)).astype(np.float32)
for eng in ("parallel", "reference"):
    for mnv in (-1e32, -1e9, float("-inf")):
        try:
            got = m._align_unchecked(q, engine=eng, max_neg_val=mnv)
            exp = o.align(q, engine=eng, max_neg_val=mnv, unchecked=True)[3][0]
            print(eng, mnv, "equal", np.array_equal(got, exp), flush=True)
        except Exception as e:
            print(eng, mnv, "ERROR", e, flush=True)
            raise
