"""BASELINE config 2's ragged lengths (SURVEY 8d recipe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def c2_lengths():
    from oracle.oracle import Oracle  # the config's length recipe
    o = Oracle()
    st = o.mix_seed(2, 0)
    t, s = [], []
    M = (1 << 64) - 1
    def sm(x):
        x = (x + 0x9e3779b97f4a7c15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        return x, z ^ (z >> 31)
    for _ in range(32):
        st, r = sm(st); tb = 100 + r % 101
        st, r = sm(st); sb = min(800, 3 * tb + r % (tb + 1))
        t.append(tb); s.append(sb)
    return np.stack([t, s], 1)
