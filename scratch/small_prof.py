import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_07704_b200 as m
q = np.random.default_rng(0).uniform(-5,5,(32,200,800)).astype(np.float32)
for _ in range(5): m.align(q)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): m.align(q)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
