import sys, torch
sys.path.insert(0, '.')
import paper_2409_07704_b200 as mas
B,T,S = (int(a) for a in sys.argv[1:4])
x = mas.generate_device(B,T,S,0)
for _ in range(2): mas.forward_parallel(x.clone())
torch.cuda.synchronize()
