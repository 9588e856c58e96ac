"""A/B timing of K1+K2 for several library builds, interleaved (A B A B ...),
min and median over rounds; SM clock sampled via NVML.
usage: python tools/ab.py B T S lib1 lib2 ..."""
import sys, os, subprocess, json
B, T, S = sys.argv[1:4]
libs = sys.argv[4:]
code = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2409_07704_b200 as m
from paper_2409_07704_b200 import _lib
B,T,S = %s,%s,%s
q = m.generate_device(B,T,S,0)
out = torch.empty((B,T,S), dtype=torch.uint8, device='cuda')
plan = m.Plan(B,T,S)
for _ in range(3): plan.enqueue(q, out)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fs=[]; bs=[]
for _ in range(15):
    e[0].record(); plan.enqueue(q, out, parts=_lib.MAS_PART_FORWARD); e[1].record(); plan.enqueue(q, out, parts=_lib.MAS_PART_BACKTRACK); e[2].record()
    torch.cuda.synchronize(); fs.append(e[0].elapsed_time(e[1])*1e3); bs.append(e[1].elapsed_time(e[2])*1e3)
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
fs.sort(); bs.sort()
print(json.dumps({"fwd_min": fs[0], "fwd_med": fs[len(fs)//2], "bt_med": bs[len(bs)//2], "clk": clk}))
''' % (B, T, S)
res = {l: [] for l in libs}
for rnd in range(3):
    for l in libs:
        env = dict(os.environ, MAS_LIB_PATH=l)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
        try:
            res[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
        except Exception:
            print(l, r.stderr[-500:])
for l in libs:
    rs = res[l]
    print(f"{l:60s} fwd min {min(x['fwd_min'] for x in rs):7.1f}  med {sorted(x['fwd_med'] for x in rs)[len(rs)//2]:7.1f}  bt {rs[0]['bt_med']:5.1f}  clk {[x['clk'] for x in rs]}")
