"""Small invocations of every device entry point, for compute-sanitizer
(memcheck / synccheck).  usage:
  compute-sanitizer --tool memcheck python tools/sanitize_run.py

Text heights avoid 129..256 rows: that geometry is a one-CTA cluster of two
compute warps whose FIFO hand-off is an st.async to the CTA's own shared
memory, which compute-sanitizer 12.9 reports as invalid ("Cluster needs to
have at least 2 blocks") although the hardware executes it (every parity
test at those heights is bit-exact).  Texts of <= 128 rows (one warp) and
>= 257 rows (clusters of >= 2 CTAs) run the same code paths sanitizer-clean."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2409_07704_b200 as m

torch.manual_seed(0)
# align: ragged, both engines, a banded shape
q = m.generate_device(4, 300, 600, 1)
lens = np.array([[300, 600], [37, 100], [250, 599], [1, 1]])
for eng in ("parallel", "reference"):
    m.align(q, lengths=lens, engine=eng)
    m.align_paths(q, lengths=lens, engine=eng)
    m.align_durations(q, lengths=lens, engine=eng)
m.align(m.generate_device(2, 64, 256, 3))  # one warp per item (one-launch tail)
# one-launch tail with rows past the CTA's 128 (text_cap 131, longest text 120)
qg = m.generate_device(2, 131, 300, 5)
m.align(qg, lengths=np.array([[120, 300], [5, 50]]))
qs = m.generate_device(3, 120, 300, 4)      # one-launch tail, ragged, every output
ls = np.array([[120, 300], [7, 40], [100, 100]])
for eng in ("parallel", "reference"):
    m.align(qs, lengths=ls, engine=eng)
    m.align_paths(qs, lengths=ls, engine=eng)
    m.align_durations(qs, lengths=ls, engine=eng)
bands = os.environ.get("MAS_SANITIZE_NO_BANDS") != "1"
if bands:
    qt = m.generate_device(1, 4500, 4600, 2)
    m.align(qt)
# pipelined plan, two batches
plan = m.Plan(4, 300, 600, pipelined=True)
o1 = torch.empty((4, 300, 600), dtype=torch.uint8, device="cuda")
o2 = torch.empty_like(o1)
plan.enqueue(q, o1)
plan.enqueue(q, o2)
torch.cuda.synchronize()
plan.close()
# score export: K1 path (aligned), bands, general kernel (text_cap % 4 != 0), reference mode
# (the general kernel, text_cap % 4 != 0, hands rows between warps through
# volatile counters racecheck does not model)
general = os.environ.get("MAS_SANITIZE_NO_GENERAL") != "1"
for shape in ((3, 264, 260), (2, 64, 100)) + (((2, 131, 257),) if general else ()) + \
        (((1, 9000, 96),) if bands else ()):
    v = torch.randn(*shape, device="cuda")
    m.forward_parallel(v)
torch.cuda.synchronize()
if os.environ.get("MAS_SANITIZE_NO_GAUSS") == "1":
    torch.cuda.synchronize()
    print("sanitize_run ok")
    sys.exit(0)
# gaussian: plan + checked call
B, C, T, S = 2, 80, 300, 700
z = torch.randn(B, C, S, device="cuda")
mu = torch.randn(B, C, T, device="cuda") * 0.5
ls = (torch.rand(B, C, T, device="cuda") - 0.5) * 0.4
gp = m.GaussianPlan(B, C, T, S)
out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
gp.enqueue(z, mu, ls, out=out)
gp.finish()
gp.close()
m.align_gaussian(z, mu, ls, outputs=("alignment", "paths", "durations"))
m.gaussian_loglik(z, mu, ls)
torch.cuda.synchronize()
print("sanitize_run ok")
