"""Fused log-likelihood + MAS vs the unfused pipeline at B32 T1024 S8192
(BASELINE config 3 shape) with C channels (Glow-TTS: 80).  Prints one JSON
line.  usage: python tools/gauss_bench.py [C] [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_07704_b200 as m

C = int(sys.argv[1]) if len(sys.argv) > 1 else 80
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
B, T, S = 32, 1024, 8192
g = torch.Generator().manual_seed(0)
z = torch.randn(B, C, S, generator=g).cuda()
mean = (torch.randn(B, C, T, generator=g) * 0.8).cuda()
ls = ((torch.rand(B, C, T, generator=g) - 0.5) * 0.6).cuda()
plan = m.Plan(B, T, S)
out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")


def ev_time(fn, n):
    fn(); fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def unfused():
    q = m.gaussian_loglik(z, mean, ls)
    plan.enqueue(q, out)
    return q


gplan = m.GaussianPlan(B, C, T, S)
gout = torch.empty_like(out)


def fused():
    gplan.enqueue(z, mean, ls, out=gout)


def fused_checked():
    return m.align_gaussian(z, mean, ls)


# parity at this size (outside the timing)
q = unfused(); torch.cuda.synchronize()
a_unf = out.clone()
a_fus = fused_checked()["alignment"]
fused(); torch.cuda.synchronize()
assert torch.equal(a_unf, a_fus) and torch.equal(a_unf, gout), "fused != unfused"
del q
t_unf = ev_time(unfused, reps)
t_fus = ev_time(fused, reps)
t_chk = ev_time(fused_checked, reps)
t_q = ev_time(lambda: m.gaussian_loglik(z, mean, ls), reps)
qq = m.gaussian_loglik(z, mean, ls)
t_k12 = ev_time(lambda: plan.enqueue(qq, out), reps)
cells = B * T * S
kp = ((2 * C + 63) // 64) * 64
print(json.dumps({
    "shape": [B, C, T, S], "Kp": kp,
    "unfused_ms": round(t_unf, 4), "fused_ms": round(t_fus, 4),
    "align_gaussian_checked_ms": round(t_chk, 4),
    "gaussian_loglik_ms": round(t_q, 4), "align_on_q_ms": round(t_k12, 4),
    "unfused_gcells": round(cells / t_unf / 1e6, 1), "fused_gcells": round(cells / t_fus / 1e6, 1),
    "speedup": round(t_unf / t_fus, 3),
    "mma_tflops_fused": round(2 * kp * cells / (t_fus / 1e3) / 1e12, 1),
}))
