"""The Gaussian log-likelihood on the tensor cores:
q from z / mean / logstd (csrc/mas_gauss.cu, tcgen05 with bf16 operands and
fp32 accumulation) against a float64 PyTorch restatement of
sum_c log N(z; mean, exp(logstd)), with the tolerance of its
bf16 operands written out, and -- tightly -- against the same expansion
evaluated in float64 on the bf16-rounded operands (checks the MMA
descriptors, layouts and accumulation, not the rounding)."""

from __future__ import annotations

import math

import pytest

pytestmark = pytest.mark.gpu


def _inputs(B, C, T, S, seed, device="cuda"):
    import torch

    g = torch.Generator(device="cpu").manual_seed(seed)
    z = torch.randn(B, C, S, generator=g).float()
    mean = torch.randn(B, C, T, generator=g).float() * 0.8
    logstd = (torch.rand(B, C, T, generator=g).float() - 0.5) * 0.6
    return z.to(device), mean.to(device), logstd.to(device)


def reference_q64(z, mean, logstd):
    """float64 sum_c log N(z[c, j]; mean[c, i], exp(logstd[c, i])), [B, T, S]."""
    z, m, ls = z.double(), mean.double(), logstd.double()
    diff = z[:, :, None, :] - m[:, :, :, None]                     # [B, C, T, S]
    lp = -0.5 * math.log(2 * math.pi) - ls[..., None] - 0.5 * diff * diff * torch_exp(-2 * ls)[..., None]
    return lp.sum(1)


def torch_exp(x):
    import torch

    return torch.exp(x)


def operands64(z, mean, logstd, bf16=True):
    """The expansion q = A . B + bias of csrc/mas_gauss.cu, A / B rounded to
    bf16 as the kernel rounds them (from fp32 values), in float64."""
    import torch

    inv = torch.exp(-2 * logstd)                                   # fp32, as the kernel
    A = torch.cat([-0.5 * inv, mean * inv], 1)                     # [B, 2C, T]
    Bm = torch.cat([z * z, z], 1)                                  # [B, 2C, S]
    if bf16:
        A, Bm = A.bfloat16(), Bm.bfloat16()
    A, Bm = A.double(), Bm.double()
    bias = (-0.91893853320467274 - logstd.double() - 0.5 * (mean * mean * inv).double()).sum(1)
    q = torch.einsum("bkt,bks->bts", A, Bm) + bias[:, :, None]
    mag = torch.einsum("bkt,bks->bts", A.abs(), Bm.abs())
    return q, mag


@pytest.mark.parametrize("shape", [(1, 80, 128, 32), (2, 80, 200, 777), (3, 17, 300, 95),
                                   (1, 192, 130, 260), (2, 1, 5, 3)])
def test_gaussian_loglik_values(mas, cuda, shape):
    import torch

    B, C, T, S = shape
    z, mean, logstd = _inputs(B, C, T, S, seed=sum(shape))
    q = mas.gaussian_loglik(z, mean, logstd)
    torch.cuda.synchronize()
    assert q.shape == (B, T, S) and q.dtype == torch.float32
    q64 = q.double()
    emul, mag = operands64(z, mean, logstd, bf16=True)
    # same operands, fp32 accumulation: a few ulps of the absolute sum
    err = (q64 - emul).abs()
    assert bool((err <= 2e-6 * mag + 1e-5 * emul.abs() + 1e-4).all()), float(err.max())
    # against the exact log-likelihood: the bf16 rounding of A and B
    # (2 x 2^-9 relative per product) over the absolute sum
    ref = reference_q64(z, mean, logstd)
    tol = 2.0 ** -7 * mag + 1e-4 * ref.abs() + 1e-3
    assert bool(((q64 - ref).abs() <= tol).all()), float(((q64 - ref).abs() - tol).max())


def test_gaussian_loglik_rejects_bad_inputs(mas, cuda):
    import torch

    z, mean, logstd = _inputs(1, 4, 6, 9, 0)
    with pytest.raises(ValueError):
        mas.gaussian_loglik(z.cpu(), mean, logstd)
    with pytest.raises(ValueError):
        mas.gaussian_loglik(z, mean, logstd[:, :, :5])
    z2, m2, l2 = _inputs(1, 193, 6, 9, 0)
    with pytest.raises(RuntimeError):
        mas.gaussian_loglik(z2, m2, l2)


def _unfused(mas, z, mean, logstd, lens, engine, want):
    q = mas.gaussian_loglik(z, mean, logstd)
    out = {}
    if "alignment" in want:
        out["alignment"] = mas.align(q, lengths=lens, engine=engine)
    if "paths" in want:
        ps = mas.align_paths(q, lengths=lens, engine=engine)
        out["paths"] = ps
    if "durations" in want:
        out["durations"] = mas.align_durations(q, lengths=lens, engine=engine)
    return q, out


@pytest.mark.parametrize("engine", ["parallel", "reference"])
@pytest.mark.parametrize("shape,ragged", [((2, 80, 200, 800), False), ((3, 80, 257, 1000), True),
                                          ((1, 192, 1024, 2048), False), ((4, 16, 37, 111), True),
                                          ((2, 80, 1024, 8192), False)])
def test_fused_equals_unfused(mas, cuda, shape, ragged, engine):
    """align_gaussian (q computed inside the forward kernel, never written)
    == align(gaussian_loglik(...)) bit for bit: same MMAs, same bias add."""
    import numpy as np
    import torch

    B, C, T, S = shape
    z, mean, logstd = _inputs(B, C, T, S, seed=B * T + S)
    lens = None
    if ragged:
        rng = np.random.default_rng(T)
        t = rng.integers(1, T + 1, B)
        t[0] = T
        s = np.maximum(t, rng.integers(1, S + 1, B))
        s[0] = S
        lens = np.stack([t, s], 1)
    want = ("alignment", "paths", "durations")
    got = mas.align_gaussian(z, mean, logstd, lengths=lens, engine=engine, outputs=want)
    q, exp = _unfused(mas, z, mean, logstd, lens, engine, want)
    assert torch.equal(got["alignment"], exp["alignment"])
    assert torch.equal(got["durations"], exp["durations"])
    for b in range(B):
        sb = S if lens is None else int(lens[b, 1])
        gp = got["paths"][b, :sb].cpu()
        ep = exp["paths"][b] if not hasattr(exp["paths"][b], "cpu") else exp["paths"][b].cpu()
        assert torch.equal(gp, torch.as_tensor(ep)), b
        assert bool((got["paths"][b, sb:] == -1).all())


def test_fused_alignment_is_near_optimal_for_exact_q(mas, cuda):
    """Against the exact (float64) log-likelihood the fused path -- optimal
    for the bf16-operand q -- scores within the q error of the exact optimum
    (the path sum of q errors bounds the loss), and mostly picks the same
    frames."""
    import numpy as np
    import torch

    B, C, T, S = 2, 80, 120, 500
    z, mean, logstd = _inputs(B, C, T, S, seed=11)
    got = mas.align_gaussian(z, mean, logstd, outputs=("paths",))["paths"].cpu().numpy()
    qx = reference_q64(z, mean, logstd).cpu().numpy()             # exact q
    qf = mas.gaussian_loglik(z, mean, logstd).double().cpu().numpy()
    exact_paths = np.stack([np.asarray(p) for p in mas.align_paths(qx.astype(np.float32))])
    cols = np.arange(S)
    for b in range(B):
        s_fused = qx[b, got[b], cols].sum()
        s_exact = qx[b, exact_paths[b], cols].sum()
        bound = np.abs(qf[b] - qx[b]).max() * 2 * S
        assert s_exact - s_fused <= bound + 1e-6 * abs(s_exact), (b, s_exact - s_fused, bound)
        assert (got[b] == exact_paths[b]).mean() > 0.5


def test_fused_nonfinite_is_located(mas, cuda):
    import torch

    z, mean, logstd = _inputs(3, 8, 40, 90, 4)
    z[1, 2, 17] = float("nan")  # column 17 of every row of item 1
    with pytest.raises(ValueError, match=r"item 1: non-finite likelihood at \(0, 17\)"):
        mas.align_gaussian(z, mean, logstd)


@pytest.mark.parametrize("engine", ["parallel", "reference"])
@pytest.mark.parametrize("mnv", [float("-inf"), -1e9, float("nan")])
def test_fused_unchecked_sentinels(mas, cuda, engine, mnv):
    """detail::align_unchecked sentinels through the fused path equal the
    unfused path on the same q (NaN: std::max semantics, parallel engine via
    the materialised score table)."""
    import torch

    z, mean, logstd = _inputs(3, 24, 90, 400, seed=21)
    got = mas.align_gaussian(z, mean, logstd, engine=engine, max_neg_val=mnv,
                             unchecked=True)["alignment"]
    q = mas.gaussian_loglik(z, mean, logstd)
    exp = mas._align_unchecked(q, engine=engine, max_neg_val=mnv)
    assert torch.equal(got, exp)


def test_fused_tall_text_falls_back_to_materialised_q(mas, cuda):
    """Texts taller than one cluster (> 4096 rows): align_gaussian still
    answers, through q materialised on the device."""
    import torch

    z, mean, logstd = _inputs(1, 16, 4200, 4300, seed=31)
    got = mas.align_gaussian(z, mean, logstd, outputs=("paths",))["paths"]
    exp = mas.align_paths(mas.gaussian_loglik(z, mean, logstd))
    assert torch.equal(got[0].cpu(), torch.as_tensor(exp[0]).cpu() if not hasattr(exp[0], "cpu")
                       else exp[0].cpu())


@pytest.mark.parametrize("engine", ["parallel", "reference"])
def test_gaussian_plan_reuse_and_graph(mas, cuda, engine):
    """GaussianPlan: enqueue-only, reused over batches and captured in a CUDA
    graph, equal to align_gaussian on every batch."""
    import numpy as np
    import torch

    B, C, T, S = 3, 80, 257, 1000
    rng = np.random.default_rng(5)
    t = rng.integers(1, T + 1, B)
    t[0] = T
    s = np.maximum(t, rng.integers(1, S + 1, B))
    lens = np.stack([t, s], 1)
    plan = mas.GaussianPlan(B, C, T, S, lengths=lens, engine=engine)
    out = torch.empty((B, T, S), dtype=torch.uint8, device="cuda")
    paths = torch.empty((B, S), dtype=torch.int32, device="cuda")
    dur = torch.empty((B, T), dtype=torch.int32, device="cuda")
    for seed in (1, 2, 3):
        z, mean, logstd = _inputs(B, C, T, S, seed=seed)
        plan.enqueue(z, mean, logstd, out=out, paths=paths, durations=dur)
        plan.finish()
        exp = mas.align_gaussian(z, mean, logstd, lengths=lens, engine=engine,
                                 outputs=("alignment", "paths", "durations"))
        assert torch.equal(out, exp["alignment"]) and torch.equal(dur, exp["durations"])
        for b in range(B):
            assert torch.equal(paths[b, :s[b]], exp["paths"][b, :s[b]])
    # graph capture: inputs updated in place between replays
    z, mean, logstd = _inputs(B, C, T, S, seed=7)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.enqueue(z, mean, logstd, out=out, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        plan.enqueue(z, mean, logstd, out=out, stream=st)
    for seed in (8, 9):
        z2, m2, l2 = _inputs(B, C, T, S, seed=seed)
        z.copy_(z2), mean.copy_(m2), logstd.copy_(l2)
        g.replay()
        torch.cuda.synchronize()
        exp = mas.align_gaussian(z, mean, logstd, lengths=lens, engine=engine)["alignment"]
        assert torch.equal(out, exp)
    plan.close()


def test_gaussian_plan_errors(mas, cuda):
    import torch

    z, mean, logstd = _inputs(3, 8, 40, 90, 4)
    plan = mas.GaussianPlan(3, 8, 40, 90)
    z[2, 1, 5] = float("inf")
    out = torch.empty((3, 40, 90), dtype=torch.uint8, device="cuda")
    plan.enqueue(z, mean, logstd, out=out)
    with pytest.raises(ValueError, match=r"item 2: non-finite likelihood at \(0, 5\)"):
        plan.finish()
    with pytest.raises(ValueError):
        plan.enqueue(z[:2], mean[:2], logstd[:2], out=out)
    # lengths are checked as align checks them: ranges at construction,
    # feasibility (t <= s) with the item's other errors at finish
    with pytest.raises(ValueError, match="item 1"):
        mas.GaussianPlan(2, 8, 40, 90, lengths=[[40, 90], [41, 90]])
    bad = mas.GaussianPlan(2, 8, 40, 90, lengths=[[40, 90], [30, 20]])
    bad.enqueue(*_inputs(2, 8, 40, 90, 5), out=out[:2])
    with pytest.raises(ValueError, match="item 1"):
        bad.finish()
    # shapes the fused kernel cannot take are refused, not silently materialised
    with pytest.raises((ValueError, RuntimeError)):
        mas.GaussianPlan(1, 16, 4200, 4300)
    with pytest.raises((ValueError, RuntimeError)):
        mas.GaussianPlan(1, 16, 40, 90, max_neg_val=float("nan"), unchecked=True)


def test_gaussian_plan_first_call_in_process(cuda):
    """The geometry choice's occupancy queries need the forward kernels'
    attributes set; a GaussianPlan (or align_gaussian) that is the process's
    first call must still find the fused geometry (regression: it used to be
    refused, and align_gaussian silently materialised q)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import paper_2409_07704_b200 as m; p = m.GaussianPlan(32, 80, 1024, 8192); "
            "p.close(); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
