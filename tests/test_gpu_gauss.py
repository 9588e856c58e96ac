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
