"""Score-table export: forward_parallel on the GPU
(csrc/mas_scores.cu through mas_forward_scores) against the reference's
parallel::forward_parallel (oracle/_ref, parallel.cpp:95-108) and the C
restatement (oracle/mas_oracle.c), bit for bit -- every cell of every item,
signed zeros included.  Cases follow test_parallel.cpp:44-103."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_reference_examples(mas, cuda):
    # test_parallel.cpp:44-52 -- the 2x3 example
    q = np.arange(1, 7, dtype=np.float32).reshape(2, 3)
    mas.forward_parallel(q)
    assert q[0].tolist() == [1.0, 3.0, 6.0]
    assert q[1, 0] <= -1e30 and q[1, 1] == 6.0 and q[1, 2] == 12.0
    # :54-62 -- an all-zero feasible region stays zero
    z = np.zeros((3, 5), np.float32)
    mas.forward_parallel(z)
    assert all(z[i, j] == 0.0 for i in range(3) for j in range(i, 5))
    # :64-68 -- a single cell is a no-op
    one = np.array([[7.0]], np.float32)
    mas.forward_parallel(one)
    assert one[0, 0] == 7.0


@pytest.mark.parametrize("t,s", [(1, 1), (1, 37), (5, 5), (12, 24), (31, 33), (33, 100),
                                 (64, 256), (200, 800), (511, 513), (512, 700), (513, 600),
                                 (1100, 1200), (2049, 2100)])
def test_items_bit_exact(mas, reference, oracle, cuda, t, s):
    rng = np.random.default_rng(t * 7919 + s)
    q = rng.uniform(-5, 5, (t, s)).astype(np.float32)
    want = reference.forward_parallel(q)
    assert _bits(oracle.forward_parallel(q)).tobytes() == _bits(want).tobytes()
    got = q.copy()
    assert mas.forward_parallel(got) is got
    np.testing.assert_array_equal(_bits(got), _bits(want))


def test_signed_zeros_and_ties(mas, reference, cuda):
    rng = np.random.default_rng(3)
    for it in range(6):
        t, s = int(rng.integers(2, 70)), int(rng.integers(70, 140))
        q = np.zeros((t, s), np.float32)
        q[rng.random((t, s)) < 0.5] = -0.0
        q[rng.random((t, s)) < 0.1] = 1.0
        want = reference.forward_parallel(q)
        got = mas.forward_parallel(q.copy())
        np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("mnv", [-1e32, -1e30, float("-inf")])
def test_sentinels(mas, reference, cuda, mnv):
    rng = np.random.default_rng(5)
    q = rng.uniform(-5, 5, (40, 90)).astype(np.float32)
    want = reference.forward_parallel(q, max_neg_val=mnv)
    got = mas.forward_parallel(q.copy(), max_neg_val=mnv)
    np.testing.assert_array_equal(_bits(got), _bits(want))


def test_ragged_batch_leaves_padding_untouched(mas, reference, cuda):
    rng = np.random.default_rng(11)
    B, T, S = 6, 300, 900
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    lens = np.array([[300, 900], [1, 1], [17, 40], [299, 777], [0, 0], [150, 151]])
    got = q.copy()
    mas.forward_parallel(got, lengths=lens)
    for b in range(B):
        t, s = lens[b]
        want = q[b].copy()
        if t and s:
            want[:t, :s] = reference.forward_parallel(q[b, :t, :s])
        np.testing.assert_array_equal(_bits(got[b]), _bits(want), err_msg=f"item {b}")


def test_torch_in_place_pitched(mas, reference, cuda):
    import torch

    rng = np.random.default_rng(13)
    B, T, S, P = 3, 520, 1000, 1040
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    buf = torch.full((B, T, P), 123.0, dtype=torch.float32, device="cuda")
    view = buf[:, :, :S]
    view.copy_(torch.from_numpy(q))
    assert mas.forward_parallel(view) is view
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    assert (got[:, :, S:] == 123.0).all()
    for b in range(B):
        np.testing.assert_array_equal(_bits(got[b, :, :S]), _bits(reference.forward_parallel(q[b])))


def test_rejects_bad_input(mas, cuda):
    with pytest.raises(ValueError):
        mas.forward_parallel(np.zeros((2, 3), np.float64))
    with pytest.raises(ValueError):
        mas.forward_parallel(np.zeros((2, 3), np.float32), lengths=[[3, 3]])
    with pytest.raises(ValueError):
        mas.forward_parallel(np.zeros((2, 3), np.float32)[:, ::2])


def test_large_batch_sequential_strips(mas, reference, cuda):
    """B >= SM count: each CTA walks its item's strips in order (the other
    scheduling mode of mas_forward_scores)."""
    rng = np.random.default_rng(17)
    B, T, S = 160, 600, 70
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    lens = np.stack([rng.integers(1, T + 1, B), np.full(B, S)], 1)
    got = q.copy()
    mas.forward_parallel(got, lengths=lens)
    for b in range(0, B, 7):
        t, s = lens[b]
        want = q[b].copy()
        want[:t, :s] = reference.forward_parallel(q[b, :t, :s])
        np.testing.assert_array_equal(_bits(got[b]), _bits(want), err_msg=f"item {b}")


# ---- the K1 score export (mas_fwd4.cu OUT 1) vs the general kernel ----------
# mas_forward_scores takes K1's TMA path when q has a 16-byte base, pitch % 4
# == 0 and text_cap % 4 == 0 (forward_scores_fwd4 in mas_abi.cu), the general
# forward_scores_kernel otherwise; both must give the reference's table.

def _same(got, want):
    """Bit-identical, NaNs of any payload counted equal (the GPU's canonical
    NaN vs the CPU's propagated payloads)."""
    g, w = _bits(got), _bits(want)
    return bool(((g == w) | (np.isnan(got) & np.isnan(want))).all())


def _scores_ex(values, engine, mnv, lengths=None):
    """mas_forward_scores_ex on a contiguous [B, T, S] CUDA tensor, in place."""
    import ctypes

    import torch
    from paper_2409_07704_b200 import _lib

    lib = _lib.load()
    B, T, S = values.shape
    err = _lib.MasError()
    lens = None if lengths is None else np.ascontiguousarray(lengths, dtype=np.uint32)
    rc = lib.mas_forward_scores_ex(values.data_ptr(), S, B, T, S,
                                   None if lens is None else lens.ctypes.data,
                                   _lib.MAS_ENGINE_REFERENCE if engine == "reference"
                                   else _lib.MAS_ENGINE_PARALLEL,
                                   float(np.float32(mnv)),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                   ctypes.byref(err))
    _lib.raise_for(rc, err)
    torch.cuda.synchronize()


def _run_export(reference, engine, q, mnv, lengths=None):
    import torch

    B, T, S = q.shape
    dev = torch.from_numpy(q).cuda()
    _scores_ex(dev, engine, mnv, lengths)
    got = dev.cpu().numpy()
    for b in range(B):
        t, s = (T, S) if lengths is None else lengths[b]
        want = q[b].copy()
        if t and s:
            f = reference.forward_parallel if engine == "parallel" else reference.forward_reference
            want[:t, :s] = f(np.ascontiguousarray(q[b, :t, :s]), max_neg_val=mnv)
        assert _same(got[b], want), f"{engine} item {b} t={t} s={s}"


@pytest.mark.parametrize("engine", ["parallel", "reference"])
@pytest.mark.parametrize("t,s", [(4, 1), (4, 33), (8, 8), (36, 40), (128, 96), (132, 300),
                                 (256, 1000), (260, 777), (1024, 640), (4096, 160)])
def test_export_shapes_both_engines(reference, cuda, engine, t, s):
    # t % 4 == 0 and a contiguous pitch s: the K1 path when s % 4 == 0,
    # the general kernel otherwise
    rng = np.random.default_rng(t * 31 + s)
    q = rng.uniform(-5, 5, (1, t, s)).astype(np.float32)
    _run_export(reference, engine, q, -1e32)


@pytest.mark.parametrize("engine", ["parallel", "reference"])
def test_export_bands(reference, cuda, engine):
    # 9000 rows: three bands of clusters in one launch (mas_fwd4 band links)
    rng = np.random.default_rng(9000)
    q = rng.uniform(-5, 5, (1, 9000, 160)).astype(np.float32)
    _run_export(reference, engine, q, -1e32)


@pytest.mark.parametrize("engine", ["parallel", "reference"])
def test_export_ragged_batch(reference, cuda, engine):
    rng = np.random.default_rng(77)
    B, T, S = 7, 264, 520
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    lens = np.array([[264, 520], [1, 1], [17, 40], [263, 519], [0, 0], [130, 131], [5, 0]])
    _run_export(reference, engine, q, -1e32, lens)


@pytest.mark.parametrize("engine", ["parallel", "reference"])
@pytest.mark.parametrize("mnv", [-1e32, -1e9, float("-inf"), float("nan")])
def test_export_sentinels_zeros_nonfinite(reference, cuda, engine, mnv):
    rng = np.random.default_rng(19)
    q = rng.uniform(-3, 3, (2, 132, 260)).astype(np.float32)
    q[0][rng.random((132, 260)) < 0.4] = -0.0
    q[0][rng.random((132, 260)) < 0.2] = 0.0
    q[1][rng.random((132, 260)) < 0.01] = np.nan
    q[1][rng.random((132, 260)) < 0.01] = -np.inf
    q[1][rng.random((132, 260)) < 0.01] = np.inf
    _run_export(reference, engine, q, mnv)


def test_export_pitched_torch_view_untouched_tail(reference, cuda):
    import torch

    rng = np.random.default_rng(23)
    B, T, S, P = 3, 520, 1000, 1040
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    buf = torch.full((B, T, P), 123.0, dtype=torch.float32, device="cuda")
    buf[:, :, :S].copy_(torch.from_numpy(q))
    import ctypes
    from paper_2409_07704_b200 import _lib
    lib = _lib.load()
    err = _lib.MasError()
    rc = lib.mas_forward_scores_ex(buf.data_ptr(), P, B, T, S, None, _lib.MAS_ENGINE_REFERENCE,
                                   -1e32, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                   ctypes.byref(err))
    _lib.raise_for(rc, err)
    got = buf.cpu().numpy()
    assert (got[:, :, S:] == 123.0).all()
    for b in range(B):
        assert _same(got[b, :, :S], reference.forward_reference(q[b]))
