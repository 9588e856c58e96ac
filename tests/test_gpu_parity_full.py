"""Full-batch parity at BASELINE's large configs, against the UNMODIFIED
reference engines (oracle/_ref, multi-threaded for the parallel engine), and
the error / sentinel edges the reference defines:

* c4 (B16 T4096 S16384, cluster + band path) and c5 (B256 T512 S4096 at
  -1e32 / -inf / -1e9, both engines): every item byte-for-byte;
* a text of 16384 rows (four bands in one launch);
* SpeechTooLong (types.cpp:95-99) and LengthsOutOfRange (types.cpp:88-94)
  through the C-ABI, where the Python binding's own checks do not run first;
* validate_item of a later item with zero lengths (item_base > 0);
* NaN sentinels under detail::align_unchecked: the reference's std::max rule
  ((a < b) ? b : a keeps a NaN first operand) is reproduced exactly.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SENT = {"m1e32": -1e32, "minf": float("-inf"), "m1e9": -1e9}


def _dev_batch(mas, B, T, S, seed=0):
    qd = mas.generate_device(B, T, S, seed)
    return qd, qd.cpu().numpy()


def _diff(got, exp):
    return f"{int((got != exp).sum())} bytes differ in items " \
           f"{sorted(set(np.nonzero(got != exp)[0].tolist()))[:10]}"


@pytest.mark.slow
def test_config_c4_every_item(mas, reference, cuda):
    import torch

    B, T, S = 16, 4096, 16384
    qd, q = _dev_batch(mas, B, T, S)
    for eng in ("parallel", "reference"):
        got = mas.align(qd, engine=eng).cpu().numpy()
        code, msg, exp, _ = reference.align(q, engine=eng, threads=0)
        assert code == -1, msg
        assert np.array_equal(got, exp), (eng, _diff(got, exp))
        del got, exp
    del qd
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_config_c5_every_item_every_sentinel(mas, reference, cuda):
    import torch

    B, T, S = 256, 512, 4096
    qd, q = _dev_batch(mas, B, T, S)
    for eng in ("parallel", "reference"):
        for name, mnv in SENT.items():
            if name == "m1e32":
                got = mas.align(qd, engine=eng).cpu().numpy()
            else:
                got = mas._align_unchecked(qd, engine=eng, max_neg_val=mnv).cpu().numpy()
            code, msg, exp, _ = reference.align(q, engine=eng, max_neg_val=mnv, threads=0,
                                                unchecked=name != "m1e32")
            assert code == -1, msg
            assert np.array_equal(got, exp), (eng, name, _diff(got, exp))
    del qd
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_text_of_four_bands(mas, reference, cuda):
    """T = 16384: texts taller than one cluster run as bands of clusters in
    one launch; four or more bands here."""
    import torch

    B, T, S = 1, 16384, 16500
    plan = mas.Plan(B, T, S + (-S % 4))
    assert T // (plan.geometry["rows_per_warp"] * plan.geometry["warps_per_cta"]
                 * plan.geometry["ctas_per_item"]) >= 3
    qd, q = _dev_batch(mas, B, T, S, seed=3)
    for eng in ("parallel", "reference"):
        got = mas.align_paths(qd, engine=eng)
        code, msg, _, exp = reference.align(q, engine=eng, threads=0, want_out=False,
                                            want_paths=True)
        assert code == -1, msg
        assert np.array_equal(np.asarray(got[0].cpu() if hasattr(got[0], "cpu") else got[0]),
                              exp[0]), eng
    del qd
    torch.cuda.empty_cache()


def _c_align(mas, q, lengths, engine=1, mnv=-1e32, flags=0, item_base=None):
    """mas_align_host (or mas_validate_host with item_base) straight through
    the C-ABI; returns (status, errc, item, message)."""
    from paper_2409_07704_b200 import _lib

    lib = _lib.load()
    q = np.ascontiguousarray(q, np.float32)
    B, T, S = q.shape
    lens = np.ascontiguousarray(lengths, np.uint32)
    err = _lib.MasError()
    if item_base is not None:
        rc = lib.mas_validate_host(q.ctypes.data, B, T, S, lens.ctypes.data, item_base,
                                   ctypes.byref(err))
    else:
        cfg = _lib.MasConfig()
        lib.mas_config_default(ctypes.byref(cfg))
        cfg.engine = engine
        cfg.max_neg_val = mnv
        cfg.flags = flags
        out = np.zeros((B, T, S), np.uint8)
        rc = lib.mas_align_host(q.ctypes.data, B, T, S, lens.ctypes.data, ctypes.byref(cfg),
                                out.ctypes.data, None, ctypes.byref(err))
    return rc, err.errc, err.item, err.message.decode()


def test_speech_too_long(mas, reference, cuda):
    """s > 100000 (types.cpp:95-99): the Python binding, the C-ABI and the
    reference agree on code and text."""
    q = np.zeros((1, 1, 100001), np.float32)
    code, msg, _, _ = reference.align(q)
    assert code == 4, msg  # SpeechTooLong
    with pytest.raises(ValueError) as ei:
        mas.align(q)
    assert str(ei.value) == msg
    rc, errc, item, cmsg = _c_align(mas, q, [[1, 100001]])
    assert (rc, errc, item, cmsg) == (1, 4, 0, msg)
    # the lowest failing item wins, also when a later item is too long
    q2 = np.zeros((2, 1, 100001), np.float32)
    lens = [[1, 100000], [1, 100001]]
    code2, msg2, _, _ = reference.align(q2, lengths=lens)
    rc, errc, item, cmsg = _c_align(mas, q2, lens)
    assert (rc, errc, item, cmsg) == (1, code2, 1, msg2)


@pytest.mark.parametrize("lens", [[[5, 9]], [[4, 10]], [[9, 12]], [[0, 3]]])
def test_lengths_out_of_range_through_the_c_abi(mas, reference, cuda, lens):
    """validate_item's LengthsOutOfRange / ZeroDim order (types.cpp:81-99) on
    lengths beyond the capacities, which the Python binding rejects before the
    library sees them (module.cpp:61-84); the C-ABI and C++ paths must match
    the reference's engine-level check."""
    q = np.random.default_rng(1).uniform(-5, 5, (1, 4, 9)).astype(np.float32)
    code, msg, _, _ = reference.align(q, lengths=lens)
    assert code >= 0
    rc, errc, item, cmsg = _c_align(mas, q, lens)
    assert (rc, errc, item, cmsg) == (1, code, 0, msg)


def test_validate_item_of_a_later_item(mas, reference, cuda):
    """validate_item(batch, b) passes item b alone with item_base = b; its
    host errors must not index past the one-item plan."""
    q3 = np.random.default_rng(2).uniform(-5, 5, (3, 4, 9)).astype(np.float32)
    lens3 = [[4, 9], [4, 9], [0, 0]]
    code, msg, _, _ = reference.align(q3, lengths=lens3)
    assert code == 0, msg  # ZeroDim, item 2
    rc, errc, item, cmsg = _c_align(mas, q3[2:], [[0, 0]], item_base=2)
    assert (rc, errc, item, cmsg) == (1, 0, 2, msg)
    q3[2, 1, 1] = np.nan
    rc, errc, item, cmsg = _c_align(mas, q3[2:], [[4, 9]], item_base=2)
    assert (rc, errc, item) == (1, 3, 2) and cmsg.startswith("item 2:")


@pytest.mark.parametrize("engine", ["parallel", "reference"])
def test_nan_sentinel_unchecked(mas, reference, cuda, engine):
    """detail::align_unchecked with max_neg_val = NaN follows std::max
    ((a < b) ? b : a): the parallel engine's table keeps NaN wherever the
    first operand is NaN; the reference engine pins i > j cells to NaN, which
    the max then discards.  Both must match the reference byte for byte."""
    rng = np.random.default_rng(5)
    cases = [rng.uniform(-5, 5, (4, 37, 130)).astype(np.float32),
             rng.uniform(-5, 5, (2, 300, 700)).astype(np.float32)]
    adv = np.where(np.arange(32)[:, None] > np.arange(2048)[None, :], 1e8, -1e8)
    cases.append(adv.astype(np.float32)[None])
    for q in cases:
        B, T, S = q.shape
        lens = np.stack([rng.integers(1, T + 1, B), np.full(B, S)], 1)
        lens[:, 1] = np.maximum(lens[:, 0], rng.integers(1, S + 1, B))
        lens[0] = (T, S)
        code, msg, exp, exp_paths = reference.align(q, lengths=lens, engine=engine,
                                                    max_neg_val=float("nan"), unchecked=True,
                                                    want_paths=True)
        assert code == -1, msg
        got = mas._align_unchecked(q, lengths=lens, engine=engine, max_neg_val=float("nan"))
        assert np.array_equal(got, exp), (q.shape, _diff(got, exp))


def test_nan_sentinel_nonfinite_still_reported(mas, reference, cuda):
    q = np.random.default_rng(6).uniform(-5, 5, (3, 20, 50)).astype(np.float32)
    q[1, 3, 7] = np.inf
    code, msg, _, _ = reference.align(q, max_neg_val=float("nan"), unchecked=True)
    assert code == 3, msg
    with pytest.raises(ValueError) as ei:
        mas._align_unchecked(q, max_neg_val=float("nan"))
    assert str(ei.value) == msg
