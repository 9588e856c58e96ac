"""Parity of the sm_100a path with the reference, on a B200.

Everything here goes through the product's C-ABI (the Python surface calls
include/monoalign_b200.h entry points) and is checked against
  * tests/golden/golden.npz -- outputs of the unmodified reference, and
  * the CPU oracle (oracle/mas_oracle.c, itself pinned to the reference by
    tests/test_oracle.py) on fresh seeded inputs.
The bar is bit-exact: identical alignment bytes and paths.
"""

from __future__ import annotations

import threading

import numpy as np
import pytest

from _golden import ENGINES, SENTINELS, G, cases, expected, inputs, paths_to_out, sha

pytestmark = pytest.mark.gpu


def _gen(oracle):
    return lambda b, t, s, seed: oracle.generate(b, t, s, seed)


def _run(mas, q, lengths, engine, sentinel):
    if sentinel == "m1e32":
        return mas.align(q, lengths=lengths, engine=engine)
    return mas._align_unchecked(q, lengths=lengths, engine=engine,
                                max_neg_val=SENTINELS[sentinel])


GOLDEN_TAGS = [t for t in cases("") if not t.startswith(("err_", "gen_"))]


@pytest.mark.parametrize("tag", GOLDEN_TAGS)
def test_golden(mas, oracle, cuda, tag):
    q, lengths = inputs(tag, _gen(oracle))
    for eng in ENGINES:
        for sn in SENTINELS:
            exp_paths, exp_sha = expected(tag, eng, sn)
            if exp_paths is None:
                continue
            out = _run(mas, q, lengths, eng, sn)
            assert out.dtype == np.uint8 and out.shape == q.shape
            assert sha(out if out.ndim == 3 else out[None]) == exp_sha, f"{tag} {eng} {sn}"
            if sn == "m1e32":
                got = mas.align_paths(q, lengths=lengths, engine=eng)
                got = [got] if q.ndim == 2 else got
                for b, p in enumerate(got):
                    sb = int(np.sum(exp_paths[b] >= 0))
                    assert p.dtype == np.int32 and p.shape == (sb,)
                    np.testing.assert_array_equal(p, exp_paths[b, :sb])


@pytest.mark.parametrize("tag", cases("err_"))
def test_errors_match_reference(mas, oracle, cuda, tag):
    g = G()
    base = oracle.generate(3, 40, 100, 9)
    q = g.get(f"{tag}/q", g["err_nonfinite/q"] if tag in ("err_nonfinite_ref", "err_order")
              else base)
    lengths = g.get(f"{tag}/lengths")
    if tag == "err_order":
        lengths = np.array([[40, 100], [40, 100], [5, 3]])
    kw = {}
    if tag.startswith("err_mnv_"):
        kw["max_neg_val"] = {"m1e9": -1e9, "minf": float("-inf"), "nan": float("nan")}[tag[8:]]
    if tag == "err_threads":
        kw["threads"] = -1
    if tag.endswith("_ref"):
        kw["engine"] = "reference"
    for fn in (mas.align, mas.align_paths):
        with pytest.raises(ValueError) as ei:
            fn(q, lengths=lengths, **kw)
        assert str(ei.value) == str(g[f"{tag}/msg"])


def test_reference_smoke_suite(mas, cuda):
    """The reference's tests/python/test_smoke.py cases (align / align_paths /
    generate_random_batch), against this package."""
    assert mas.__version__ == "1.0.0"
    q = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    out = mas.align(q)
    assert out.dtype == np.uint8 and out.shape == (2, 3)
    np.testing.assert_array_equal(out, [[1, 0, 0], [0, 1, 1]])
    rng = np.random.default_rng(7)
    qb = rng.uniform(-5, 5, size=(4, 8, 20)).astype(np.float32)
    np.testing.assert_array_equal(mas.align(qb, engine="reference"),
                                  mas.align(qb, engine="parallel"))
    np.testing.assert_array_equal(mas.align(q.astype(np.float64)), [[1, 0, 0], [0, 1, 1]])
    p = mas.align_paths(q)
    assert p.dtype == np.int32
    np.testing.assert_array_equal(p, [0, 1, 1])
    ps = mas.align_paths(np.zeros((2, 3, 5), np.float32))
    assert isinstance(ps, list) and len(ps) == 2
    for pp in ps:
        np.testing.assert_array_equal(pp, [0, 1, 2, 2, 2])
    out = mas.align(np.ones((2, 4, 6), np.float32),
                    lengths=np.array([[2, 3], [4, 6]], np.uint32))
    assert out[0, 2:, :].sum() == 0 and out[0, :, 3:].sum() == 0
    assert out[0, :2, :3].sum() == 3 and out[1].sum() == 6
    with pytest.raises(ValueError):
        mas.align(np.zeros((3, 2), np.float32))
    with pytest.raises(ValueError):
        mas.align(np.zeros((2, 3), np.float32), engine="turbo")
    a = mas.generate_random_batch(2, 8, 32, seed=5)
    b = mas.generate_random_batch(2, 8, 32, seed=5)
    c = mas.generate_random_batch(2, 8, 32, seed=6)
    assert a.dtype == np.float32 and a.shape == (2, 8, 32)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    assert a.min() >= -5.0 and a.max() <= 5.0


def test_reference_smoke_suite_io(mas, cuda, tmp_path):
    """The reference's test_smoke.py tensor-file cases (:73-103)."""
    path = str(tmp_path / "batch.bin")
    rng = np.random.default_rng(11)
    values = rng.uniform(-5, 5, size=(3, 4, 9)).astype(np.float32)
    lengths = np.array([[2, 5], [4, 9], [1, 1]], dtype=np.uint32)
    mas.write_tensor(path, values, lengths=lengths)
    got_values, got_lengths = mas.read_tensor(path)
    np.testing.assert_array_equal(got_values, values)
    np.testing.assert_array_equal(got_lengths, lengths)
    path = str(tmp_path / "matrix.bin")
    out = mas.align(np.zeros((2, 3, 5), dtype=np.float32))
    mas.write_tensor(path, out)
    got_values, _ = mas.read_tensor(path)
    assert got_values.dtype == np.uint8
    np.testing.assert_array_equal(got_values, out)
    with pytest.raises(OSError):
        mas.read_tensor(str(tmp_path / "absent.bin"))
    with pytest.raises(ValueError):
        mas.write_tensor(str(tmp_path / "bad.bin"), np.zeros((1, 2, 3), dtype=np.int64))


@pytest.mark.parametrize("tag", cases("gen_"))
def test_device_generator_pinned(mas, cuda, tag):
    _, b, t, s, seed = tag.split("_")
    got = mas.generate_random_batch(int(b), int(t), int(s), int(seed))
    assert sha(got) == str(G()[f"{tag}/sha"])


def test_device_generator_shards(mas, oracle, cuda):
    full = oracle.generate(8, 33, 70, 123)
    for first, n in [(0, 3), (3, 4), (7, 1)]:
        got = mas.generate_device(n, 33, 70, 123, first_item=first, row_pitch=72)
        np.testing.assert_array_equal(got.cpu().numpy(), full[first:first + n])


def _check_random(mas, oracle, rng, B, T, S, ragged, poison=False, engines=ENGINES,
                  sentinels=("m1e32",)):
    q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
    lens = None
    if ragged:
        lt = rng.integers(1, T + 1, B)
        lens = np.stack([lt, [int(rng.integers(a, S + 1)) for a in lt]], 1)
        if poison:
            for b in range(B):
                q[b, lens[b, 0]:, :] = np.nan
                q[b, :, lens[b, 1]:] = np.nan
    for eng in engines:
        for sn in sentinels:
            code, _, _, exp, exp_p = oracle.align(q, lens, engine=eng,
                                                  max_neg_val=SENTINELS[sn], unchecked=True)
            assert code == -1
            got = _run(mas, q, lens, eng, sn)
            if not np.array_equal(got, exp):
                bad = np.argwhere(got != exp)
                pytest.fail(f"B{B} T{T} S{S} {eng} {sn} ragged={ragged}: "
                            f"{len(bad)} bytes differ, first {bad[:3].tolist()}")
            if sn == "m1e32":
                gp = mas.align_paths(q, lengths=lens, engine=eng)
                for b in range(B):
                    sb = S if lens is None else int(lens[b, 1])
                    np.testing.assert_array_equal(gp[b], exp_p[b, :sb])


def test_random_small(mas, oracle, cuda):
    rng = np.random.default_rng(11)
    for _ in range(60):
        T = int(rng.integers(1, 150))
        S = int(rng.integers(T, 700))
        _check_random(mas, oracle, rng, int(rng.integers(1, 5)), T, S, ragged=False,
                      sentinels=("m1e32", "m1e9"))


@pytest.mark.parametrize("T", [63, 64, 65, 127, 128, 129, 255, 256, 257, 300, 511, 512, 513,
                               1000, 1024, 1025, 2047, 2049, 4096])
def test_text_geometries(mas, oracle, cuda, T):
    """Every warp / CTA / cluster boundary of the T split."""
    rng = np.random.default_rng(T)
    S = T + int(rng.integers(0, 3 * T)) + int(rng.integers(0, 97))
    _check_random(mas, oracle, rng, 2, T, S, ragged=False)


@pytest.mark.parametrize("S", [1, 2, 3, 31, 32, 33, 63, 64, 65, 95, 127, 129, 1000, 4097])
def test_speech_edges(mas, oracle, cuda, S):
    """Partial TMA boxes / direction words / 64-column iterations."""
    rng = np.random.default_rng(1000 + S)
    T = max(1, min(S, int(rng.integers(1, 200))))
    _check_random(mas, oracle, rng, 3, T, S, ragged=False, sentinels=("m1e32", "minf"))


def test_ragged_and_poisoned_padding(mas, oracle, cuda):
    rng = np.random.default_rng(5)
    for _ in range(25):
        T = int(rng.integers(1, 400))
        S = int(rng.integers(T, 1500))
        _check_random(mas, oracle, rng, int(rng.integers(1, 7)), T, S, ragged=True,
                      poison=True)


def test_torch_device_tensors(mas, oracle, cuda):
    import torch

    rng = np.random.default_rng(3)
    q = rng.uniform(-5, 5, (3, 130, 515)).astype(np.float32)
    _, _, _, exp, exp_p = oracle.align(q)
    qd = torch.from_numpy(q).to(cuda)
    out = mas.align(qd)
    assert out.is_cuda and out.dtype == torch.uint8
    np.testing.assert_array_equal(out.cpu().numpy(), exp)
    # a strided (pitched) view: no copy on the TMA path when aligned
    big = torch.zeros((3, 130, 520), device=cuda)
    big[:, :, :515] = qd
    np.testing.assert_array_equal(mas.align(big[:, :, :515]).cpu().numpy(), exp)
    # odd pitch / odd T -> re-pitched copy inside the library
    big2 = torch.zeros((3, 130, 517), device=cuda)
    big2[:, :, :515] = qd
    np.testing.assert_array_equal(mas.align(big2[:, :, :515]).cpu().numpy(), exp)
    paths = mas.align_paths(qd)
    for b in range(3):
        np.testing.assert_array_equal(paths[b].cpu().numpy(), exp_p[b])


def test_plan_reuse_and_graph_capture(mas, oracle, cuda):
    import torch

    B, T, S = 4, 300, 1200
    q = mas.generate_device(B, T, S, 42)
    exp = oracle.align(oracle.generate(B, T, S, 42))[3]
    plan = mas.Plan(B, T, S)
    out = torch.empty((B, T, S), dtype=torch.uint8, device=cuda)
    paths = torch.empty((B, S), dtype=torch.int32, device=cuda)
    for _ in range(3):
        out.fill_(7)
        plan.enqueue(q, out, paths)
        plan.finish(q)
        np.testing.assert_array_equal(out.cpu().numpy(), exp)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            plan.enqueue(q, out, paths, stream=s)
    out.fill_(9)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), exp)
    assert plan.launches == 2
    plan.close()


def test_concurrent_host_threads(mas, oracle, cuda):
    """Reentrant per call: several host threads align at once."""
    rng = np.random.default_rng(8)
    qs = [rng.uniform(-5, 5, (2, 100 + 50 * k, 700)).astype(np.float32) for k in range(4)]
    exps = [oracle.align(q)[3] for q in qs]
    res = [None] * 4

    def work(k):
        res[k] = mas.align(qs[k])

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(4):
        np.testing.assert_array_equal(res[k], exps[k])


def _invariants(out_np, lengths=None):
    """acceptance.cpp criterion 3: one 1 per valid column, zeros elsewhere,
    monotone path with unit steps, path[0]=0, path[s-1]=t-1."""
    B, T, S = out_np.shape
    for b in range(B):
        t, s = (T, S) if lengths is None else lengths[b]
        o = out_np[b]
        assert o[:, s:].sum() == 0 and o[t:, :].sum() == 0
        assert (o[:t, :s].sum(0) == 1).all()
        p = o[:t, :s].argmax(0)
        assert p[0] == 0 and p[-1] == t - 1
        assert set(np.unique(np.diff(p)).tolist()) <= {0, 1}


@pytest.mark.slow
def test_config_c3_full_bit_exact(mas, oracle, cuda):
    """BASELINE config 3 (B32 T1024 S8192): all 32 items vs the oracle."""
    import torch

    B, T, S = 32, 1024, 8192
    qd = mas.generate_device(B, T, S, 0)
    out = mas.align(qd)
    q = oracle.generate(B, T, S, 0)
    np.testing.assert_array_equal(qd.cpu().numpy()[:2], q[:2])
    exp = oracle.align(q)[3]
    got = out.cpu().numpy()
    assert np.array_equal(got, exp), f"{int((got != exp).sum())} bytes differ"
    ref = mas.align(qd, engine="reference").cpu().numpy()
    assert np.array_equal(ref, exp)
    del qd, out
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_config_c4_cluster_path(mas, oracle, cuda):
    """BASELINE config 4 (B16 T4096 S16384, 16-CTA clusters): invariants on
    all items, bit-exact on items 0, 7 and 15 (oracle on shards)."""
    import torch

    B, T, S = 16, 4096, 16384
    qd = mas.generate_device(B, T, S, 0)
    got = mas.align(qd).cpu().numpy()
    del qd
    torch.cuda.empty_cache()
    _invariants(got)
    for b in (0, 7, 15):
        q = oracle.generate(1, T, S, 0, first_item=b)
        exp = oracle.align(q)[3]
        assert np.array_equal(got[b:b + 1], exp), f"item {b}"


@pytest.mark.slow
def test_config_c5_sentinel_boundary(mas, oracle, cuda):
    """BASELINE config 5 (B256 T512 S4096): -1e32 (public), -inf and -1e9
    (unchecked) give identical alignments, equal to the CPU engines; the
    public API rejects -inf / -1e9."""
    import torch

    B, T, S = 256, 512, 4096
    qd = mas.generate_device(B, T, S, 0)
    outs = {}
    for eng in ENGINES:
        outs[(eng, "m1e32")] = mas.align(qd, engine=eng).cpu().numpy()
        for sn in ("minf", "m1e9"):
            with pytest.raises(ValueError, match="max_neg_val must be finite"):
                mas.align(qd[:1], engine=eng, max_neg_val=SENTINELS[sn])
            outs[(eng, sn)] = mas._align_unchecked(qd, engine=eng,
                                                   max_neg_val=SENTINELS[sn]).cpu().numpy()
    first = outs[("parallel", "m1e32")]
    for k, v in outs.items():
        assert np.array_equal(v, first), k
    _invariants(first)
    for b in (0, 100, 255):
        q = oracle.generate(1, T, S, 0, first_item=b)
        for sn in ("m1e32", "minf", "m1e9"):
            exp = oracle.align(q, max_neg_val=SENTINELS[sn], unchecked=True)[3]
            assert np.array_equal(first[b:b + 1], exp), (b, sn)
    del qd
    torch.cuda.empty_cache()


def test_config_c2_ragged_glowtts(mas, oracle, cuda):
    """BASELINE config 2 with its ragged lengths, padding poisoned to NaN."""
    q, lengths = inputs("c2", _gen(oracle))
    exp_paths, exp_sha = expected("c2", "parallel", "m1e32")
    q2 = q.copy()
    for b in range(q.shape[0]):
        q2[b, lengths[b, 0]:, :] = np.nan
        q2[b, :, lengths[b, 1]:] = np.nan
    for arr in (q, q2):
        out = mas.align(arr, lengths=lengths)
        assert sha(out) == exp_sha
    _invariants(out, lengths)


@pytest.mark.parametrize("shape", [(2, 900, 1500), (3, 1300, 2100), (1, 2048, 2048)])
def test_banded_forward_small_bands(mas, oracle, cuda, shape):
    """Texts taller than one cluster run in bands (mas_fwd4.cu banded mode);
    MAS_BAND_WARPS=2 forces 256-row bands so band hand-offs are exercised
    at oracle-friendly sizes.  Runs in a subprocess (the cap is read once)."""
    import os
    import subprocess
    import sys

    B, T, S = shape
    code = f"""
import sys, numpy as np
sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
import paper_2409_07704_b200 as m
from oracle.oracle import Oracle
o = Oracle()
rng = np.random.default_rng({B * T})
q = rng.uniform(-5, 5, ({B}, {T}, {S})).astype(np.float32)
lt = np.array([{T}] + [int(x) for x in rng.integers(1, {T} + 1, {B} - 1)])
ls = np.array([max(int(a), int(rng.integers(a, {S} + 1))) for a in lt])
lens = np.stack([lt, ls], 1)
assert m.Plan({B}, {T}, {S} + 3 - ({S} + 3) % 4, lengths=lens).geometry['rows_per_warp'] == 128
for eng in ('parallel', 'reference'):
    got = m.align(q, lengths=lens, engine=eng)
    exp = o.align(q, lens, engine=eng)[3]
    assert np.array_equal(got, exp), (eng, int((got != exp).sum()))
    gp = m.align_paths(q, lengths=lens, engine=eng)
    ep = o.align(q, lens, engine=eng)[4]
    for b in range({B}):
        assert np.array_equal(gp[b], ep[b, :ls[b]]), (eng, b)
    gd = m.align_durations(q, lengths=lens, engine=eng)
    assert np.array_equal(gd, exp.sum(axis=2, dtype=np.int64).astype(np.int32)), eng
# a pipelined plan over the banded geometry (band tickets are reset between
# batches, so batches do not overlap there; results must still be exact)
import torch
qd = torch.from_numpy(q).cuda()
exp = torch.from_numpy(o.align(q, lens)[3]).cuda()
pp = m.Plan({B}, {T}, {S}, lengths=lens, pipelined=True)
outs = [torch.empty_like(exp) for _ in range(2)]
for k in range(5):
    pp.enqueue(qd, outs[k % 2])
torch.cuda.synchronize()
assert torch.equal(outs[0], exp) and torch.equal(outs[1], exp)
print('OK')
"""
    env = dict(os.environ, MAS_BAND_WARPS="2")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=600)
    assert res.returncode == 0 and "OK" in res.stdout, res.stdout[-2000:] + res.stderr[-3000:]


@pytest.mark.slow
def test_text_longer_than_a_cluster(mas, oracle, cuda):
    """T > 8192 (more than 16 CTAs x 4 warps x 128 rows): two bands."""
    rng = np.random.default_rng(9001)
    T, S = 9000, 9300
    q = rng.uniform(-5, 5, (1, T, S)).astype(np.float32)
    got = mas.align_paths(q)
    exp = oracle.align(q)[4]
    np.testing.assert_array_equal(got[0], exp[0])


# ---- durations: row sums of the alignment ---------
def _durations_of(out, lens=None):
    d = out.sum(axis=-1, dtype=np.int64).astype(np.int32)
    return d


def test_durations_match_alignment_row_sums(mas, oracle, cuda):
    rng = np.random.default_rng(77)
    for it in range(30):
        B = int(rng.integers(1, 6))
        T = int(rng.integers(1, 300))
        S = int(rng.integers(T, 1400))
        q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
        lt = rng.integers(1, T + 1, B)
        ls = np.array([int(rng.integers(a, S + 1)) for a in lt])
        lens = np.stack([lt, ls], 1) if it % 3 else None
        for eng in ("parallel", "reference"):
            exp = oracle.align(q, lens, engine=eng)[3]
            got = mas.align_durations(q, lengths=lens, engine=eng)
            assert got.dtype == np.int32 and got.shape == (B, T)
            np.testing.assert_array_equal(got, _durations_of(exp), err_msg=f"{it} {eng}")
            if lens is not None:
                assert np.all(got.sum(axis=1) == ls)
                for b in range(B):
                    assert np.all(got[b, lt[b]:] == 0)


def test_durations_golden_and_2d(mas, oracle, cuda):
    for tag in ("c1", "c2"):
        q, lengths = inputs(tag, _gen(oracle))
        exp_paths, _ = expected(tag, "parallel", "m1e32")
        T, S = q.shape[-2:]
        exp_out = paths_to_out(exp_paths, T, S)
        got = mas.align_durations(q, lengths=lengths)
        got = got[None] if got.ndim == 1 else got
        np.testing.assert_array_equal(got, _durations_of(exp_out))
    q = np.random.default_rng(4).uniform(-5, 5, (70, 333)).astype(np.float32)
    d = mas.align_durations(q)
    assert d.shape == (70,) and int(d.sum()) == 333
    np.testing.assert_array_equal(d, _durations_of(oracle.align(q[None])[3])[0])


def test_durations_device_plan_and_errors(mas, oracle, cuda):
    import torch

    B, T, S = 3, 257, 1031
    q = mas.generate_device(B, T, S, 5)
    exp = _durations_of(oracle.align(oracle.generate(B, T, S, 5))[3])
    d = mas.align_durations(q)
    assert d.is_cuda and d.dtype == torch.int32
    np.testing.assert_array_equal(d.cpu().numpy(), exp)
    # plan (aligned layout: T % 4 == 0, pitch % 4 == 0): durations only (no
    # dense output), then with the dense output
    T = 256
    q = mas.generate_device(B, T, S, 5, row_pitch=1032)
    exp = _durations_of(oracle.align(oracle.generate(B, T, S, 5))[3])
    plan = mas.Plan(B, T, S, row_pitch=1032)
    dur = torch.full((B, T), -5, dtype=torch.int32, device=cuda)
    plan.enqueue(q, durations=dur)
    plan.finish(q)
    np.testing.assert_array_equal(dur.cpu().numpy(), exp)
    out = torch.empty((B, T, S), dtype=torch.uint8, device=cuda)
    dur.fill_(-1)
    plan.enqueue(q, out=out, durations=dur)
    plan.finish(q)
    np.testing.assert_array_equal(dur.cpu().numpy(), exp)
    np.testing.assert_array_equal(out.sum(dim=2, dtype=torch.int32).cpu().numpy(), exp)
    plan.close()
    # the same errors as align
    bad = oracle.generate(2, 20, 50, 1)
    bad[1, 3, 7] = np.inf
    with pytest.raises(ValueError, match=r"item 1: non-finite likelihood at \(3, 7\)"):
        mas.align_durations(bad)
    with pytest.raises(ValueError):
        mas.align_durations(bad[:, :, :10], lengths=[[20, 10], [20, 10]])


def test_torch_check_false_is_enqueue_only(mas, oracle, cuda):
    """align(torch, check=False): same alignment, no NonFinite readback
    (a non-finite likelihood is not reported), host-side length errors still
    raised; repeated calls reuse the cached plan."""
    import torch

    rng = np.random.default_rng(12)
    q = rng.uniform(-5, 5, (4, 40, 120)).astype(np.float32)
    lens = np.array([[40, 120], [13, 50], [7, 7], [30, 100]])
    exp = oracle.align(q, lens)[3]
    qd = torch.from_numpy(q).cuda()
    for _ in range(3):
        got = mas.align(qd, lengths=lens, check=False)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), exp)
    bad = qd.clone()
    bad[1, 2, 3] = float("nan")
    mas.align(bad, lengths=lens, check=False)  # not reported
    with pytest.raises(ValueError, match="non-finite"):
        mas.align(bad, lengths=lens)
    with pytest.raises(ValueError):
        mas.align(qd, lengths=np.array([[40, 120], [13, 50], [8, 7], [30, 100]]), check=False)
    d1 = mas.align_durations(qd, lengths=lens, check=False)
    assert np.array_equal(d1.cpu().numpy(), exp.sum(2).astype(np.int32))


def test_pipelined_plan_overlapping_batches(mas, oracle, cuda):
    """Plan(pipelined=True): consecutive enqueues overlap (backtrack of batch
    i alongside the forward of batch i+1, two direction-word buffers); with
    distinct outputs per enqueue every batch's result is exact."""
    import torch

    B, T, S = 8, 256, 1024
    qs = [mas.generate_device(B, T, S, seed) for seed in (3, 4, 5)]
    exp = [mas.align(q).clone() for q in qs]
    exp_p = [torch.stack([torch.as_tensor(p) for p in mas.align_paths(q.cpu().numpy())]).cuda()
             for q in qs]
    plan = mas.Plan(B, T, S, pipelined=True)
    outs = [torch.empty((B, T, S), dtype=torch.uint8, device="cuda") for _ in range(3)]
    paths = [torch.empty((B, S), dtype=torch.int32, device="cuda") for _ in range(3)]
    for rep in range(4):
        for k in range(9):
            plan.enqueue(qs[k % 3], outs[k % 3], paths[k % 3])
        torch.cuda.synchronize()
        for k in range(3):
            assert torch.equal(outs[k], exp[k]), (rep, k)
            assert torch.equal(paths[k], exp_p[k]), (rep, k)
    plan.finish(qs[2])


@pytest.mark.parametrize("engine", ["parallel", "reference"])
@pytest.mark.parametrize("shape,ragged", [((1, 64, 256), False), ((32, 200, 800), True),
                                          ((5, 128, 1000), True), ((3, 256, 2100), False)])
def test_one_launch_tail(mas, oracle, cuda, engine, shape, ragged):
    """Small batches (every item one single-CTA cluster) run as ONE launch:
    the forward kernel walks and expands its own items from direction words
    in shared memory (mas_fwd4.cu OUT 2).  Alignment, paths and durations
    equal the oracle; a plan of a taller text still launches two kernels."""
    import torch

    B, T, S = shape
    rng = np.random.default_rng(B * T + S)
    lens = None
    if ragged:
        t = rng.integers(1, T + 1, B)
        s = np.maximum(t, rng.integers(1, S + 1, B))
        t[0], s[0] = T, S
        lens = np.stack([t, s], 1)
    q = mas.generate_device(B, T, S, 7)
    exp = oracle.align(oracle.generate(B, T, S, 7), lengths=lens, engine=engine)[3]
    plan = mas.Plan(B, T, S, lengths=lens, engine=engine)
    out = torch.full((B, T, S), 5, dtype=torch.uint8, device=cuda)
    paths = torch.empty((B, S), dtype=torch.int32, device=cuda)
    dur = torch.empty((B, T), dtype=torch.int32, device=cuda)
    plan.enqueue(q, out, paths, durations=dur)
    plan.finish(q)
    assert plan.launches == 1
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got, exp)
    pth, du = paths.cpu().numpy(), dur.cpu().numpy()
    for b in range(B):
        tb, sb = (T, S) if lens is None else lens[b]
        np.testing.assert_array_equal(pth[b, :sb], got[b, :, :sb].argmax(0))
        assert (pth[b, sb:] == -1).all()
        np.testing.assert_array_equal(du[b], got[b].sum(1))
    # durations only / paths only
    plan.enqueue(q, None, None, durations=dur)
    np.testing.assert_array_equal(dur.cpu().numpy(), got.sum(2))
    plan.enqueue(q, None, paths)
    for b in range(B):
        sb = S if lens is None else lens[b][1]
        np.testing.assert_array_equal(paths.cpu().numpy()[b, :sb], got[b, :, :sb].argmax(0))
    plan.close()
    tall = mas.Plan(1, 600, 900)
    tall.enqueue(mas.generate_device(1, 600, 900, 1), torch.empty((1, 600, 900), dtype=torch.uint8,
                                                                  device=cuda))
    assert tall.launches == 2
    tall.close()
