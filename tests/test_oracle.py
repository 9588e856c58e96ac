"""Pins the CPU oracle (oracle/mas_oracle.c) to the reference: golden
vectors from the unmodified reference, the reference tests' known answers,
and -- where oracle/_ref was built -- direct byte comparison.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from _golden import ENGINES, SENTINELS, G, cases, expected, inputs, paths_to_out, sha


def _gen(oracle):
    return lambda b, t, s, seed: oracle.generate(b, t, s, seed)


GOLDEN_TAGS = [t for t in cases("") if not t.startswith(("err_", "gen_"))]


@pytest.mark.parametrize("tag", GOLDEN_TAGS)
def test_oracle_matches_golden(oracle, tag):
    q, lengths = inputs(tag, _gen(oracle))
    qq = q if q.ndim == 3 else q[None]
    for eng in ENGINES:
        for sn, mnv in SENTINELS.items():
            exp_paths, exp_sha = expected(tag, eng, sn)
            if exp_paths is None:
                continue
            code, _, _, out, paths = oracle.align(q, lengths, engine=eng, max_neg_val=mnv,
                                                  unchecked=True)
            assert code == -1
            np.testing.assert_array_equal(paths, exp_paths, err_msg=f"{tag} {eng} {sn}")
            assert sha(out) == exp_sha
            assert sha(paths_to_out(exp_paths, qq.shape[1], qq.shape[2])) == exp_sha


def test_kat_2x3(oracle):
    """test_reference.cpp:25-35 / test_smoke.py:13-18: path [0, 1, 1]."""
    q = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    for eng in ENGINES:
        _, _, _, out, paths = oracle.align(q, engine=eng)
        assert paths.tolist() == [[0, 1, 1]]
        assert out[0].tolist() == [[1, 0, 0], [0, 1, 1]]
    # Q table of the parallel engine: [[1, 3, 6], [mnv, 6, 12]] (test_parallel.cpp:71-76)
    Q = oracle.forward_parallel(q)
    assert Q[0].tolist() == [1, 3, 6] and Q[1, 1:].tolist() == [6, 12]


def test_kat_tie_rule(oracle):
    """All-zero 3x5: stay unless upper-left strictly greater (backtrack.hpp:26)."""
    _, _, _, _, paths = oracle.align(np.zeros((3, 5), np.float32))
    assert paths.tolist() == [[0, 1, 2, 2, 2]]


def test_kat_t_equals_s_and_t1(oracle):
    q = oracle.generate(1, 6, 6, 1)
    _, _, _, out, paths = oracle.align(q)
    assert paths.tolist() == [list(range(6))]
    _, _, _, out, paths = oracle.align(oracle.generate(1, 1, 9, 1))
    assert paths.tolist() == [[0] * 9]


@pytest.mark.parametrize("tag", cases("gen_"))
def test_generator_pinned(oracle, tag):
    _, b, t, s, seed = tag.split("_")
    got = oracle.generate(int(b), int(t), int(s), int(seed))
    assert sha(got) == str(G()[f"{tag}/sha"])


def test_generator_shard_addressable(oracle):
    full = oracle.generate(6, 5, 13, 77)
    for first in range(6):
        np.testing.assert_array_equal(oracle.generate(2 if first < 5 else 1, 5, 13, 77, first),
                                      full[first:first + 2])


@pytest.mark.parametrize("tag", cases("err_"))
def test_oracle_error_codes(oracle, tag):
    g = G()
    base = oracle.generate(3, 40, 100, 9)
    q = g.get(f"{tag}/q", g["err_nonfinite/q"] if tag in ("err_nonfinite_ref", "err_order")
              else base)
    lengths = g.get(f"{tag}/lengths")
    kw = {}
    if tag == "err_order":
        lengths = np.array([[40, 100], [40, 100], [5, 3]])
    if tag.startswith("err_mnv_"):
        kw["max_neg_val"] = {"m1e9": -1e9, "minf": float("-inf"), "nan": float("nan")}[tag[8:]]
    if tag == "err_threads":
        code = oracle.lib.oracle_validate_config(np.float32(-1e32), -1)
    else:
        code, item, (i, j), _, _ = oracle.align(
            q, lengths, engine="reference" if tag.endswith("_ref") else "parallel", **kw)
        msg = str(g[f"{tag}/msg"])
        if code == 3:
            assert msg == f"item {item}: non-finite likelihood at ({i}, {j})"
        elif item >= 0:
            assert msg.startswith(f"item {item}: ")
    assert code == int(g[f"{tag}/code"])


def test_oracle_vs_reference_random(oracle, reference):
    """Direct byte comparison with the reference build on fresh seeds."""
    rng = np.random.default_rng(1234)
    for k in range(40):
        B = int(rng.integers(1, 4))
        T = int(rng.integers(1, 80))
        S = int(rng.integers(T, 300))
        q = rng.uniform(-5, 5, (B, T, S)).astype(np.float32)
        lt = rng.integers(1, T + 1, B)
        lens = np.stack([lt, [int(rng.integers(a, S + 1)) for a in lt]], 1)
        for eng in ENGINES:
            for sn in ("m1e32", "m1e9"):
                c1, _, o1, _ = reference.align(q, lens, engine=eng, max_neg_val=SENTINELS[sn],
                                               unchecked=True)
                c2, _, _, o2, _ = oracle.align(q, lens, engine=eng, max_neg_val=SENTINELS[sn],
                                               unchecked=True)
                assert c1 == -1 and c2 == -1
                np.testing.assert_array_equal(o1, o2)


def test_generator_vs_reference(oracle, reference):
    for (b, t, s, seed) in [(2, 17, 40, 3), (1, 64, 256, 0), (4, 3, 9, 2**64 - 1)]:
        np.testing.assert_array_equal(oracle.generate(b, t, s, seed),
                                      reference.generate(b, t, s, seed))


def test_forward_parallel_matches_reference(oracle, reference):
    """The score-table restatement (oracle_forward_parallel) against the
    reference's parallel::forward_parallel, bit for bit (test_parallel.cpp:91-103)."""
    rng = np.random.default_rng(21)
    for it in range(40):
        t = int(rng.integers(1, 40))
        s = int(rng.integers(t, 90))
        q = rng.uniform(-5, 5, (t, s)).astype(np.float32)
        if it % 4 == 0:
            q[rng.random((t, s)) < 0.5] = 0.0
            q[rng.random((t, s)) < 0.3] = -0.0
        mnv = [-1e32, -1e30, float("-inf")][it % 3]
        a = oracle.forward_parallel(q, max_neg_val=mnv)
        b = reference.forward_parallel(q, max_neg_val=mnv)
        assert a.view(np.uint32).tobytes() == b.view(np.uint32).tobytes(), it
