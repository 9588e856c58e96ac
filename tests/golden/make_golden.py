"""Generates tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libmonoalign_ref.so, i.e. the
reference engines compiled in place from /root/reference/proj/src by
oracle/Makefile):

    python tests/golden/make_golden.py

Every array in the file is an output of the reference's own public C++ API
(monoalign::align, parallel/reference ::detail::align_unchecked,
path_from_matrix, bench::generate_random_batch) called through
oracle/ref_shim.cpp.  Inputs are either literal (the reference tests' KATs)
or regenerated from seeds with the reference generator; a SHA-256 of each
generated input is stored so the generator restatement is pinned as well.
Cases follow the reference's own tests:
  kat_*          test_reference.cpp:25-35, test_parallel.cpp:78-89, test_smoke.py:13-48
  c1             BASELINE config 1, generate_random_batch(1, 64, 256, 0)
  single_*       acceptance.cpp:138-147 (random_item(mix_seed(2002, k), 64, 256))
  batched_*      acceptance.cpp:149-156 (B32 T128 S512, mix_seed(2003, k))
  ragged_*       acceptance.cpp:159-174 (B4 T64 S256, lengths from mix_seed(2005, k))
  adv_*          acceptance.cpp:208-244 (t=32, s=2048, +-1e8), sentinels -1e32/-1e9/-inf
  c2             BASELINE config 2 (B32 T200 S800, SURVEY.md 8(d) length recipe)
  err_*          validation codes + exact messages (types.cpp:59-130)
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, build  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
SENTINELS = {"m1e32": -1e32, "m1e9": -1e9, "minf": float("-inf")}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def splitmix64(state: int):
    M = (1 << 64) - 1
    state = (state + 0x9E3779B97F4A7C15) & M
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31), state


def mix_seed(seed: int, index: int) -> int:
    M = (1 << 64) - 1
    v, _ = splitmix64((seed ^ ((0xD1342543DE82EF95 * (index + 1)) & M)) & M)
    return v


def random_item_dims(seed: int, t_max: int, s_max: int):
    """tests/helpers.hpp:32-42."""
    v, st = splitmix64(seed)
    t = 1 + v % t_max
    t = min(t, s_max)
    v, st = splitmix64(st)
    s = t + v % (s_max - t + 1)
    return int(t), int(s)


def ragged_lengths(seed: int, B: int, T: int, S: int):
    """acceptance.cpp:162-168."""
    st = seed
    out = []
    for _ in range(B):
        v, st = splitmix64(st)
        t = 1 + v % T
        v, st = splitmix64(st)
        s = t + v % (S - t + 1)
        out.append((t, s))
    return np.array(out, np.int64)


def c2_lengths():
    """st = mix_seed(2, 0); t_b = 100 + r % 101;
    s_b = min(800, 3 t_b + r % (t_b + 1))."""
    st = mix_seed(2, 0)
    out = []
    for _ in range(32):
        v, st = splitmix64(st)
        t = 100 + v % 101
        v, st = splitmix64(st)
        s = min(800, 3 * t + v % (t + 1))
        out.append((t, s))
    return np.array(out, np.int64)


def main():
    build()
    ref = Reference()
    G = {}

    def run(tag, q, lengths=None, sentinels=("m1e32",)):
        for eng in ("parallel", "reference"):
            for sn in sentinels:
                mnv = SENTINELS[sn]
                code, msg, out, paths = ref.align(q, lengths, engine=eng, max_neg_val=mnv,
                                                  unchecked=sn != "m1e32", want_out=True,
                                                  want_paths=True)
                assert code == -1, (tag, eng, sn, msg)
                G[f"{tag}/{eng}/{sn}/paths"] = paths
                G[f"{tag}/{eng}/{sn}/out_sha"] = np.array(sha(out))

    # KATs (literal inputs).
    kat = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    G["kat_2x3/q"] = kat
    run("kat_2x3", kat)
    z = np.zeros((2, 3, 5), np.float32)
    G["kat_zeros/q"] = z
    run("kat_zeros", z)
    ones = np.ones((2, 4, 6), np.float32)
    G["kat_ragged_ones/q"] = ones
    G["kat_ragged_ones/lengths"] = np.array([[2, 3], [4, 6]], np.int64)
    run("kat_ragged_ones", ones, G["kat_ragged_ones/lengths"])
    t1 = ref.generate(1, 1, 7, 3)
    G["kat_t1/q"] = t1
    run("kat_t1", t1)
    ts = ref.generate(1, 9, 9, 4)
    G["kat_tes/q"] = ts
    run("kat_tes", ts)

    # c1: BASELINE config 1.
    c1 = ref.generate(1, 64, 256, 0)
    G["c1/q"] = c1
    G["c1/q_sha"] = np.array(sha(c1))
    run("c1", c1, sentinels=("m1e32", "m1e9", "minf"))

    # acceptance criterion 2, single items (first 64 seeds).
    for k in range(64):
        seed = mix_seed(2002, k)
        t, s = random_item_dims(seed, 64, 256)
        q = ref.generate(1, t, s, seed)
        G[f"single_{k}/seed"] = np.array(seed, np.uint64)
        G[f"single_{k}/dims"] = np.array([t, s], np.int64)
        G[f"single_{k}/q_sha"] = np.array(sha(q))
        run(f"single_{k}", q)

    # acceptance criterion 2, batched (first 3 seeds).
    for k in range(3):
        seed = mix_seed(2003, k)
        q = ref.generate(32, 128, 512, seed)
        G[f"batched_{k}/seed"] = np.array(seed, np.uint64)
        G[f"batched_{k}/q_sha"] = np.array(sha(q))
        run(f"batched_{k}", q)

    # acceptance criterion 2, ragged (first 8 seeds).
    for k in range(8):
        seed = mix_seed(2004, k)
        q = ref.generate(4, 64, 256, seed)
        lens = ragged_lengths(mix_seed(2005, k), 4, 64, 256)
        G[f"ragged_{k}/seed"] = np.array(seed, np.uint64)
        G[f"ragged_{k}/lengths"] = lens
        run(f"ragged_{k}", q, lens)

    # acceptance criterion 4: sentinel adversarial.
    i = np.arange(32)[:, None]
    j = np.arange(2048)[None, :]
    adv = np.where(i > j, np.float32(1e8), np.float32(-1e8)).astype(np.float32)
    run("adv", adv, sentinels=("m1e32", "m1e9", "minf"))

    # BASELINE config 2 (ragged Glow-TTS batch).
    c2 = ref.generate(32, 200, 800, 0)
    G["c2/lengths"] = c2_lengths()
    G["c2/q_sha"] = np.array(sha(c2))
    run("c2", c2, G["c2/lengths"], sentinels=("m1e32", "m1e9", "minf"))

    # Validation errors: code + exact message of the reference.
    def err(tag, q, lengths=None, **kw):
        code, msg, _, _ = ref.align(q, lengths, **kw)
        assert code >= 0, tag
        G[f"err_{tag}/code"] = np.array(code, np.int32)
        G[f"err_{tag}/msg"] = np.array(msg)

    base = ref.generate(3, 40, 100, 9)
    nan = base.copy()
    nan[1, 5, 7] = np.nan
    nan[2, 0, 0] = np.inf
    G["err_nonfinite/q"] = nan
    err("nonfinite", nan)
    err("nonfinite_ref", nan, engine="reference")
    late = base.copy()
    late[0, 39, 99] = -np.inf
    G["err_nonfinite_last/q"] = late
    err("nonfinite_last", late)
    G["err_infeasible/q"] = np.zeros((1, 3, 2), np.float32)
    err("infeasible", G["err_infeasible/q"])
    G["err_ragged/lengths"] = np.array([[40, 100], [0, 5], [30, 60]], np.int64)
    err("ragged", base, G["err_ragged/lengths"])
    G["err_ragged2/lengths"] = np.array([[40, 100], [30, 20], [5, 0]], np.int64)
    err("ragged2", base, G["err_ragged2/lengths"])
    err("mnv_m1e9", base, max_neg_val=-1e9)
    err("mnv_minf", base, max_neg_val=float("-inf"))
    err("mnv_nan", base, max_neg_val=float("nan"))
    err("threads", base, threads=-1)
    # the NaN item precedes a bad-length item: lowest index wins
    G["err_order/lengths"] = np.array([[40, 100], [40, 100], [41, 100]], np.int64)
    err("order", nan, np.array([[40, 100], [40, 100], [5, 3]], np.int64))

    # generator pins
    for (b, t, s, seed) in [(2, 8, 32, 5), (1, 64, 256, 0), (3, 7, 11, 2**63 + 5)]:
        G[f"gen_{b}_{t}_{s}_{seed}/sha"] = np.array(sha(ref.generate(b, t, s, seed)))

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT}: {len(G)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
