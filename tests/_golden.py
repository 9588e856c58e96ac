"""Helpers over tests/golden/golden.npz (made by tests/golden/make_golden.py
from the unmodified reference)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
SENTINELS = {"m1e32": -1e32, "m1e9": -1e9, "minf": float("-inf")}
ENGINES = ("parallel", "reference")

_G = None


def G():
    global _G
    if _G is None:
        _G = dict(np.load(GOLDEN))
    return _G


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cases(prefix: str):
    """Tags present in the golden file whose name starts with `prefix`."""
    tags = set()
    for k in G():
        tag = k.split("/")[0]
        if tag.startswith(prefix):
            tags.add(tag)
    return sorted(tags)


def inputs(tag: str, gen):
    """(q, lengths) of a golden case; `gen(b, t, s, seed)` regenerates seeded
    inputs (checked against the stored SHA-256)."""
    g = G()
    lengths = g.get(f"{tag}/lengths")
    if f"{tag}/q" in g:
        q = g[f"{tag}/q"]
    elif tag.startswith("single_"):
        t, s = (int(x) for x in g[f"{tag}/dims"])
        q = gen(1, t, s, int(g[f"{tag}/seed"]))
    elif tag.startswith("batched_"):
        q = gen(32, 128, 512, int(g[f"{tag}/seed"]))
    elif tag.startswith("ragged_"):
        q = gen(4, 64, 256, int(g[f"{tag}/seed"]))
    elif tag == "adv":
        i = np.arange(32)[:, None]
        j = np.arange(2048)[None, :]
        q = np.where(i > j, np.float32(1e8), np.float32(-1e8)).astype(np.float32)
    elif tag == "c2":
        q = gen(32, 200, 800, 0)
    else:
        raise KeyError(tag)
    if f"{tag}/q_sha" in g:
        assert sha(q) == str(g[f"{tag}/q_sha"]), f"{tag}: regenerated input differs"
    return q, lengths


def expected(tag: str, engine: str, sentinel: str):
    g = G()
    key = f"{tag}/{engine}/{sentinel}/paths"
    if key not in g:
        return None, None
    return g[key], str(g[f"{tag}/{engine}/{sentinel}/out_sha"])


def paths_to_out(paths, T, S):
    """write_path (types.cpp:181-185) of [B][S] paths (-1 = past s_b)."""
    paths = np.asarray(paths)
    B = paths.shape[0]
    out = np.zeros((B, T, S), np.uint8)
    for b in range(B):
        j = np.nonzero(paths[b] >= 0)[0]
        out[b, paths[b, j], j] = 1
    return out
