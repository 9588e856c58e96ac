"""The C-ABI boundary on CPU: the in-tree sm_100a library loads, exports
every symbol include/*.h declares, and the host-side validation that runs
before any device work reproduces the reference's codes and messages.  No
compute is launched here (no GPU in the build container)."""

from __future__ import annotations

import ctypes
import glob
import os
import re
import subprocess

import numpy as np
import pytest

from _golden import G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        names |= set(re.findall(r"MAS_API\s+[\w\s\*]+?\b(mas_\w+)\s*\(", src))
    return sorted(names)


def test_header_declares_entry_points():
    names = _declared_symbols()
    for must in ("mas_align_host", "mas_align_device", "mas_plan_create", "mas_plan_enqueue",
                 "mas_plan_finish", "mas_generate_device"):
        assert must in names


def test_library_exports_every_declared_symbol(mas):
    lib = mas._lib.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", mas._lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(_declared_symbols()) <= exported
    # only the C-ABI and the C++ mirror of the reference API (namespace
    # monoalign, mangled _ZN9monoalign...) are exported
    other = [n for n in exported if not n.startswith(("mas_", "_init", "_fini", "_ZN9monoalign"))]
    assert not other, other[:10]


def test_library_is_sm100a(mas):
    out = subprocess.run(["cuobjdump", "--list-elf", mas._lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tma_and_cluster_stores(mas):
    sass = subprocess.run(["cuobjdump", "-sass", mas._lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTMALDG" in sass  # TMA tile loads of q
    assert "UTMASTG" in sass  # TMA stores of the output zero tiles
    assert "STAS" in sass  # st.async DSMEM boundary-row FIFO


def test_config_default_and_names(mas):
    lib = mas._lib.load()
    cfg = mas._lib.MasConfig()
    lib.mas_config_default(ctypes.byref(cfg))
    assert cfg.engine == mas._lib.MAS_ENGINE_PARALLEL
    assert cfg.max_neg_val == np.float32(-1e32)
    assert cfg.threads == 0 and cfg.flags == 0
    assert lib.mas_abi_version() == 3
    for code, name in enumerate(mas._lib.ERRC_NAMES):
        assert lib.mas_errc_name(code).decode() == name
    assert lib.mas_errc_name(99).decode() == "Unknown"


@pytest.mark.parametrize("tag,kw", [("err_mnv_m1e9", {"max_neg_val": -1e9}),
                                    ("err_mnv_minf", {"max_neg_val": float("-inf")}),
                                    ("err_mnv_nan", {"max_neg_val": float("nan")}),
                                    ("err_threads", {"threads": -1})])
def test_invalid_config_message_matches_reference(mas, tag, kw):
    """validate_config runs before any device work (align_parallel,
    parallel.cpp:171-174), so this is checkable without a GPU."""
    q = np.zeros((3, 40, 100), np.float32)
    with pytest.raises(ValueError) as ei:
        mas.align(q, **kw)
    assert str(ei.value) == str(G()[f"{tag}/msg"])


def test_binding_argument_errors(mas):
    """module.cpp:21-84: rank, zero dims, lengths shape / range, engine name."""
    with pytest.raises(ValueError, match=r"values must be a \[T, S\] or \[B, T, S\] array"):
        mas.align(np.zeros(4, np.float32))
    with pytest.raises(ValueError, match="every array dimension must be at least 1"):
        mas.align(np.zeros((2, 0, 3), np.float32))
    with pytest.raises(ValueError, match=r"lengths must have shape \[B, 2\]"):
        mas.align(np.zeros((2, 3, 4), np.float32), lengths=np.zeros((3, 2)))
    with pytest.raises(ValueError, match=r"item 1: lengths must lie in \[0, T\] x \[0, S\]"):
        mas.align(np.zeros((2, 3, 4), np.float32), lengths=[[1, 1], [4, 4]])
    with pytest.raises(ValueError, match="unknown engine name: turbo"):
        mas.align(np.zeros((2, 3), np.float32), engine="turbo")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2409_07704_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
                assert "mas_oracle" not in src and "_ref/" not in src, f
