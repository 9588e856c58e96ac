"""Builds the in-tree CUDA library ``_lib/libmonoalign_b200.so`` for sm_100a.

One shared object holds the kernels (csrc/mas_fwd4.cu, csrc/mas_bt.cu, csrc/mas_scores.cu), the
extern "C" boundary (csrc/mas_abi.cu, include/monoalign_b200.h) and the C++
mirror of the reference API (csrc/monoalign_api.cpp, include/monoalign/).
The CUDA runtime is linked statically so the library does not clash with
torch's bundled libcudart.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libmonoalign_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
HOST_CXX = "/usr/bin/g++"  # dynamic libstdc++ 

SOURCES = ["mas_abi.cu", "mas_fwd4.cu", "mas_bt.cu", "monoalign_api.cpp",
           "mas_io.cpp", "mas_scores.cu", "mas_bench.cpp", "mas_gauss.cu"]
CLI = os.path.join(LIBDIR, "monoalign")  # the `monoalign` command line (tools/main.cpp surface)
HEADERS = ["mas_kernels.h", "mas_ptx.cuh", "mas_umma.cuh"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    inc = os.path.join(ROOT, "include")
    for dirpath, _, files in os.walk(inc):
        deps += [os.path.join(dirpath, f) for f in files]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compiles the library (``out``; ``defines`` are extra -D macros for
    experiment variants built next to the product library)."""
    if out == LIB and not defines and not force and not _stale():
        build_cli()
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [
        NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++20",
        "-ccbin", HOST_CXX, "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
        "-o", out,
    ] + [f"-D{d}" for d in defines] + [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc build of libmonoalign_b200.so failed")
    if verbose:
        sys.stderr.write(res.stderr)
    if out == LIB:
        build_cli(force=True)
    return out


def build_cli(force: bool = False) -> str:
    """The `monoalign` command line (csrc/mas_cli.cpp), linked to the library."""
    src = os.path.join(CSRC, "mas_cli.cpp")
    if not force and os.path.exists(CLI) and os.path.getmtime(CLI) >= max(
            os.path.getmtime(src), os.path.getmtime(LIB)):
        return CLI
    cmd = [HOST_CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           src, "-L", LIBDIR, "-lmonoalign_b200", "-Wl,-rpath,$ORIGIN", "-o", CLI]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build of the monoalign CLI failed")
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
