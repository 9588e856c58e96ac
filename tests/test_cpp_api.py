"""The C++ drop-in (include/monoalign/*.hpp over libmonoalign_b200.so): a
program written against the reference's public C++ API builds and links
here (CPU) and passes the reference's known answers on the GPU."""

from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "test_api")


def build_cpp_test(force: bool = False) -> str:
    from paper_2409_07704_b200 import build as b

    lib = b.build()
    if not force and os.path.exists(BIN) and os.path.getmtime(BIN) >= max(
            os.path.getmtime(SRC), os.path.getmtime(lib)):
        return BIN
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(lib)
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", libdir, "-lmonoalign_b200",
                    "-Wl,-rpath," + os.path.relpath(libdir, os.path.dirname(BIN)).join(
                        ["$ORIGIN/", ""]), "-o", BIN], check=True)
    return BIN


def test_cpp_api_builds_and_links():
    path = build_cpp_test()
    assert os.path.exists(path)


@pytest.mark.gpu
def test_cpp_api_known_answers(cuda):
    path = build_cpp_test()
    res = subprocess.run([path], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ALL OK" in res.stdout
