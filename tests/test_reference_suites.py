"""The reference's OWN tests, run unmodified against the B200 build.

oracle/Makefile (target ``dropin``, run by ``build()`` where /root/reference
exists) compiles, from /root/reference/proj without modification:

* ``bindings/module.cpp`` -> ``oracle/_ref/dropin/monoalign/_monoalign*.so``,
  against include/monoalign/ and linked to libmonoalign_b200.so -- the
  reference's pybind11 module over our library (module.cpp:206-248), next to
  the reference's ``python/monoalign/__init__.py``;
* ``tests/test_{types,reference,parallel,io,oracle}.cpp`` + ``doctest_main.cpp``
  -> ``oracle/_ref/dropin/unit`` against the same headers and library, with
  the doctest stand-in of tests/cpp/doctest_shim and the reference's
  exhaustive oracle (src/oracle.cpp, test infrastructure as in the reference's
  own test build, tests/CMakeLists.txt:1-12);

and stages ``tests/python/test_smoke.py`` unmodified.  The GPU tests below run
them on the B200: the reference's 14 Python smoke tests against both the
reference binding over our library and this repo's ``monoalign`` package, and
the reference's doctest suites file by file.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROP = os.path.join(ROOT, "oracle", "_ref", "dropin")
UNIT = os.path.join(DROP, "unit")
SMOKE = os.path.join(DROP, "tests", "test_smoke.py")
SUITES = ["test_types", "test_reference", "test_parallel", "test_io", "test_oracle", "test_bench"]
ACCEPT = os.path.join(DROP, "acceptance")
CLI_TESTS = os.path.join(DROP, "cli_tests")
CLI = os.path.join(ROOT, "paper_2409_07704_b200", "_lib", "monoalign")


def _binding():
    d = os.path.join(DROP, "monoalign")
    if not os.path.isdir(d):
        return None
    for f in os.listdir(d):
        if f.startswith("_monoalign") and f.endswith(".so"):
            return os.path.join(d, f)
    return None


def _need_dropin():
    if not all(os.path.exists(p) for p in (UNIT, SMOKE, ACCEPT, CLI_TESTS)) or not _binding():
        pytest.skip("drop-in programs not built (oracle/Makefile dropin needs /root/reference "
                    "at build time)")


def _needed(path):
    out = subprocess.run(["readelf", "-d", path], capture_output=True, text=True, check=True).stdout
    return [line.split("[")[1].split("]")[0] for line in out.splitlines() if "(NEEDED)" in line]


def test_dropin_programs_link_our_library_only():
    _need_dropin()
    for path in (UNIT, ACCEPT, CLI_TESTS, _binding()):
        needed = _needed(path)
        assert "libmonoalign_b200.so" in needed, (path, needed)
        assert not any("monoalign_ref" in n or "monoalign_core" in n for n in needed), needed


def test_dropin_binding_imports():
    _need_dropin()
    code = "import monoalign, sys; print(monoalign.__version__, monoalign._monoalign.__file__)"
    res = subprocess.run([sys.executable, "-c", code], cwd=DROP, capture_output=True, text=True,
                         env={**os.environ, "PYTHONPATH": DROP}, timeout=120)
    assert res.returncode == 0, res.stderr
    version, path = res.stdout.split()
    assert version == "1.0.0" and path == _binding()


def test_repo_monoalign_package_is_the_gpu_path():
    import monoalign
    import paper_2409_07704_b200.api as api

    assert monoalign.__version__ == "1.0.0"
    for name in monoalign.__all__:
        assert getattr(monoalign, name) is getattr(api, name), name


def _run_smoke(cwd, pythonpath):
    return subprocess.run(
        [sys.executable, "-m", "pytest", SMOKE, "-q", "-p", "no:cacheprovider", "--rootdir",
         os.path.dirname(SMOKE)],
        cwd=cwd, capture_output=True, text=True, timeout=600,
        env={**os.environ, "PYTHONPATH": pythonpath})


@pytest.mark.gpu
def test_reference_python_smoke_on_reference_binding(cuda):
    """proj/tests/python/test_smoke.py against the reference's own pybind11
    module compiled over libmonoalign_b200.so."""
    _need_dropin()
    res = _run_smoke(DROP, DROP)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "14 passed" in res.stdout, res.stdout


@pytest.mark.gpu
def test_reference_python_smoke_on_repo_package(cuda):
    """The same file against this repo's ``monoalign`` package."""
    _need_dropin()
    res = _run_smoke(ROOT, ROOT)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "14 passed" in res.stdout, res.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite(cuda, suite):
    _need_dropin()
    res = subprocess.run([UNIT, suite + ".cpp"], capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "failed checks: 0" in res.stdout, res.stdout + res.stderr
    assert "test cases: 0," not in res.stdout


@pytest.mark.gpu
def test_reference_acceptance(cuda):
    """proj/tests/acceptance.cpp (8 criteria: exhaustive oracle over 1000
    instances, engine equivalence over 1000 + 100 + 50 batches, invariants,
    sentinel adversarial, scaling law, speedup (soft), IO, trivia)."""
    _need_dropin()
    res = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=1800)
    fails = [ln for ln in res.stdout.splitlines() if ln.startswith("[FAIL]")]
    if res.returncode != 0 and fails and all(ln.startswith("[FAIL] 5.") for ln in fails):
        # Criterion 5 is a wall-clock fit (R^2 of host-path medians over
        # T*S); on a shared host a burst of memory-bandwidth contention during
        # one size's repeats can sink it.  Only that timing criterion gets one
        # re-run; every correctness criterion must pass the first time.
        res = subprocess.run([ACCEPT], capture_output=True, text=True, timeout=1800)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "acceptance: all gated criteria passed" in res.stdout, res.stdout


@pytest.mark.gpu
def test_reference_cli_driver(cuda):
    """proj/tests/cli_driver.cpp against this repo's `monoalign` CLI."""
    _need_dropin()
    res = subprocess.run([CLI_TESTS], capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "failed checks: 0" in res.stdout


def _cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=60)


@pytest.mark.parametrize("args,code", [
    ((), 2), (("frobnicate",), 2), (("--help",), 0), (("align", "--help"), 0),
    (("verify", "--t-max", "7"), 2), (("verify", "--s-max", "11"), 2), (("verify", "--t-max", "0"), 2),
    (("align", "--input", "a", "--output", "b", "--engine", "turbo"), 2),
    (("align", "--input", "a"), 2),
    (("bench", "--engines", "turbo", "--t-values", "8"), 2),
    (("bench", "--t-values", "8", "--repeats", "0"), 2),
    (("bench", "--format", "xml"), 2),
    (("align", "--input", "/no/such/file.bin", "--output", "/tmp/x.bin"), 1),
])
def test_cli_usage_and_exit_codes(args, code):
    """tools/main.cpp exit codes that need no device (usage 2, IO 1)."""
    from paper_2409_07704_b200 import build as b

    b.build()
    assert _cli(*args).returncode == code, args
