"""Shared fixtures.  Tests marked ``gpu`` need a B200 (run with -m gpu on
the GPU box); everything else runs on CPU."""

from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size configuration (seconds of CPU oracle)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.build()
    return o.Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference engines (oracle/_ref), when they were built."""
    from oracle import oracle as o

    if not o.Reference.available():
        o.build()
    if not o.Reference.available():
        pytest.skip("reference library oracle/_ref not built (no /root/reference at build time)")
    return o.Reference()


@pytest.fixture(scope="session")
def mas():
    """The product package; on the GPU box its CUDA library must load."""
    import paper_2409_07704_b200 as m

    m._lib.load()
    return m


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    return torch.device("cuda:0")
