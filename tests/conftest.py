"""Shared fixtures. Markers: `gpu` needs a B200 (cuda:0); everything else runs on CPU."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (always buildable: plain gcc)."""
    from oracle.bindings import ORACLE_SO, build, load

    if not ORACLE_SO.exists():
        build(ref=False)
    return load("oracle")


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref), built here from /root/reference and shipped prebuilt."""
    from oracle.bindings import REF_SO, available, build, load

    if not REF_SO.exists() and Path("/root/reference/proj/include").exists():
        build(ref=True)
    if not available("ref"):
        pytest.skip("oracle/_ref/libgpile_ref.so not built (no /root/reference here)")
    return load("ref")


@pytest.fixture(scope="session")
def gp():
    import paper_2603_20611_b200 as gp

    return gp


@pytest.fixture
def session(gp):
    s = gp.Session(0)
    yield s
    s.close()


def f32(a):
    """Round to the device's stored precision (both sides see identical inputs)."""
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)
