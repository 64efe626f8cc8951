"""GPU: the C++ drop-in (include/gpile_b200.hpp) against the reference's own
C++ functions in one binary (tests/cpp/dropin_parity.cpp): the fit-loop call
sequence prepare -> rasterize -> loss -> backward -> adam, random-pose
rasterize/backward, voxelize/voxelize_backward and the exception types.
The binary is built in the build container (needs the reference headers) and
shipped prebuilt; it links the in-tree libgpile_b200.so."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "dropin_parity"


def test_cpp_dropin_matches_reference():
    if not BIN.exists():
        pytest.skip("tests/cpp/_build/dropin_parity not built (needs /root/reference headers)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN PARITY OK" in r.stdout
