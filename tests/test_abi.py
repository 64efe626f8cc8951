"""CPU: the C-ABI boundary (include/gpile_b200.h) without a GPU.

* the in-tree sm_100a library loads and exports every symbol the header
  declares (and the ctypes prototypes cover all of them);
* the library really is sm_100a device code (cuobjdump lists the arch);
* host-only entry points agree with the reference: init_random's seeded stream
  bit for bit, slice_pose_for_index, lr_at;
* device entry points fail cleanly (status code + message, no crash) when no
  GPU is present, and the Python layer refuses to run without the library
  (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol(gp):
    from paper_2603_20611_b200 import _native as N

    declared = N.declared_symbols()
    assert len(declared) >= 50
    raw = C.CDLL(str(N.LIB_PATH))
    missing = [s for s in declared if not hasattr(raw, s)]
    assert not missing, f"declared in include/gpile_b200.h but not exported: {missing}"
    unbound = [s for s in declared if s not in N._PROTOS]
    assert not unbound, f"no ctypes prototype for: {unbound}"
    assert N.lib.gpk_abi_version() == N.GPK_ABI_VERSION


def test_library_is_sm100a_code(gp):
    from paper_2603_20611_b200 import _native as N

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_random_bitwise_equals_reference(gp, ref):
    """init_random (optimize.hpp:94-108) on the reference's mt19937_64 stream."""
    from oracle.bindings import Bounds

    lo, hi = (-0.5, -1.0, 2.0), (30.5, 20.0, 9.0)
    got = gp.init_random(5000, lo, hi, 1.5, 42).records
    want = np.zeros_like(got)
    b = Bounds((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
    ref.lib.gref_init_random.argtypes = [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64,
                                         C.POINTER(C.c_double)]
    assert ref.lib.gref_init_random(5000, C.byref(b), 1.5, 42, want.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert np.array_equal(got, want)


def test_slice_pose_for_index_matches_reference(gp, ref):
    """slice_pose_for_index (core.hpp:202-211)."""
    from oracle.bindings import PoseC

    dims = np.array([40, 30, 12], np.int32)
    sp = np.array([0.5, 0.75, 2.0])
    o = np.array([1.0, -2.0, 3.5])
    for k in (0, 5, 11):
        p = gp.slice_pose_for_index(tuple(dims), tuple(sp), tuple(o), k)
        q = PoseC()
        ref.lib.gref_slice_pose_for_index.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                                      C.POINTER(C.c_double), C.c_int, C.POINTER(PoseC)]
        assert ref.lib.gref_slice_pose_for_index(dims.ctypes.data_as(C.POINTER(C.c_int32)),
                                                 sp.ctypes.data_as(C.POINTER(C.c_double)),
                                                 o.ctypes.data_as(C.POINTER(C.c_double)), k, C.byref(q)) == 0
        assert np.array_equal(np.asarray(p.rotation).reshape(9), np.array(q.rotation[:]))
        assert tuple(p.translation) == tuple(q.translation[:])
        assert (p.width, p.height) == (q.width, q.height)
        assert tuple(p.pixel_spacing) == tuple(q.pixel_spacing[:])


def test_lr_schedule_matches_reference(gp, ref):
    """lr_at (optimize.hpp:71-73); test_optim.cpp:148-151."""
    for lr0, it, tot in ((6e-4, 1, 30000), (6e-4, 15000, 30000), (0.02, 30000, 30000), (1e-3, 7, 10)):
        assert gp.lr_at(lr0, it, tot) == ref.lib.gref_lr_at(lr0, it, tot)


def test_device_calls_fail_cleanly_without_gpu(gp):
    """No device here: session creation returns a CUDA status and a message."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2603_20611_b200 import _native as N

    h = C.c_void_p()
    st = N.lib.gpk_session_create(0, None, C.byref(h))
    assert st != N.GPK_OK
    assert N.lib.gpk_last_error_message()
    with pytest.raises(Exception):
        gp.Session(0)


def test_null_arguments_rejected(gp):
    from paper_2603_20611_b200 import _native as N

    assert N.lib.gpk_session_destroy(None) == N.GPK_OK
    assert N.lib.gpk_session_synchronize(None) == N.GPK_ERR_INVALID_ARGUMENT
    assert N.lib.gpk_prepare(None, None, None, None) == N.GPK_ERR_INVALID_ARGUMENT
    assert b"null" in N.lib.gpk_last_error_message()


def test_python_layer_refuses_without_library(tmp_path):
    """The product path has no CPU fallback: a package copy without _lib fails to import."""
    pkg = tmp_path / "paper_2603_20611_b200"
    shutil.copytree(ROOT / "paper_2603_20611_b200", pkg, ignore=shutil.ignore_patterns("_lib", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2603_20611_b200"], cwd=tmp_path,
                       capture_output=True, text=True, env={**os.environ, "PYTHONPATH": str(tmp_path)})
    assert r.returncode != 0 and "missing" in r.stderr
