"""Checkpoint ingest / egress (checkpoint.hpp:38-97) of a resident session,
against the reference's own save_checkpoint / load_checkpoint (oracle/_ref):
files are byte-identical both ways, loads round-trip bitwise, and the
reference's error classes (LoadError, CorruptContainer) map 1:1.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu


def _ref_load(ref, path, cap):
    from oracle.bindings import Bounds

    L = ref.lib
    L.gref_load_checkpoint.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_uint64),
                                       C.POINTER(Bounds)]
    out = np.zeros((max(cap, 1), 11))
    n = C.c_uint64()
    b = Bounds()
    st = L.gref_load_checkpoint(str(path).encode(), out.ctypes.data_as(C.POINTER(C.c_double)), cap,
                                C.byref(n), C.byref(b))
    return st, out[:n.value], (tuple(b.min), tuple(b.max))


@pytest.mark.parametrize("n", [0, 1, 1000, 70001])
def test_checkpoint_bytes_match_reference(gp, ref, session, tmp_path, n):
    lo, hi = (-0.5, -1.5, 0.25), (31.5, 20.5, 9.75)
    gs = gp.init_random(max(n, 1), lo, hi, 1.5, 5)
    rec = f32(gs.records[:n])
    session.set_gaussians(gp.GaussianSet(rec, lo, hi))
    mine = tmp_path / "dev.gpile"
    session.save_checkpoint(mine)
    # the reference writes the same set
    theirs = tmp_path / "ref.gpile"
    h = ref._set(rec, (lo, hi))
    ref.lib.gref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
    assert ref.lib.gref_save_checkpoint(C.c_void_p(h.h), str(theirs).encode()) == 0
    assert mine.read_bytes() == theirs.read_bytes()
    assert mine.stat().st_size == gp.checkpoint_bytes(n)
    # reference file -> device -> records bitwise; device file -> reference
    with gp.Session(0) as s2:
        s2.load_checkpoint(theirs)
        assert s2.n == n
        assert np.array_equal(s2.get_gaussians().astype(np.float64), rec)
        assert s2.bounds() == (lo, hi)
    st, back, bb = _ref_load(ref, mine, n)
    assert st == 0 and np.array_equal(back, rec) and bb == (lo, hi)


def test_checkpoint_errors_map_to_reference_classes(gp, ref, session, tmp_path):
    gs = gp.init_random(50, (0, 0, 0), (8, 8, 8), 1.0, 3)
    session.set_gaussians(gs)
    good = tmp_path / "good.gpile"
    session.save_checkpoint(good)
    raw = good.read_bytes()
    cases = {
        "missing": (None, gp.LoadError, 9),
        "magic": (b"GPILX" + raw[5:], gp.CorruptContainer, 8),
        "version": (raw[:5] + (2).to_bytes(4, "little") + raw[9:], gp.CorruptContainer, 8),
        "header": (raw[:30], gp.CorruptContainer, 8),
        "records": (raw[:-7], gp.CorruptContainer, 8),
    }
    for name, (data, exc, code) in cases.items():
        p = tmp_path / f"{name}.gpile"
        if data is not None:
            p.write_bytes(data)
        with pytest.raises(exc):
            session.load_checkpoint(p)
        st, _, _ = _ref_load(ref, p, 100)
        assert st == code, name
    with pytest.raises(gp.LoadError):
        session.save_checkpoint(tmp_path / "no" / "such" / "dir.gpile")
    # a failed load leaves the session's set untouched
    assert session.n == 50
