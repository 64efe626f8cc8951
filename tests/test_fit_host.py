"""Host side of the fit driver, checked against the reference (oracle/_ref) on
CPU: the seeded generator the slice sampler and the split draws use (Rng,
rng.hpp:14-70), init_grid (optimize.hpp:111-133), default_init_count
(optimize.hpp:64-66) and FitConfig validation (optimize.hpp:45-58). No GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest


def test_rng_stream_equals_reference(gp, ref):
    from oracle.bindings import RefRng

    for seed in (0, 7, 0x9E3779B97F4A7C15 + 21):
        a, b = gp.Rng(seed), RefRng(seed)
        for k in range(200):
            # interleave the draws fit makes (below for the slice, normal for splits)
            if k % 3 == 0:
                assert a.below(37) == b.below(37)
            elif k % 3 == 1:
                assert a.normal() == b.normal()
            else:
                assert a.uniform() == b.uniform()


def test_init_grid_bitwise_equals_reference(gp, ref):
    from oracle.bindings import Bounds

    lo, hi = (-0.5, -0.5, -0.5), (15.5, 11.5, 7.5)
    for n in (1, 27, 28, 1000, 1048):
        got = gp.init_grid(n, lo, hi, 1.5, 9).records
        want = np.zeros_like(got)
        b = Bounds((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
        ref.lib.gref_init_grid.argtypes = [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64,
                                           C.POINTER(C.c_double)]
        assert ref.lib.gref_init_grid(n, C.byref(b), 1.5, 9, want.ctypes.data_as(C.POINTER(C.c_double))) == 0
        assert np.array_equal(got, want), n


def test_default_init_count(gp, ref):
    # test_optim.cpp:371-375
    assert gp.default_init_count(64 * 64 * 64) == 1048
    assert gp.default_init_count(1000000000) == 100000
    assert gp.default_init_count(10) == 1
    ref.lib.gref_default_init_count.restype = C.c_uint64
    ref.lib.gref_default_init_count.argtypes = [C.c_uint64]
    for v in (0, 10, 999, 250001, 64**3, 512 * 512 * 128):
        assert gp.default_init_count(v) == ref.lib.gref_default_init_count(v)


def test_fit_config_validation(gp):
    """test_optim.cpp:377-388: FitConfig::validate runs before any device work
    (a null session reaches the validation first, so this needs no GPU)."""
    from paper_2603_20611_b200 import _native as N

    dims = np.array([4, 4, 4], np.int32)
    sp = np.ones(3)
    org = np.zeros(3)
    psf = gp.PsfSpec().to_c()

    def status(**kw):
        c = gp.FitConfig(**kw).to_c()
        st = N.lib.gpk_fit(None, None, N.i32ptr(dims), N.dptr(sp), N.dptr(org), C.byref(psf), C.byref(c),
                           N.PROGRESS_FN(), None)
        return st, N.lib.gpk_last_error_message().decode()

    st, msg = status()
    assert st == N.GPK_ERR_INVALID_ARGUMENT and "null session" in msg  # the config itself is valid
    for bad in (dict(lam=-0.1), dict(densify_start=30000), dict(iterations=0), dict(tau=1.0),
                dict(densify_interval=0), dict(lr_scale=0.0)):
        st, msg = status(**bad)
        assert st == N.GPK_ERR_INVALID_ARGUMENT and msg.startswith("FitConfig"), (bad, msg)


def test_fit_config_layout_matches_header(gp):
    """gpk_fit_config is passed by pointer: the ctypes mirror must match the C layout."""
    from paper_2603_20611_b200 import _native as N
    from oracle.bindings import FitCfgC

    assert C.sizeof(N.FitConfigC) == C.sizeof(FitCfgC)
    assert [f[0] for f in N.FitConfigC._fields_] == [f[0] for f in FitCfgC._fields_]
    c = gp.FitConfig().to_c()
    assert c.iterations == 30000 and c.densify_start == 500 and c.densify_end == 25000
    with pytest.raises(gp.InvalidArgument):
        gp.FitConfig(init_mode="hexagonal").to_c()


def test_reference_pack_unpack_round_trip(ref):
    """The reference's pack_deltas / unpack_deltas (container.hpp:136-181), built
    into oracle/_ref against the declaration-only lzma stub, invert each other."""
    U32 = C.POINTER(C.c_uint32)
    rng = np.random.default_rng(2)
    for comps, bits in ((3, 14), (1, 12), (4, 21), (3, 4)):
        v = rng.integers(0, 1 << bits, 999 * comps).astype(np.uint32)
        w = (bits + 7) // 8
        b = np.zeros(v.size * w, np.uint8)
        ref.lib.gref_pack_deltas.argtypes = [U32, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
        assert ref.lib.gref_pack_deltas(v.ctypes.data_as(U32), v.size, comps, bits,
                                        b.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
        back = np.zeros_like(v)
        ref.lib.gref_unpack_deltas.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.c_uint64, C.c_int, C.c_int, U32]
        assert ref.lib.gref_unpack_deltas(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.size, 999, comps, bits,
                                          back.ctypes.data_as(U32)) == 0
        assert np.array_equal(back, v)
