"""The codec's front half on the device against the
reference's own morton.hpp / quant.hpp / container.hpp (oracle/_ref):
the stable Z-order permutation, the quantized attribute streams (set order and
encode()'s Morton order) and the delta + zig-zag packed byte streams are
bit-exact; the error paths name the same primitive.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu

U32 = C.POINTER(C.c_uint32)


def _u32(a):
    return a.ctypes.data_as(U32)


def _set(gp, n, seed, lo=(-2.0, 0.5, 1.0), hi=(30.0, 17.5, 9.0)):
    gs = gp.init_random(n, lo, hi, 1.5, seed)
    rec = f32(gs.records)
    rng = np.random.default_rng(seed)
    # some duplicated positions (equal codes at any depth) and negative-w quats
    dup = rng.choice(n, n // 10, replace=False)
    rec[dup, 0:3] = rec[rng.choice(n, n // 10), 0:3]
    rec[::7, 6:10] *= -1.0
    rec[::11, 6] = 0.0
    return gp.GaussianSet(rec, lo, hi)


def _ref_quant(ref, gs, spec, morton):
    from oracle.bindings import Bounds  # noqa: F401

    n = gs.size()
    h = ref._set(gs.records, (gs.bbox_min, gs.bbox_max))
    pos, opa = np.zeros(3 * n, np.uint32), np.zeros(n, np.uint32)
    ls, qt = np.zeros(3 * n, np.uint32), np.zeros(4 * n, np.uint32)
    lo, hi = np.zeros(3), np.zeros(3)
    import paper_2603_20611_b200._native as N

    c = spec.to_c()
    ref.lib.gref_quantize.argtypes = [C.c_void_p, C.c_void_p, C.c_int, U32, U32, U32, U32,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
    st = ref.lib.gref_quantize(C.c_void_p(h.h), C.byref(c), 1 if morton else 0, _u32(pos), _u32(opa), _u32(ls),
                               _u32(qt), N.dptr(lo), N.dptr(hi))
    msg = (ref.lib.gref_last_error() or b"").decode()
    return st, msg, (pos, opa, ls, qt, lo, hi)


@pytest.mark.parametrize("bits", [4, 14, 21])
def test_morton_sort_bitwise(gp, ref, session, bits):
    gs = _set(gp, 60000, bits)
    session.set_gaussians(gs)
    got = session.morton_sort(bits)
    h = ref._set(gs.records, (gs.bbox_min, gs.bbox_max))
    want = np.zeros(gs.size(), np.uint64)
    ref.lib.gref_morton_sort.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]
    assert ref.lib.gref_morton_sort(C.c_void_p(h.h), bits, want.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    assert np.array_equal(got, want)


@pytest.mark.parametrize("morton", [False, True])
def test_quantize_bitwise(gp, ref, session, morton):
    gs = _set(gp, 50000, 3)
    spec = gp.QuantSpec()
    session.set_gaussians(gs)
    q = session.quantize(spec, morton_order=morton)
    st, _, (pos, opa, ls, qt, lo, hi) = _ref_quant(ref, gs, spec, morton)
    assert st == 0
    assert np.array_equal(q.positions, pos) and np.array_equal(q.opacities, opa)
    assert np.array_equal(q.log_scales, ls) and np.array_equal(q.quats, qt)
    assert q.scale_min == tuple(lo) and q.scale_max == tuple(hi)


@pytest.mark.parametrize("spec_bits", [(14, 12, 12, 12, 14), (21, 4, 9, 16, 10)])
def test_encode_streams_bitwise(gp, ref, session, spec_bits):
    gs = _set(gp, 40000, 8)
    spec = gp.QuantSpec(*spec_bits)
    session.set_gaussians(gs)
    enc = session.encode_streams(spec)
    st, _, (pos, opa, ls, qt, lo, hi) = _ref_quant(ref, gs, spec, True)
    assert st == 0
    ref.lib.gref_pack_deltas.argtypes = [U32, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
    for got, vals, comps, bits in ((enc.positions, pos, 3, spec.pos_bits), (enc.opacities, opa, 1, spec.opacity_bits),
                                   (enc.log_scales, ls, 3, spec.scale_bits), (enc.quats, qt, 4, spec.quat_bits)):
        want = np.zeros(got.size, np.uint8)
        assert ref.lib.gref_pack_deltas(_u32(vals), vals.size, comps, bits,
                                        want.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
        assert np.array_equal(got, want), (comps, bits)
    assert enc.scale_min == tuple(lo) and enc.scale_max == tuple(hi)


def test_quantize_errors_match_reference(gp, ref, session):
    base = _set(gp, 5000, 4)
    for col, val, morton in ((4, np.nan, False), (1, np.inf, True), (None, 0.0, False)):
        rec = base.records.copy()
        if col is None:
            rec[1234, 6:10] = 0.0  # zero quaternion
        else:
            rec[[777, 3000], col] = val
        gs = gp.GaussianSet(rec, base.bbox_min, base.bbox_max)
        session.set_gaussians(gs)
        with pytest.raises(gp.InvalidArgument) as e:
            session.quantize(gp.QuantSpec(), morton_order=morton)
        st, msg, _ = _ref_quant(ref, gs, gp.QuantSpec(), morton)
        assert st == 1 and str(e.value) == msg
    with pytest.raises(gp.InvalidArgument):
        session.quantize(gp.QuantSpec(pos_bits=22))


def test_decode_streams_matches_reference(gp, ref, session):
    """encode_streams -> decode_streams on the device vs the reference's
    unpack_deltas + dequantize of the same bytes (container.hpp:158-181,
    quant.hpp:134-176): the records equal the reference's rounded to fp32
    (log / division in fp64 on both sides: within one fp32 ulp)."""
    import paper_2603_20611_b200._native as N

    gs = _set(gp, 30000, 9)
    spec = gp.QuantSpec()
    session.set_gaussians(gs)
    enc = session.encode_streams(spec)
    n = gs.size()
    bbox = (gs.bbox_min, gs.bbox_max)
    with gp.Session(0) as s2:
        got = s2.decode_streams(enc, n, bbox, spec, load=True)
        assert s2.n == n
        assert np.array_equal(s2.get_gaussians(), got)
    vals = []
    ref.lib.gref_unpack_deltas.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.c_uint64, C.c_int, C.c_int, U32]
    for b, comps, bits in ((enc.positions, 3, 14), (enc.opacities, 1, 12), (enc.log_scales, 3, 12), (enc.quats, 4, 12)):
        v = np.zeros(n * comps, np.uint32)
        assert ref.lib.gref_unpack_deltas(b.ctypes.data_as(C.POINTER(C.c_uint8)), b.size, n, comps, bits, _u32(v)) == 0
        vals.append(v)
    want = np.zeros((n, 11))
    b = N.Bounds((C.c_double * 3)(*bbox[0]), (C.c_double * 3)(*bbox[1]))
    lo, hi = np.array(enc.scale_min), np.array(enc.scale_max)
    c = spec.to_c()
    ref.lib.gref_dequantize.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), U32, U32, U32, U32, C.POINTER(C.c_double)]
    assert ref.lib.gref_dequantize(C.byref(c), n, C.byref(b), N.dptr(lo), N.dptr(hi), *[_u32(v) for v in vals],
                                   N.dptr(want)) == 0
    w32 = want.astype(np.float32)
    ulp = np.abs(np.spacing(w32))
    assert np.all(np.abs(got - w32) <= ulp), np.abs(got - w32).max()
    # a corrupted delta (zig-zag value >= 2^bits) is refused like the reference
    bad = gp.QuantizedStreams(enc.positions.copy(), enc.opacities.copy(), enc.log_scales, enc.quats,
                              enc.scale_min, enc.scale_max)
    bad.opacities[1::2][5] = 0xFF  # high byte of a 12-bit delta
    with gp.Session(0) as s3, pytest.raises(gp.CorruptContainer):
        s3.decode_streams(bad, n, bbox, spec)
