"""Codec front-half throughput probe (not a test): gpk_encode_streams (Morton
sort + quantize + delta/zig-zag packing on the device, streams copied back to
the host) vs the reference's morton_sort + apply_permutation + quantize +
pack_deltas (oracle/_ref, single-threaded as the reference runs them), bitwise
equal outputs checked on the way. Prints one JSON line per size.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2603_20611_b200 as gp  # noqa: E402
import paper_2603_20611_b200._native as N  # noqa: E402

U32 = C.POINTER(C.c_uint32)


def main(sizes):
    from oracle.bindings import load

    ref = load("ref")
    ref.lib.gref_quantize.argtypes = [C.c_void_p, C.c_void_p, C.c_int, U32, U32, U32, U32,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
    ref.lib.gref_pack_deltas.argtypes = [U32, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
    spec = gp.QuantSpec()
    for n in sizes:
        gs = gp.init_random(n, (-0.5, -0.5, -0.5), (511.5, 511.5, 127.5), 1.5, 1)
        gs = gp.GaussianSet(gs.records.astype(np.float32).astype(np.float64), gs.bbox_min, gs.bbox_max)
        with gp.Session(0) as s:
            s.set_gaussians(gs)
            s.encode_streams(spec)  # warm-up
            reps = 5
            t0 = time.perf_counter()
            for _ in range(reps):
                enc = s.encode_streams(spec)
            dev = (time.perf_counter() - t0) / reps
        h = ref._set(gs.records, (gs.bbox_min, gs.bbox_max))
        t0 = time.perf_counter()
        q = [np.zeros(3 * n, np.uint32), np.zeros(n, np.uint32), np.zeros(3 * n, np.uint32), np.zeros(4 * n, np.uint32)]
        lo, hi = np.zeros(3), np.zeros(3)
        c = spec.to_c()
        assert ref.lib.gref_quantize(C.c_void_p(h.h), C.byref(c), 1, *[a.ctypes.data_as(U32) for a in q],
                                     N.dptr(lo), N.dptr(hi)) == 0
        outs = []
        for vals, comps, bits in zip(q, (3, 1, 3, 4), (14, 12, 12, 12)):
            b = np.zeros(vals.size * ((bits + 7) // 8), np.uint8)
            assert ref.lib.gref_pack_deltas(vals.ctypes.data_as(U32), vals.size, comps, bits,
                                            b.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
            outs.append(b)
        cpu = time.perf_counter() - t0
        same = all(np.array_equal(a, b) for a, b in zip((enc.positions, enc.opacities, enc.log_scales, enc.quats), outs))
        print(json.dumps({"probe": "codec_front_half", "n": n, "device_s": dev, "reference_s": cpu,
                          "speedup": cpu / dev, "bitwise_equal": same,
                          "stream_bytes": int(sum(o.size for o in outs)),
                          "note": "device time = wall clock of gpk_encode_streams incl. D2H of the streams; "
                                  "reference = morton_sort+apply_permutation+quantize+4x pack_deltas, 1 thread"}),
              flush=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [1_000_000, 8_000_000])
