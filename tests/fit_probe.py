"""Fit-driver throughput probe (not a test): gpk_fit (device) vs the reference
fit (oracle/_ref, all host threads) on synthetic volumes; prints one JSON line
per configuration. Usage: python tests/fit_probe.py [c1|c2 ...]
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2603_20611_b200 as gp  # noqa: E402

CASES = {
    # dims, init_count, device iterations, reference iterations
    "c1": ((128, 128, 32), 20000, 3000, 600),
    "c2": ((512, 512, 128), 1000000, 3000, 12),
}


def volume(dims, seed=7):
    X, Y, Z = dims
    return np.random.default_rng(seed).uniform(0.0, 0.1, (Z, Y, X)).astype(np.float32)


def main(names):
    from oracle.bindings import load

    ref = load("ref")
    ref.lib.gref_set_threads(0)
    for name in names:
        dims, n0, iters, ref_iters = CASES[name]
        vol = volume(dims)
        cfg = gp.FitConfig(iterations=iters, init_count=n0, densify_start=100, densify_end=400,
                           densify_interval=100, rng_seed=1, progress_interval=100)
        rows = []
        with gp.Session(0) as s:
            t0 = time.perf_counter()
            s.fit(vol, (1, 1, 1), (0, 0, 0), gp.PsfSpec(), cfg,
                  lambda p: rows.append((p.iteration, p.loss, p.count, p.psnr2d)))
            dt = time.perf_counter() - t0
        rcfg = gp.FitConfig(iterations=ref_iters, init_count=n0, densify_start=100, densify_end=400,
                            densify_interval=100, rng_seed=1, progress_interval=100)
        c = rcfg.to_c()
        t0 = time.perf_counter()
        _, wrows = ref.fit(vol.astype(np.float64), (1, 1, 1), (0, 0, 0), gp.PsfSpec(),
                           {f: getattr(c, f) for f, _ in type(c)._fields_}, capacity=4 * n0 + 16)
        rdt = time.perf_counter() - t0
        print(json.dumps({
            "probe": "fit", "config": name, "dims": dims, "init_count": n0,
            "device": {"iterations": iters, "seconds": dt, "iterations_per_s": iters / dt,
                       "progress": rows},
            "reference": {"iterations": ref_iters, "seconds": rdt, "iterations_per_s": ref_iters / rdt,
                          "threads": os.cpu_count(), "progress": wrows.tolist()},
            "note": "wall clock of the whole fit call (init, volume upload, densify events, monitor)",
        }), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
