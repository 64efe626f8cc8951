"""Parity report: GPU path vs the reference (oracle/_ref) and the C oracle.

Prints error statistics per config; used to set and justify the tolerances
in the -m gpu tests. Run on a GPU box:  python tests/parity_report.py [--big]
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2603_20611_b200 as gp  # noqa: E402
from oracle.bindings import available, load  # noqa: E402


def grad_err(g, r):
    scale = np.abs(r).max(axis=0) + 1e-300
    rel = np.abs(g - r) / (np.abs(r) + 1e-3 * scale)
    return float(rel.max()), float((np.abs(g - r) / scale).max())


def report(name, n, dims, k, sigma_z=1.0, tau=0.02, seed=1, ref=None):
    ck = ref or load("oracle")
    lo = (-0.5, -0.5, -0.5)
    hi = (dims[0] - 0.5, dims[1] - 0.5, dims[2] - 0.5)
    gs = gp.init_random(n, lo, hi, 1.5, seed)
    rec = gs.records.astype(np.float32).astype(np.float64)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k)
    psf = gp.PsfSpec(sigma_z=sigma_z)
    cfg = gp.RasterConfig(tau=tau)
    rng = np.random.default_rng(5)
    P = dims[0] * dims[1]
    dl = (rng.uniform(-1, 1, (dims[1], dims[0])) / P).astype(np.float32)
    s = gp.Session(0)
    s.set_gaussians(gp.GaussianSet(rec, lo, hi))
    t0 = time.time()
    s.prepare(pose, psf, cfg)
    img = s.rasterize()
    grads = s.backward(dl)
    t_gpu = time.time() - t0
    prep = s.prepared()
    off, ent = s.tile_lists()
    t0 = time.time()
    idx, bnd, fld = ck.prepare(rec, pose, psf, cfg)
    roff, rent = ck.tile_lists(rec, pose, psf, cfg)
    rimg = ck.rasterize(rec, pose, psf, cfg)
    rg, _ = ck.backward(rec, pose, psf, cfg, dl.astype(np.float64))
    t_cpu = time.time() - t0
    same_idx = np.array_equal(prep.index, idx)
    same_b = same_idx and np.array_equal(prep.bounds, bnd)
    same_t = np.array_equal(off, roff) and np.array_equal(ent, rent)
    peak = np.abs(rimg).max()
    rel = np.abs(img - rimg) / np.maximum(np.abs(rimg), 1e-300)
    big = np.abs(rimg) > 1e-3 * peak
    e_img_rel = float(rel[big].max()) if big.any() else 0.0
    e_img_abs = float(np.abs(img - rimg).max() / max(peak, 1e-300))
    ge = grad_err(grads.astype(np.float64), rg)
    print(f"[{name}] n={n} S={len(idx)}/{len(prep.index)} T={len(rent)}/{len(ent)} "
          f"idx={same_idx} bounds={same_b} tiles={same_t} img_rel(>1e-3pk)={e_img_rel:.2e} "
          f"img_abs/pk={e_img_abs:.2e} grad_rel(floor1e-3)={ge[0]:.2e} grad_abs/plane={ge[1]:.2e} "
          f"gpu={t_gpu:.3f}s cpu={t_cpu:.3f}s", flush=True)
    if not same_idx:
        a, b = set(prep.index.tolist()), set(idx.tolist())
        print("   only gpu:", sorted(a - b)[:10], " only ref:", sorted(b - a)[:10])
    s.close()


def main():
    ref = load("ref") if available("ref") else None
    print("checker:", "reference (oracle/_ref)" if ref else "C restatement")
    report("C1 k=16", 20000, (128, 128, 32), 16, ref=ref)
    report("C1 k=0", 20000, (128, 128, 32), 0, ref=ref)
    report("C1 tau=0", 20000, (128, 128, 32), 7, tau=0.0, ref=ref)
    report("C3-like sz=3", 50000, (256, 256, 320), 160, sigma_z=3.0, ref=ref)
    if "--big" in sys.argv:
        report("C2 k=64", 1000000, (512, 512, 128), 64, ref=ref)


if __name__ == "__main__":
    main()
