"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

    python tests/golden/make_golden.py      (needs oracle/_ref, i.e. /root/reference)

The reference ships no golden vectors: its tests regenerate
scenes from its seeded Rng. This script runs the REAL reference (header-only
C++ compiled by oracle/Makefile into oracle/_ref/libgpile_ref.so) on small,
seeded scenes and stores inputs and outputs as .npz, so the checks in
tests/test_oracle.py and the GPU parity tests have vectors that travel to
machines without /root/reference. Scenes follow the reference's own test
fixtures (proj/tests/test_render.cpp, test_grad.cpp, test_loss.cpp,
test_optim.cpp, test_voxelize.cpp).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.bindings import RefRng, load  # noqa: E402

OUT = Path(__file__).resolve().parent


def pose(w, h, rot=None, t=(0.0, 0.0, 0.0), sp=(1.0, 1.0), pp=(0.0, 0.0)):
    return NS(rotation=np.eye(3) if rot is None else np.asarray(rot, np.float64).reshape(3, 3),
              translation=tuple(t), width=w, height=h, pixel_spacing=tuple(sp), principal_point=tuple(pp))


def pose_of(pc):
    return pose(pc.width, pc.height, np.array(pc.rotation[:]).reshape(3, 3), tuple(pc.translation[:]),
                tuple(pc.pixel_spacing[:]), tuple(pc.principal_point[:]))


def psf(sz=1.0):
    return NS(sigma_x=1.0, sigma_y=1.0, sigma_z=sz)


def rcfg(tau=0.02, fs=3.0, mod=1.0):
    return NS(tau=tau, tile_size=16, footprint_sigmas=fs, scale_modifier=mod)


def pose_dict(p):
    return {"rotation": np.asarray(p.rotation, np.float64).reshape(9).tolist(),
            "translation": list(p.translation), "width": p.width, "height": p.height,
            "pixel_spacing": list(p.pixel_spacing), "principal_point": list(p.principal_point)}


def init_random(ref, n, lo, hi, scale, seed):
    """init_random (optimize.hpp:94-108) through the reference's own Rng stream."""
    import ctypes as C

    from oracle.bindings import Bounds
    rec = np.zeros((n, 11), np.float64)
    b = Bounds((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
    ref.lib.gref_init_random.argtypes = [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64,
                                         C.POINTER(C.c_double)]
    st = ref.lib.gref_init_random(n, C.byref(b), scale, seed, rec.ctypes.data_as(C.POINTER(C.c_double)))
    assert st == 0
    return rec


def render_case(ref, name, rec, p, f, c, bbox, dl_seed, dl_scale):
    idx, bnd, fld = ref.prepare(rec, p, f, c, bbox)
    off, ent = ref.tile_lists(rec, p, f, c, bbox)
    img = ref.rasterize(rec, p, f, c, bbox)
    dl = (np.random.default_rng(dl_seed).uniform(-1.0, 1.0, (p.height, p.width)) * dl_scale).astype(
        np.float32).astype(np.float64)  # inputs exactly representable on the f32 device
    g, (nrm, obs, wld) = ref.backward(rec, p, f, c, dl, bbox)
    meta = {"pose": pose_dict(p), "psf": [f.sigma_x, f.sigma_y, f.sigma_z],
            "cfg": [c.tau, c.tile_size, c.footprint_sigmas, c.scale_modifier],
            "bbox": [list(bbox[0]), list(bbox[1])]}
    np.savez_compressed(OUT / f"{name}.npz", meta=json.dumps(meta), records=rec, index=idx, bounds=bnd,
                        fields=fld, offsets=off, entries=ent, image=img, dl_di=dl, grads=g, stat_norm=nrm,
                        stat_observed=obs, stat_world=wld)
    print(f"{name}: n={len(rec)} survivors={len(idx)} pairs={len(ent)}")


def main():
    ref = load("ref")
    # 1. stack scene (C1-like geometry, reduced): init_random, mid slices, default config
    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (dims[0] - 0.5, dims[1] - 0.5, dims[2] - 0.5)
    rec = init_random(ref, 3000, lo, hi, 1.5, 1).astype(np.float32).astype(np.float64)
    for k in (3, 6):
        p = pose(dims[0], dims[1], t=(0.0, 0.0, -float(k)))
        render_case(ref, f"render_stack_k{k}", rec, p, psf(), rcfg(), (lo, hi), k, 1.0 / (dims[0] * dims[1]))
    # 2. random poses, tau = 0, footprint 8 sigma (test_grad.cpp:128-177 scenes)
    rng = RefRng(11)
    bb = ((-3.0, -3.0, -3.0), (3.0, 3.0, 3.0))
    prims = np.stack([rng.random_primitive(bb, 0.5, 2.0) for _ in range(40)]).astype(np.float32).astype(np.float64)
    p = pose_of(rng.random_pose_c(24, 20))
    render_case(ref, "render_random_pose", prims, p, psf(0.8), rcfg(0.0, 8.0), bb, 5, 0.05)
    # 3. thick PSF, scale modifier, non-unit spacing, shifted principal point
    rec3 = init_random(ref, 1500, (0, 0, 0), (40.0, 30.0, 20.0), 1.2, 7).astype(np.float32).astype(np.float64)
    p = pose(50, 40, t=(0.0, 0.0, -9.5), sp=(0.8, 0.75), pp=(2.5, -1.5))
    render_case(ref, "render_thick_psf", rec3, p, psf(3.0), rcfg(0.01, 3.0, 1.3), ((0, 0, 0), (40, 30, 20)), 9,
                1e-3)

    # 4. photometric loss (loss.hpp:13 / metrics.hpp:187)
    r = np.random.default_rng(3)
    ren = r.uniform(0.0, 1.0, (29, 37)).astype(np.float32).astype(np.float64)   # device stores f32
    tgt = r.uniform(0.0, 1.0, (29, 37)).astype(np.float32).astype(np.float64)
    out = {}
    for lam in (0.0, 0.2, 1.0):
        L, dl = ref.loss(ren, tgt, lam, 0.5)
        out[f"loss_{lam}"] = np.array(L)
        out[f"dl_{lam}"] = dl
    np.savez_compressed(OUT / "loss.npz", rendered=ren, target=tgt, **out)
    print("loss: 3 lambdas")

    # 5. Adam (optimize.hpp:195-221): 3 steps from zero state, bbox clamp, quat renorm
    rec5 = init_random(ref, 200, (0, 0, 0), (8.0, 8.0, 8.0), 1.0, 5)
    rec5[:5, 0:3] = [[-0.5, 3, 3], [8.5, 3, 3], [3, -1, 3], [3, 3, 9], [1e-4, 1e-4, 1e-4]]
    rec5 = rec5.astype(np.float32).astype(np.float64)
    bbox5 = ((0, 0, 0), (8.0, 8.0, 8.0))
    m = np.zeros_like(rec5)
    v = np.zeros_like(rec5)
    step = 0
    lrs = (6e-4, 0.02, 2e-3, 1e-3)
    gseq = [np.random.default_rng(100 + s).normal(0.0, 1.0, rec5.shape).astype(np.float32).astype(np.float64)
            for s in range(3)]
    cur = rec5.copy()
    outs = {}
    for s, g in enumerate(gseq):
        cur, m, v, step = ref.adam_step(cur, bbox5, g, m, v, step, lrs)
        outs[f"rec_{s}"] = cur.copy()
        outs[f"m_{s}"] = m.copy()
        outs[f"v_{s}"] = v.copy()
    lr_tab = np.array([[ref.lib.gref_lr_at(lr0, it, tot) for lr0, it, tot in
                        ((6e-4, 1, 30000), (6e-4, 15000, 30000), (0.02, 30000, 30000), (1e-3, 7, 10))]])
    np.savez_compressed(OUT / "adam.npz", records=rec5, bbox=np.array(bbox5), lrs=np.array(lrs),
                        grads=np.stack(gseq), lr_at=lr_tab, **outs)
    print("adam: 3 steps")

    # 6. voxelizer (voxelize.hpp:113-240)
    vc = NS(dims=(24, 20, 16), spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), tile_dims=(8, 8, 8),
            support_sigmas=3.0, scale_modifier=1.0)
    rec6 = init_random(ref, 300, (2, 2, 2), (22.0, 18.0, 14.0), 1.0, 13).astype(np.float32).astype(np.float64)
    vol = ref.voxelize(rec6, vc)
    voff, vent = ref.voxel_tiles(rec6, vc)
    dlv = np.random.default_rng(17).uniform(-1.0, 1.0, vol.shape).astype(np.float32).astype(np.float64)
    vg = ref.voxelize_backward(rec6, vc, dlv)
    np.savez_compressed(OUT / "voxel.npz", meta=json.dumps({k: list(getattr(vc, k)) if isinstance(
        getattr(vc, k), tuple) else getattr(vc, k) for k in vars(vc)}), records=rec6, volume=vol, offsets=voff,
        entries=vent, dl_dv=dlv, grads=vg)
    print(f"voxel: pairs={len(vent)}")


if __name__ == "__main__":
    main()
