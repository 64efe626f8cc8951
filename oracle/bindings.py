"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

``load("ref")``    -> oracle/_ref/libgpile_ref.so   (the reference itself)
``load("oracle")`` -> oracle/_build/libgpile_oracle.so (the C restatement)

Both expose the same methods on plain numpy arrays (records are (n, 11)
float64 in checkpoint order; images (H, W); volumes (Z, Y, X)).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libgpile_ref.so"
ORACLE_SO = HERE / "_build" / "libgpile_oracle.so"


def build(ref: bool = True) -> None:
    """Build the checkers (the reference one only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref and Path(os.environ.get("REF_ROOT", "/root/reference"), "proj", "include").exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class Bounds(C.Structure):
    _fields_ = [("min", C.c_double * 3), ("max", C.c_double * 3)]


class PoseC(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3), ("width", C.c_int32),
                ("height", C.c_int32), ("pixel_spacing", C.c_double * 2),
                ("principal_point", C.c_double * 2)]


class PsfC(C.Structure):
    _fields_ = [("sigma_x", C.c_double), ("sigma_y", C.c_double), ("sigma_z", C.c_double)]


class CfgC(C.Structure):
    _fields_ = [("tau", C.c_double), ("tile_size", C.c_int32), ("footprint_sigmas", C.c_double),
                ("scale_modifier", C.c_double)]


class LrC(C.Structure):
    _fields_ = [("position", C.c_double), ("opacity", C.c_double), ("scale", C.c_double),
                ("rotation", C.c_double)]


class HpC(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class VcfgC(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("spacing", C.c_double * 3), ("origin", C.c_double * 3),
                ("tile_dims", C.c_int32 * 3), ("support_sigmas", C.c_double),
                ("scale_modifier", C.c_double)]


class DcfgC(C.Structure):
    _fields_ = [("tau", C.c_double), ("grad_threshold", C.c_double),
                ("split_scale_fraction", C.c_double), ("split_scale_divisor", C.c_double),
                ("scale_modifier", C.c_double)]


class FitCfgC(C.Structure):
    """gpk_fit_config (include/gpile_b200.h) = FitConfig (optimize.hpp:21-44)."""
    _fields_ = [
        ("iterations", C.c_int32), ("lr_position", C.c_double), ("lr_opacity", C.c_double),
        ("lr_scale", C.c_double), ("lr_rotation", C.c_double), ("init_count", C.c_uint64),
        ("tau", C.c_double), ("densify_start", C.c_int32), ("densify_end", C.c_int32),
        ("grad_threshold", C.c_double), ("lambda_", C.c_double), ("densify_interval", C.c_int32),
        ("rng_seed", C.c_uint64), ("init_mode", C.c_int32), ("scale_modifier", C.c_double),
        ("split_scale_fraction", C.c_double), ("split_scale_divisor", C.c_double),
        ("dssim_scale", C.c_double), ("progress_interval", C.c_int32), ("tile_size", C.c_int32),
        ("footprint_sigmas", C.c_double),
    ]


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def pose_c(pose) -> PoseC:
    r = np.asarray(pose.rotation, np.float64).reshape(9)
    return PoseC((C.c_double * 9)(*r), (C.c_double * 3)(*pose.translation), int(pose.width),
                 int(pose.height), (C.c_double * 2)(*pose.pixel_spacing),
                 (C.c_double * 2)(*pose.principal_point))


def psf_c(psf) -> PsfC:
    return PsfC(psf.sigma_x, psf.sigma_y, psf.sigma_z)


def cfg_c(cfg) -> CfgC:
    return CfgC(cfg.tau, int(cfg.tile_size), cfg.footprint_sigmas, cfg.scale_modifier)


def vcfg_c(v) -> VcfgC:
    return VcfgC((C.c_int32 * 3)(*v.dims), (C.c_double * 3)(*v.spacing), (C.c_double * 3)(*v.origin),
                 (C.c_int32 * 3)(*v.tile_dims), v.support_sigmas, v.scale_modifier)


class CpuChecker:
    """Uniform interface over libgpile_ref.so (prefix gref_) / libgpile_oracle.so (gor_)."""

    def __init__(self, kind: str):
        self.kind = kind
        path = REF_SO if kind == "ref" else ORACLE_SO
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (oracle/Makefile)")
        self.lib = C.CDLL(str(path))
        self.is_ref = kind == "ref"
        L = self.lib
        if self.is_ref:
            L.gref_last_error.restype = C.c_char_p
            L.gref_set_new.restype = C.c_void_p
            L.gref_set_new.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.POINTER(Bounds)]
            L.gref_set_free.argtypes = [C.c_void_p]
            L.gref_set_get.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
            L.gref_lr_at.restype = C.c_double
            L.gref_lr_at.argtypes = [C.c_double, C.c_int, C.c_int]
            L.gref_render_oracle.restype = C.c_double
            L.gref_render_oracle.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(PoseC), C.POINTER(PsfC),
                                             C.c_double, C.c_double, C.c_double]
            L.gref_rng_new.restype = C.c_void_p
            L.gref_rng_new.argtypes = [C.c_uint64]
            L.gref_rng_free.argtypes = [C.c_void_p]
            L.gref_rng_uniform.restype = C.c_double
            L.gref_rng_uniform.argtypes = [C.c_void_p]
            L.gref_rng_uniform_range.restype = C.c_double
            L.gref_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
            L.gref_rng_normal.restype = C.c_double
            L.gref_rng_normal.argtypes = [C.c_void_p]
            L.gref_rng_below.restype = C.c_uint64
            L.gref_rng_below.argtypes = [C.c_void_p, C.c_uint64]
            L.gref_random_primitive.argtypes = [C.c_void_p, C.POINTER(Bounds), C.c_double, C.c_double,
                                                C.POINTER(C.c_double)]
            L.gref_random_pose.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(PoseC)]
            L.gref_alpha_activation_inverse.restype = C.c_double
            L.gref_alpha_activation_inverse.argtypes = [C.c_double]
        else:
            L.gor_last_error.restype = C.c_char_p

    # -- plumbing ------------------------------------------------------------
    def _call(self, name, *args):
        fn = getattr(self.lib, ("gref_" if self.is_ref else "gor_") + name)
        st = fn(*args)
        if st != 0:
            msg = (self.lib.gref_last_error() if self.is_ref else self.lib.gor_last_error()) or b""
            raise CheckerError(st, msg.decode(errors="replace"))

    def _set(self, rec, bbox=((0, 0, 0), (1, 1, 1))):
        rec = np.ascontiguousarray(rec, np.float64).reshape(-1, 11)
        if self.is_ref:
            b = Bounds((C.c_double * 3)(*bbox[0]), (C.c_double * 3)(*bbox[1]))
            h = self.lib.gref_set_new(rec.shape[0], _d(rec), C.byref(b))
            return _SetHandle(self.lib, h, rec)
        return _SetHandle(None, None, rec)

    def _head(self, h):
        """Leading arguments selecting the Gaussian set."""
        if self.is_ref:
            return (C.c_void_p(h.h),)
        return (C.c_uint64(h.rec.shape[0]), _d(h.rec))

    # -- hot path ------------------------------------------------------------
    def prepare(self, rec, pose, psf, cfg, bbox=((0, 0, 0), (1, 1, 1))):
        h = self._set(rec, bbox)
        n = h.rec.shape[0]
        cnt = C.c_uint64()
        idx = np.zeros(max(n, 1), np.uint32)
        bnd = np.zeros((max(n, 1), 4), np.int32)
        fld = np.zeros((max(n, 1), 19), np.float64)
        p, f, c = pose_c(pose), psf_c(psf), cfg_c(cfg)
        self._call("prepare", *self._head(h), C.byref(p), C.byref(f), C.byref(c), C.byref(cnt),
                   idx.ctypes.data_as(C.POINTER(C.c_uint32)), bnd.ctypes.data_as(C.POINTER(C.c_int32)),
                   _d(fld))
        k = cnt.value
        return idx[:k].copy(), bnd[:k].copy(), fld[:k].copy()

    def prepare_full(self, rec, pose, psf, cfg, bbox=((0, 0, 0), (1, 1, 1))):
        """Every PreparedGaussian field (47 doubles per survivor, ref only)."""
        assert self.is_ref, "prepare_full: the reference build only"
        h = self._set(rec, bbox)
        n = h.rec.shape[0]
        cnt = C.c_uint64()
        fld = np.zeros((max(n, 1), 47), np.float64)
        p, f, c = pose_c(pose), psf_c(psf), cfg_c(cfg)
        self._call("prepare_full", C.c_void_p(h.h), C.byref(p), C.byref(f), C.byref(c), C.byref(cnt), _d(fld),
                   C.c_uint64(fld.shape[0]))
        return fld[:cnt.value].copy()

    def tile_lists(self, rec, pose, psf, cfg, bbox=((0, 0, 0), (1, 1, 1))):
        h = self._set(rec, bbox)
        p, f, c = pose_c(pose), psf_c(psf), cfg_c(cfg)
        tot, tiles = C.c_uint64(), C.c_uint64()
        self._call("tile_lists", *self._head(h), C.byref(p), C.byref(f), C.byref(c), None, None,
                   C.c_uint64(0), C.byref(tot), C.byref(tiles))
        off = np.zeros(tiles.value + 1, np.uint32)
        ent = np.zeros(max(tot.value, 1), np.uint32)
        self._call("tile_lists", *self._head(h), C.byref(p), C.byref(f), C.byref(c),
                   off.ctypes.data_as(C.POINTER(C.c_uint32)), ent.ctypes.data_as(C.POINTER(C.c_uint32)),
                   C.c_uint64(ent.size), C.byref(tot), C.byref(tiles))
        return off, ent[:tot.value]

    def rasterize(self, rec, pose, psf, cfg, bbox=((0, 0, 0), (1, 1, 1)), naive=False):
        h = self._set(rec, bbox)
        img = np.zeros((pose.height, pose.width), np.float64)
        p, f, c = pose_c(pose), psf_c(psf), cfg_c(cfg)
        self._call("rasterize_naive" if naive else "rasterize", *self._head(h), C.byref(p), C.byref(f),
                   C.byref(c), _d(img))
        return img

    def backward(self, rec, pose, psf, cfg, dl_di, bbox=((0, 0, 0), (1, 1, 1))):
        h = self._set(rec, bbox)
        n = h.rec.shape[0]
        g = np.zeros((max(n, 1), 11), np.float64)
        nrm = np.zeros(max(n, 1), np.float64)
        obs = np.zeros(max(n, 1), np.uint8)
        wld = np.zeros((max(n, 1), 3), np.float64)
        dl = np.ascontiguousarray(dl_di, np.float64)
        p, f, c = pose_c(pose), psf_c(psf), cfg_c(cfg)
        self._call("backward", *self._head(h), C.byref(p), C.byref(f), C.byref(c), _d(dl), _d(g),
                   _d(nrm), obs.ctypes.data_as(C.POINTER(C.c_uint8)), _d(wld))
        return g[:n], (nrm[:n], obs[:n], wld[:n])

    def loss(self, rendered, target, lam, dssim_scale=0.5):
        r = np.ascontiguousarray(rendered, np.float64)
        t = np.ascontiguousarray(target, np.float64)
        h, w = r.shape
        dl = np.zeros_like(r)
        L = C.c_double()
        self._call("loss", C.c_int(w), C.c_int(h), _d(r), _d(t), C.c_double(lam), C.c_double(dssim_scale),
                   _d(dl), C.byref(L))
        return L.value, dl

    def adam_step(self, rec, bbox, grads, m, v, step, lrs, hp=(0.9, 0.999, 1e-8)):
        rec = np.ascontiguousarray(rec, np.float64).copy()
        m = np.ascontiguousarray(m, np.float64).copy()
        v = np.ascontiguousarray(v, np.float64).copy()
        g = np.ascontiguousarray(grads, np.float64)
        st = C.c_int64(step)
        lr = LrC(*lrs)
        hpc = HpC(*hp)
        if self.is_ref:
            h = self._set(rec, bbox)
            self._call("adam_step", C.c_void_p(h.h), _d(g), _d(m), _d(v), C.byref(st), C.byref(lr),
                       C.byref(hpc))
            self.lib.gref_set_get(h.h, _d(rec))
        else:
            b = Bounds((C.c_double * 3)(*bbox[0]), (C.c_double * 3)(*bbox[1]))
            self._call("adam_step", C.c_uint64(rec.shape[0]), _d(rec), C.byref(b), _d(g), _d(m), _d(v),
                       C.byref(st), C.byref(lr), C.byref(hpc))
        return rec, m, v, st.value

    def densify_and_prune(self, rec, bbox, m, v, step, grad_norm_sum, observations, world_grad_sum,
                          dcfg, rng):
        """densify_and_prune (optimize.hpp:255-344) through the reference (ref only);
        dcfg = (tau, grad_threshold, split_scale_fraction, split_scale_divisor, mod);
        rng a RefRng. Returns (records, m, v, (pruned, cloned, split))."""
        assert self.is_ref, "densify_and_prune: the reference build only"
        rec = np.ascontiguousarray(rec, np.float64).reshape(-1, 11)
        n = rec.shape[0]
        h = self._set(rec, bbox)
        m = np.ascontiguousarray(m, np.float64).reshape(n, 11).copy()
        v = np.ascontiguousarray(v, np.float64).reshape(n, 11).copy()
        g = np.ascontiguousarray(grad_norm_sum, np.float64).reshape(n)
        o = np.ascontiguousarray(observations, np.int32).reshape(n)
        w = np.ascontiguousarray(world_grad_sum, np.float64).reshape(n, 3)
        cap = max(2 * n, 1)
        out = np.zeros((cap, 11))
        om = np.zeros((cap, 11))
        ov = np.zeros((cap, 11))
        on = C.c_uint64()
        rep = (C.c_uint64 * 3)()
        dc = DcfgC(*dcfg)
        self._call("densify_and_prune", C.c_void_p(h.h), _d(m), _d(v), C.c_int64(step), _d(g),
                   o.ctypes.data_as(C.POINTER(C.c_int32)), _d(w), C.byref(dc), C.c_void_p(rng.h), _d(out),
                   _d(om), _d(ov), C.byref(on), rep)
        k = on.value
        return out[:k].copy(), om[:k].copy(), ov[:k].copy(), tuple(int(x) for x in rep)

    def fit(self, volume, spacing, origin, psf, fit_fields: dict, capacity: int = 1 << 20,
            max_progress: int = 4096):
        """fit (optimize.hpp:360-424) through the reference (ref only); volume (Z, Y, X).
        Returns (records, progress rows [iteration, loss, count, psnr2d, monitor_loss])."""
        assert self.is_ref, "fit: the reference build only"
        vol = np.ascontiguousarray(volume, np.float64)
        dims = (C.c_int32 * 3)(vol.shape[2], vol.shape[1], vol.shape[0])
        sp = (C.c_double * 3)(*spacing)
        org = (C.c_double * 3)(*origin)
        fc = FitCfgC(**fit_fields)
        out = np.zeros((capacity, 11))
        prog = np.zeros((max_progress, 5))
        on, npg = C.c_uint64(), C.c_uint64()
        pc = psf_c(psf)
        self._call("fit", _d(vol), dims, sp, org, C.byref(pc), C.byref(fc), _d(out), C.c_uint64(capacity),
                   C.byref(on), _d(prog), C.c_uint64(max_progress), C.byref(npg))
        return out[:on.value].copy(), prog[:min(npg.value, max_progress)].copy()

    def voxelize(self, rec, vcfg):
        h = self._set(rec)
        X, Y, Z = vcfg.dims
        out = np.zeros((Z, Y, X), np.float64)
        vc = vcfg_c(vcfg)
        self._call("voxelize", *self._head(h), C.byref(vc), _d(out))
        return out

    def voxel_tiles(self, rec, vcfg):
        h = self._set(rec)
        vc = vcfg_c(vcfg)
        tot, tiles = C.c_uint64(), C.c_uint64()
        self._call("voxel_tiles", *self._head(h), C.byref(vc), None, None, C.c_uint64(0), C.byref(tot),
                   C.byref(tiles))
        off = np.zeros(tiles.value + 1, np.uint32)
        ent = np.zeros(max(tot.value, 1), np.uint32)
        self._call("voxel_tiles", *self._head(h), C.byref(vc), off.ctypes.data_as(C.POINTER(C.c_uint32)),
                   ent.ctypes.data_as(C.POINTER(C.c_uint32)), C.c_uint64(ent.size), C.byref(tot),
                   C.byref(tiles))
        return off, ent[:tot.value]

    def voxelize_backward(self, rec, vcfg, dl_dv):
        h = self._set(rec)
        n = h.rec.shape[0]
        g = np.zeros((max(n, 1), 11), np.float64)
        d = np.ascontiguousarray(dl_dv, np.float64)
        vc = vcfg_c(vcfg)
        self._call("voxelize_backward", *self._head(h), C.byref(vc), _d(d), _d(g))
        return g[:n]

    # -- reference-only helpers --------------------------------------------------
    def render_oracle(self, rec, i, pose, psf, px, py, mod=1.0):
        h = self._set(rec)
        p, f = pose_c(pose), psf_c(psf)
        return self.lib.gref_render_oracle(h.h, i, C.byref(p), C.byref(f), px, py, mod)


class _SetHandle:
    def __init__(self, lib, h, rec):
        self.lib, self.h, self.rec = lib, h, rec

    def __del__(self):
        if self.lib is not None and self.h:
            self.lib.gref_set_free(self.h)


class RefRng:
    """The reference Rng (rng.hpp:14-70) — fixture streams identical to its tests."""

    def __init__(self, seed: int):
        self.ck = load("ref")
        self.L = self.ck.lib
        self.h = self.L.gref_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.gref_rng_free(self.h)

    def uniform(self, lo=None, hi=None):
        if lo is None:
            return self.L.gref_rng_uniform(self.h)
        return self.L.gref_rng_uniform_range(self.h, lo, hi)

    def normal(self):
        return self.L.gref_rng_normal(self.h)

    def below(self, n):
        return self.L.gref_rng_below(self.h, n)

    def random_primitive(self, bbox, lo=0.5, hi=2.0):
        out = np.zeros(11, np.float64)
        b = Bounds((C.c_double * 3)(*bbox[0]), (C.c_double * 3)(*bbox[1]))
        self.L.gref_random_primitive(self.h, C.byref(b), lo, hi, _d(out))
        return out

    def random_pose_c(self, w=24, h=24) -> PoseC:
        p = PoseC()
        self.L.gref_random_pose(self.h, w, h, C.byref(p))
        return p


_cache: dict[str, CpuChecker] = {}


def load(kind: str) -> CpuChecker:
    if kind not in _cache:
        _cache[kind] = CpuChecker(kind)
    return _cache[kind]


def available(kind: str) -> bool:
    return (REF_SO if kind == "ref" else ORACLE_SO).exists()
