"""Reference-shaped host API over the sm_100a C-ABI.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/gpile): ``rasterize_slice`` (render.hpp:194),
``prepare_gaussians`` (render.hpp:83), ``backward_slice`` (backward.hpp:189),
``photometric_loss`` (loss.hpp:13), ``adam_step`` / ``AdamState`` / ``lr_at``
(optimize.hpp:71-221), ``voxelize`` / ``voxelize_backward``
(voxelize.hpp:113-240), ``init_random`` (optimize.hpp:94) and
``slice_pose_for_index`` (core.hpp:202). Exceptions map the reference's
taxonomy: ``InvalidArgument`` (std::invalid_argument, also a ValueError),
``DegenerateCovariance`` and ``NumericFailure``.

Data conventions: a GaussianSet holds an (n, 11) float64 array of stored
parameters in the checkpoint record order (mu xyz, log-scale xyz, quat wxyz,
raw alpha) plus the bbox; the device keeps them as float32. Images are
(height, width) arrays, row-major like SliceImage::pixels[j*W + i]; volumes
are (Z, Y, X). Gradients come back as (n, 11) arrays in the same slot order.

``Session`` is the device-resident form used by the training loop: parameters
and Adam moments stay in HBM and only slice-sized data crosses PCIe.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import (CorruptContainer, DegenerateCovariance, GpileError, InvalidArgument,
                      LoadError, NumericFailure, StateError, check)

__all__ = [
    "GaussianSet", "SlicePose", "PsfSpec", "RasterConfig", "LearningRates", "AdamState",
    "VoxelizerConfig", "ScreenGradStats", "Session", "Prepared",
    "rasterize_slice", "prepare_gaussians", "tile_lists", "backward_slice", "photometric_loss",
    "adam_step", "lr_at", "voxelize", "voxelize_backward", "init_random",
    "slice_pose_for_index", "default_session", "init_grid", "default_init_count", "Rng",
    "DensifyConfig", "DensifyReport", "DensifyAccum", "FitConfig", "FitProgress", "fit",
    "save_checkpoint", "load_checkpoint", "checkpoint_bytes", "CorruptContainer", "LoadError",
    "QuantSpec", "QuantizedStreams",
    "DegenerateCovariance", "NumericFailure", "InvalidArgument", "GpileError", "StateError",
]

RECORD = 11


# ---- value types -------------------------------------------------------------
@dataclass
class GaussianSet:
    """GaussianSet (core.hpp:67-74): ordered primitives + world bbox."""

    records: np.ndarray
    bbox_min: tuple = (0.0, 0.0, 0.0)
    bbox_max: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self):
        self.records = np.ascontiguousarray(np.asarray(self.records, dtype=np.float64).reshape(-1, RECORD))

    def size(self) -> int:
        return int(self.records.shape[0])

    def __len__(self) -> int:
        return self.size()

    def bounds(self) -> N.Bounds:
        return N.Bounds((C.c_double * 3)(*self.bbox_min), (C.c_double * 3)(*self.bbox_max))

    def copy(self) -> "GaussianSet":
        return GaussianSet(self.records.copy(), tuple(self.bbox_min), tuple(self.bbox_max))


@dataclass
class SlicePose:
    """SlicePose (core.hpp:78-105). rotation is R_c (3x3)."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: tuple = (0.0, 0.0, 0.0)
    width: int = 0
    height: int = 0
    pixel_spacing: tuple = (1.0, 1.0)
    principal_point: tuple = (0.0, 0.0)

    def to_c(self) -> N.SlicePoseC:
        r = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        return N.SlicePoseC((C.c_double * 9)(*r), (C.c_double * 3)(*self.translation),
                            int(self.width), int(self.height),
                            (C.c_double * 2)(*self.pixel_spacing),
                            (C.c_double * 2)(*self.principal_point))

    @staticmethod
    def from_c(p: N.SlicePoseC) -> "SlicePose":
        return SlicePose(np.array(list(p.rotation)).reshape(3, 3), tuple(p.translation),
                         p.width, p.height, tuple(p.pixel_spacing), tuple(p.principal_point))

    def pixel_center(self, i: int, j: int) -> tuple:
        return ((i - self.principal_point[0]) * self.pixel_spacing[0],
                (j - self.principal_point[1]) * self.pixel_spacing[1])


@dataclass
class PsfSpec:
    """PsfSpec (core.hpp:109-117)."""

    sigma_x: float = 1.0
    sigma_y: float = 1.0
    sigma_z: float = 1.0

    def to_c(self) -> N.PsfC:
        return N.PsfC(self.sigma_x, self.sigma_y, self.sigma_z)


@dataclass
class RasterConfig:
    """RasterConfig (render.hpp:26-31)."""

    tau: float = 0.02
    tile_size: int = 16
    footprint_sigmas: float = 3.0
    scale_modifier: float = 1.0

    def to_c(self) -> N.RasterConfigC:
        return N.RasterConfigC(self.tau, int(self.tile_size), self.footprint_sigmas, self.scale_modifier)


@dataclass
class LearningRates:
    """LearningRates (optimize.hpp:178-180)."""

    position: float
    opacity: float
    scale: float
    rotation: float

    def to_c(self) -> N.LearningRatesC:
        return N.LearningRatesC(self.position, self.opacity, self.scale, self.rotation)


@dataclass
class AdamState:
    """AdamState (optimize.hpp:156-176); moments as (n, 11) arrays."""

    n: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m: np.ndarray | None = None
    v: np.ndarray | None = None

    def __post_init__(self):
        if self.m is None:
            self.m = np.zeros((self.n, RECORD))
        if self.v is None:
            self.v = np.zeros((self.n, RECORD))

    def size(self) -> int:
        return int(self.m.shape[0])


@dataclass
class VoxelizerConfig:
    """VoxelizerConfig (voxelize.hpp:16-38)."""

    dims: tuple = (0, 0, 0)
    spacing: tuple = (1.0, 1.0, 1.0)
    origin: tuple = (0.0, 0.0, 0.0)
    tile_dims: tuple = (8, 8, 8)
    support_sigmas: float = 3.0
    scale_modifier: float = 1.0

    def to_c(self) -> N.VoxelizerConfigC:
        return N.VoxelizerConfigC((C.c_int32 * 3)(*self.dims), (C.c_double * 3)(*self.spacing),
                                  (C.c_double * 3)(*self.origin), (C.c_int32 * 3)(*self.tile_dims),
                                  self.support_sigmas, self.scale_modifier)


@dataclass
class ScreenGradStats:
    """ScreenGradStats (backward.hpp:19-26)."""

    mu2d_grad_norm: np.ndarray
    observed: np.ndarray
    world_pos_grad: np.ndarray


@dataclass
class Prepared:
    """Survivors of prepare_gaussians (render.hpp:83) in ascending set order."""

    index: np.ndarray      # uint32 set indices
    bounds: np.ndarray     # int32 (S, 4): lo_x, hi_x, lo_y, hi_y (inclusive)
    fields: np.ndarray     # float64 (S, 6): alpha_tilde, mu2d.x, mu2d.y, conic a, b, d
    pairs: int = 0         # (tile, Gaussian) pairs of the binning


class Rng:
    """The reference's seeded generator (Rng, rng.hpp:14-70), native: same stream."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        check(N.lib.gpk_rng_create(int(seed) & (2**64 - 1), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            N.lib.gpk_rng_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def uniform(self) -> float:
        v = C.c_double()
        check(N.lib.gpk_rng_uniform(self._h, C.byref(v)))
        return v.value

    def below(self, n: int) -> int:
        v = C.c_uint64()
        check(N.lib.gpk_rng_below(self._h, int(n), C.byref(v)))
        return int(v.value)

    def normal(self) -> float:
        v = C.c_double()
        check(N.lib.gpk_rng_normal(self._h, C.byref(v)))
        return v.value


@dataclass
class DensifyConfig:
    """The FitConfig fields densify_and_prune reads (optimize.hpp:21-44)."""

    tau: float = 0.02
    grad_threshold: float = 5e-5
    split_scale_fraction: float = 0.01
    split_scale_divisor: float = 1.6
    scale_modifier: float = 1.0

    def to_c(self) -> N.DensifyConfigC:
        return N.DensifyConfigC(self.tau, self.grad_threshold, self.split_scale_fraction,
                                self.split_scale_divisor, self.scale_modifier)


@dataclass
class DensifyReport:
    """DensifyReport (optimize.hpp:251-253)."""

    pruned: int = 0
    cloned: int = 0
    split: int = 0


@dataclass
class DensifyAccum:
    """DensifyAccum (optimize.hpp:228-249) as host arrays."""

    grad_norm_sum: np.ndarray
    observations: np.ndarray
    world_grad_sum: np.ndarray   # (n, 3)


@dataclass
class FitConfig:
    """FitConfig (optimize.hpp:21-62); init_mode "random" | "grid"."""

    iterations: int = 30000
    lr_position: float = 0.0006
    lr_opacity: float = 0.02
    lr_scale: float = 0.002
    lr_rotation: float = 0.001
    init_count: int = 0
    tau: float = 0.02
    densify_start: int = 500
    densify_end: int = 25000
    grad_threshold: float = 5e-5
    lam: float = 0.2
    densify_interval: int = 100
    rng_seed: int = 0
    init_mode: str = "random"
    scale_modifier: float = 1.0
    split_scale_fraction: float = 0.01
    split_scale_divisor: float = 1.6
    dssim_scale: float = 0.5
    progress_interval: int = 200
    tile_size: int = 16
    footprint_sigmas: float = 3.0

    def to_c(self) -> N.FitConfigC:
        if self.init_mode not in ("random", "grid"):
            raise InvalidArgument("FitConfig: init_mode must be random or grid")
        return N.FitConfigC(int(self.iterations), self.lr_position, self.lr_opacity, self.lr_scale,
                            self.lr_rotation, int(self.init_count), self.tau, int(self.densify_start),
                            int(self.densify_end), self.grad_threshold, self.lam,
                            int(self.densify_interval), int(self.rng_seed) & (2**64 - 1),
                            0 if self.init_mode == "random" else 1, self.scale_modifier,
                            self.split_scale_fraction, self.split_scale_divisor, self.dssim_scale,
                            int(self.progress_interval), int(self.tile_size), self.footprint_sigmas)


@dataclass
class QuantSpec:
    """QuantSpec (quant.hpp:13-26)."""

    pos_bits: int = 14
    opacity_bits: int = 12
    scale_bits: int = 12
    quat_bits: int = 12
    morton_bits: int = 14

    def to_c(self) -> N.QuantSpecC:
        return N.QuantSpecC(self.pos_bits, self.opacity_bits, self.scale_bits, self.quat_bits, self.morton_bits)


@dataclass
class QuantizedStreams:
    """QuantizedSet's integer streams (quant.hpp:29-39) or encode()'s packed byte streams."""

    positions: np.ndarray
    opacities: np.ndarray
    log_scales: np.ndarray
    quats: np.ndarray
    scale_min: tuple
    scale_max: tuple


@dataclass
class FitProgress:
    """FitProgress (optimize.hpp:350-356)."""

    iteration: int
    loss: float
    count: int
    psnr2d: float
    monitor_loss: float


# ---- session -----------------------------------------------------------------
class Session:
    """One device-resident GaussianPile session on one GPU (one CUDA stream)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        check(N.lib.gpk_session_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h)))
        self._h = h
        self.device = device
        self.n = 0
        self.bbox = ((0.0,) * 3, (1.0,) * 3)
        self.shape = (0, 0)

    # lifecycle
    def close(self):
        if getattr(self, "_h", None):
            N.lib.gpk_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        check(N.lib.gpk_session_synchronize(self._h))

    def reserve_pairs(self, pairs: int):
        check(N.lib.gpk_session_reserve_pairs(self._h, int(pairs)))

    def stream(self) -> int:
        p = C.c_void_p()
        check(N.lib.gpk_session_get_stream(self._h, C.byref(p)))
        return int(p.value or 0)

    def set_stream(self, stream: int):
        check(N.lib.gpk_session_set_stream(self._h, C.c_void_p(stream)))

    def device_buffer(self, which: int) -> tuple[int, int]:
        p, b = C.c_void_p(), C.c_uint64()
        check(N.lib.gpk_device_buffer(self._h, int(which), C.byref(p), C.byref(b)))
        return int(p.value or 0), int(b.value)

    def upload(self, which: int, host_ptr: int, nbytes: int):
        check(N.lib.gpk_upload(self._h, int(which), C.c_void_p(host_ptr), int(nbytes)))

    def download(self, which: int, host_ptr: int, nbytes: int):
        check(N.lib.gpk_download(self._h, int(which), C.c_void_p(host_ptr), int(nbytes)))

    STAGES = ("prepare", "sort", "raster", "backward", "chain", "loss", "adam", "voxel", "bin", "voxel_eval",
              "adam_rest")

    def set_loss_sink(self, host_ptr: int | None):
        """The loss kernel also writes each loss (f64) to this page-locked host
        address (include/gpile_b200.h gpk_set_loss_sink); None: off."""
        check(N.lib.gpk_set_loss_sink(self._h, C.c_void_p(host_ptr or None)))

    def set_target_slot(self, slot: int):
        """Select target buffer 0 or 1 for later uploads and losses (include/
        gpile_b200.h gpk_set_target_slot): alternating slots lets the next
        slice's target upload overlap the previous step entirely."""
        check(N.lib.gpk_set_target_slot(self._h, int(slot)))

    def set_lazy_adam(self, on: bool = True):
        """Lazy single-GPU training steps (include/gpile_b200.h gpk_set_lazy_adam;
        off by default, measured slower): deferred zero-gradient Adam steps,
        bit-identical results; off: every step updates all n. Graphs captured
        before a mode change must be recaptured."""
        check(N.lib.gpk_set_lazy_adam(self._h, 1 if on else 0))

    def stage_timing(self, enable: bool = True):
        check(N.lib.gpk_stage_timing(self._h, 1 if enable else 0))

    def stage_times(self, reset: bool = False) -> dict:
        ms = np.zeros(len(self.STAGES), np.float64)
        cnt = np.zeros(len(self.STAGES), np.uint64)
        check(N.lib.gpk_stage_times(self._h, N.dptr(ms), cnt.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    1 if reset else 0))
        return {name: (float(ms[k]), int(cnt[k])) for k, name in enumerate(self.STAGES)}

    # parameters
    def set_gaussians(self, gs: GaussianSet):
        rec = np.ascontiguousarray(gs.records, dtype=np.float32)
        b = gs.bounds()
        check(N.lib.gpk_set_gaussians(self._h, gs.size(), N.fptr(rec), C.byref(b)))
        self.n = gs.size()
        self.bbox = (tuple(gs.bbox_min), tuple(gs.bbox_max))

    def get_gaussians(self) -> np.ndarray:
        out = np.zeros((self.n, RECORD), dtype=np.float32)
        check(N.lib.gpk_get_gaussians(self._h, N.fptr(out)))
        return out

    def set_gradients(self, grads: np.ndarray):
        g = np.ascontiguousarray(grads, dtype=np.float32).reshape(self.n, RECORD)
        check(N.lib.gpk_set_gradients(self._h, N.fptr(g)))

    def get_gradients(self) -> np.ndarray:
        out = np.zeros((self.n, RECORD), np.float32)
        check(N.lib.gpk_get_gradients(self._h, N.fptr(out)))
        return out

    # slice pipeline
    def prepare(self, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig):
        p, f, c = pose.to_c(), psf.to_c(), cfg.to_c()
        check(N.lib.gpk_prepare(self._h, C.byref(p), C.byref(f), C.byref(c)))
        self.shape = (pose.height, pose.width)

    def prepared_count(self) -> tuple[int, int]:
        s, t = C.c_uint64(), C.c_uint64()
        check(N.lib.gpk_prepared_count(self._h, C.byref(s), C.byref(t)))
        return int(s.value), int(t.value)

    def prepare_stats(self) -> dict:
        """Counters of the last prepare: candidates, survivors, pairs, fp64-decided survivors."""
        v = [C.c_uint64() for _ in range(4)]
        check(N.lib.gpk_prepare_stats(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("candidates", "survivors", "pairs", "fp64_decided"), (int(x.value) for x in v)))

    def prepared(self) -> Prepared:
        s, t = self.prepared_count()
        idx = np.zeros(s, np.uint32)
        bnd = np.zeros((s, 4), np.int32)
        fld = np.zeros((s, 6), np.float64)
        check(N.lib.gpk_get_prepared(self._h, N.u32ptr(idx), N.i32ptr(bnd), N.dptr(fld)))
        return Prepared(idx, bnd, fld, t)

    PREPARED_FIELDS = ("alpha", "opacity_r", "alpha_tilde", "mu_c", "mu_e", "sigma_c", "sigma_c_inv",
                       "sigma_e", "mu_2d", "cov2d", "conic", "det2")

    def prepared_fields(self) -> dict:
        """Every PreparedGaussian field (render.hpp:68-79) of the survivors, set
        order, in the reference's fp64 operation order (gpk_get_prepared_fields)."""
        S, _ = self.prepared_count()
        raw = np.zeros((max(S, 1), 47), np.float64)
        check(N.lib.gpk_get_prepared_fields(self._h, N.dptr(raw)))
        raw = raw[:S]
        return {"alpha": raw[:, 0], "opacity_r": raw[:, 1], "alpha_tilde": raw[:, 2], "mu_c": raw[:, 3:6],
                "mu_e": raw[:, 6:9], "sigma_c": raw[:, 9:18].reshape(-1, 3, 3),
                "sigma_c_inv": raw[:, 18:27].reshape(-1, 3, 3), "sigma_e": raw[:, 27:36].reshape(-1, 3, 3),
                "mu_2d": raw[:, 36:38], "cov2d": raw[:, 38:42].reshape(-1, 2, 2),
                "conic": raw[:, 42:46].reshape(-1, 2, 2), "det2": raw[:, 46]}

    def tile_lists(self) -> tuple[np.ndarray, np.ndarray]:
        s, t = self.prepared_count()
        h, w = self.shape
        tiles = ((w + 15) // 16) * ((h + 15) // 16)
        off = np.zeros(tiles + 1, np.uint32)
        ent = np.zeros(max(t, 1), np.uint32)
        check(N.lib.gpk_get_tile_lists(self._h, N.u32ptr(off), N.u32ptr(ent)))
        return off, ent[:t]

    def rasterize(self, to_host: bool = True) -> np.ndarray | None:
        if not to_host:
            check(N.lib.gpk_rasterize(self._h, None))
            return None
        h, w = self.shape
        img = np.zeros((h, w), np.float32)
        check(N.lib.gpk_rasterize(self._h, N.fptr(img)))
        return img

    def backward(self, dl_di: np.ndarray | None = None, to_host: bool = True,
                 stats: bool = False):
        d = None if dl_di is None else np.ascontiguousarray(dl_di, dtype=np.float32)
        if d is not None and d.shape != self.shape:
            raise InvalidArgument("backward_slice: gradient image shape mismatch")
        out = np.zeros((self.n, RECORD), np.float32) if to_host else None
        st = None
        if stats:
            nrm = np.zeros(self.n, np.float64)
            obs = np.zeros(self.n, np.uint8)
            wld = np.zeros((self.n, 3), np.float64)
            st = N.ScreenStatsC(nrm.ctypes.data_as(C.POINTER(C.c_double)),
                                obs.ctypes.data_as(C.POINTER(C.c_uint8)),
                                wld.ctypes.data_as(C.POINTER(C.c_double)))
        check(N.lib.gpk_backward(self._h, None if d is None else N.fptr(d),
                                 None if out is None else N.fptr(out),
                                 None if st is None else C.byref(st)))
        if stats:
            return out, ScreenGradStats(nrm, obs, wld)
        return out

    def photometric_loss(self, target: np.ndarray | None, lam: float, dssim_scale: float = 0.5,
                         to_host: bool = True):
        t = None if target is None else np.ascontiguousarray(target, dtype=np.float32)
        if not to_host:
            check(N.lib.gpk_photometric_loss(self._h, None if t is None else N.fptr(t), lam,
                                             dssim_scale, None, None))
            return None
        loss = C.c_double()
        dl = np.zeros(self.shape, np.float32)
        check(N.lib.gpk_photometric_loss(self._h, None if t is None else N.fptr(t), lam,
                                         dssim_scale, C.byref(loss), N.fptr(dl)))
        return float(loss.value), dl

    def adam_step(self, lrs: LearningRates, beta1=0.9, beta2=0.999, eps=1e-8):
        l = lrs.to_c()
        hp = N.AdamHparamsC(beta1, beta2, eps)
        check(N.lib.gpk_adam_step(self._h, C.byref(l), C.byref(hp)))

    def adam_reset(self):
        """AdamState reset: zero moments, step 0."""
        check(N.lib.gpk_adam_reset(self._h))

    def adam_state(self) -> tuple[np.ndarray, np.ndarray, int]:
        m = np.zeros((self.n, RECORD), np.float32)
        v = np.zeros((self.n, RECORD), np.float32)
        st = C.c_int64()
        check(N.lib.gpk_get_adam_state(self._h, N.fptr(m), N.fptr(v), C.byref(st)))
        return m, v, int(st.value)

    def set_adam_state(self, m: np.ndarray, v: np.ndarray, step: int):
        m32 = np.ascontiguousarray(m, np.float32)
        v32 = np.ascontiguousarray(v, np.float32)
        check(N.lib.gpk_set_adam_state(self._h, N.fptr(m32), N.fptr(v32), int(step)))

    def fwd_bwd_slice(self, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig):
        p, f, c = pose.to_c(), psf.to_c(), cfg.to_c()
        check(N.lib.gpk_fwd_bwd_slice(self._h, C.byref(p), C.byref(f), C.byref(c)))
        self.shape = (pose.height, pose.width)

    def train_step(self, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig, lam: float,
                   dssim_scale: float, lr0: LearningRates, total_iterations: int,
                   next_pose: SlicePose | None = None):
        """One training step on `pose` (target from GPK_BUF_TARGET). With
        next_pose, Adam is fused with the next slice's cull (gpk_train_step_next)."""
        p, f, c, l = pose.to_c(), psf.to_c(), cfg.to_c(), lr0.to_c()
        if next_pose is None:
            check(N.lib.gpk_train_step(self._h, C.byref(p), C.byref(f), C.byref(c), lam, dssim_scale,
                                       C.byref(l), int(total_iterations)))
        else:
            nx = next_pose.to_c()
            check(N.lib.gpk_train_step_next(self._h, C.byref(p), C.byref(f), C.byref(c), lam, dssim_scale,
                                            C.byref(l), int(total_iterations), C.byref(nx)))
        self.shape = (pose.height, pose.width)

    # CUDA graphs of the fused paths
    def capture_fwd_bwd(self, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig) -> int:
        p, f, c = pose.to_c(), psf.to_c(), cfg.to_c()
        gid = C.c_int32()
        check(N.lib.gpk_graph_capture_fwd_bwd(self._h, C.byref(p), C.byref(f), C.byref(c), C.byref(gid)))
        self.shape = (pose.height, pose.width)
        return int(gid.value)

    def capture_train(self, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig, lam: float,
                      dssim_scale: float, lr0: LearningRates, total_iterations: int,
                      next_pose: SlicePose | None = None) -> int:
        p, f, c, l = pose.to_c(), psf.to_c(), cfg.to_c(), lr0.to_c()
        gid = C.c_int32()
        if next_pose is not None:
            nx = next_pose.to_c()
            check(N.lib.gpk_graph_capture_train_next(self._h, C.byref(p), C.byref(f), C.byref(c), lam,
                                                     dssim_scale, C.byref(l), int(total_iterations),
                                                     C.byref(nx), C.byref(gid)))
            self.shape = (pose.height, pose.width)
            return int(gid.value)
        check(N.lib.gpk_graph_capture_train(self._h, C.byref(p), C.byref(f), C.byref(c), lam,
                                            dssim_scale, C.byref(l), int(total_iterations),
                                            C.byref(gid)))
        self.shape = (pose.height, pose.width)
        return int(gid.value)

    # batched slices (gpk_slice_context / gpk_*_batch)
    def context(self, k: int) -> "Session":
        """Slice context k (0 = this session): per-slice buffers on their own
        stream, sharing this session's parameters (include/gpile_b200.h)."""
        if k == 0:
            return self
        h = C.c_void_p()
        check(N.lib.gpk_slice_context(self._h, int(k), C.byref(h)))
        ctx = _SliceContext.__new__(_SliceContext)
        ctx._h, ctx.device, ctx.n, ctx.bbox, ctx.shape = h, self.device, self.n, self.bbox, self.shape
        return ctx

    @staticmethod
    def _poses(poses):
        arr = (N.SlicePoseC * len(poses))(*[p.to_c() for p in poses])
        return arr

    def fwd_bwd_batch(self, poses, psf: PsfSpec, cfg: RasterConfig):
        """U1 x B: slice k's backward takes context k's GPK_BUF_DL_DI; the dense
        gradient is the sum over the slices (slice order)."""
        arr, f, c = self._poses(poses), psf.to_c(), cfg.to_c()
        check(N.lib.gpk_fwd_bwd_batch(self._h, len(poses), arr, C.byref(f), C.byref(c)))
        self.shape = (poses[0].height, poses[0].width)

    def train_step_batch(self, poses, psf: PsfSpec, cfg: RasterConfig, lam: float, dssim_scale: float,
                         lr0: LearningRates, total_iterations: int):
        """U2 x B: B slices (targets from the contexts), one Adam on the summed gradient."""
        arr, f, c, l = self._poses(poses), psf.to_c(), cfg.to_c(), lr0.to_c()
        check(N.lib.gpk_train_step_batch(self._h, len(poses), arr, C.byref(f), C.byref(c), lam, dssim_scale,
                                         C.byref(l), int(total_iterations)))
        self.shape = (poses[0].height, poses[0].width)

    def capture_fwd_bwd_batch(self, poses, psf: PsfSpec, cfg: RasterConfig) -> int:
        arr, f, c = self._poses(poses), psf.to_c(), cfg.to_c()
        gid = C.c_int32()
        check(N.lib.gpk_graph_capture_fwd_bwd_batch(self._h, len(poses), arr, C.byref(f), C.byref(c),
                                                    C.byref(gid)))
        self.shape = (poses[0].height, poses[0].width)
        return int(gid.value)

    def capture_train_batch(self, poses, psf: PsfSpec, cfg: RasterConfig, lam: float, dssim_scale: float,
                            lr0: LearningRates, total_iterations: int) -> int:
        arr, f, c, l = self._poses(poses), psf.to_c(), cfg.to_c(), lr0.to_c()
        gid = C.c_int32()
        check(N.lib.gpk_graph_capture_train_batch(self._h, len(poses), arr, C.byref(f), C.byref(c), lam,
                                                  dssim_scale, C.byref(l), int(total_iterations), C.byref(gid)))
        self.shape = (poses[0].height, poses[0].width)
        return int(gid.value)

    # data parallelism with the union-compacted exchange (gpk_train_step_dp)
    def train_step_dp(self, world: int, rank: int, poses, psf: PsfSpec, cfg: RasterConfig, lam: float,
                      dssim_scale: float, lr0: LearningRates, total_iterations: int, phases: int = 7):
        """Rank `rank` of `world` renders poses[rank]; the gradients of the union
        of the step's candidates are summed across ranks (phases: 1 render, 2
        exchange (NCCL), 4 update)."""
        arr, f, c, l = self._poses(poses), psf.to_c(), cfg.to_c(), lr0.to_c()
        check(N.lib.gpk_train_step_dp(self._h, int(world), int(rank), arr, C.byref(f), C.byref(c), lam, dssim_scale,
                                      C.byref(l), int(total_iterations), int(phases)))
        self.shape = (poses[rank].height, poses[rank].width)

    def capture_train_dp(self, world: int, rank: int, poses, psf: PsfSpec, cfg: RasterConfig, lam: float,
                         dssim_scale: float, lr0: LearningRates, total_iterations: int) -> int:
        arr, f, c, l = self._poses(poses), psf.to_c(), cfg.to_c(), lr0.to_c()
        gid = C.c_int32()
        check(N.lib.gpk_graph_capture_train_dp(self._h, int(world), int(rank), arr, C.byref(f), C.byref(c), lam,
                                               dssim_scale, C.byref(l), int(total_iterations), C.byref(gid)))
        self.shape = (poses[rank].height, poses[rank].width)
        return int(gid.value)

    def dp_union_rows(self) -> tuple[int, int]:
        """(rows of the last step's union, exchanged row capacity)."""
        r, c = C.c_uint64(), C.c_uint64()
        check(N.lib.gpk_dp_union_rows(self._h, C.byref(r), C.byref(c)))
        return int(r.value), int(c.value)

    def dp_reserve_union(self, rows: int):
        check(N.lib.gpk_dp_reserve_union(self._h, int(rows)))

    def graph_launch(self, graph_id: int):
        check(N.lib.gpk_graph_launch(self._h, int(graph_id)))

    def graph_destroy_all(self):
        check(N.lib.gpk_graph_destroy_all(self._h))

    # voxelizer
    def voxelize(self, cfg: VoxelizerConfig, to_host: bool = True) -> np.ndarray | None:
        c = cfg.to_c()
        if not to_host:
            check(N.lib.gpk_voxelize(self._h, C.byref(c), None))
            return None
        X, Y, Z = cfg.dims
        vol = np.zeros((Z, Y, X), np.float32)
        check(N.lib.gpk_voxelize(self._h, C.byref(c), N.fptr(vol)))
        return vol

    def voxel_tile_lists(self) -> tuple[np.ndarray, np.ndarray]:
        t, n = C.c_uint64(), C.c_uint64()
        check(N.lib.gpk_voxel_tile_count(self._h, C.byref(t), C.byref(n)))
        off = np.zeros(int(t.value) + 1, np.uint32)
        ent = np.zeros(max(int(n.value), 1), np.uint32)
        check(N.lib.gpk_get_voxel_tile_lists(self._h, N.u32ptr(off), N.u32ptr(ent)))
        return off, ent[:int(n.value)]

    def voxelize_backward(self, cfg: VoxelizerConfig, dl_dv: np.ndarray | None) -> np.ndarray:
        c = cfg.to_c()
        d = None if dl_dv is None else np.ascontiguousarray(dl_dv, dtype=np.float32)
        if d is not None and d.shape != (cfg.dims[2], cfg.dims[1], cfg.dims[0]):
            raise InvalidArgument("voxelize_backward: gradient volume shape mismatch")
        out = np.zeros((self.n, RECORD), np.float32)
        check(N.lib.gpk_voxelize_backward(self._h, C.byref(c), None if d is None else N.fptr(d),
                                          N.fptr(out)))
        return out

    # ---- codec front half (morton.hpp, quant.hpp, container.hpp) ----
    def morton_sort(self, bits: int = 14) -> np.ndarray:
        perm = np.zeros(self.n, np.uint64)
        check(N.lib.gpk_morton_sort(self._h, int(bits), perm.ctypes.data_as(C.POINTER(C.c_uint64))))
        return perm

    def quantize(self, spec: QuantSpec | None = None, morton_order: bool = False) -> QuantizedStreams:
        spec = spec or QuantSpec()
        n = self.n
        pos, opa = np.zeros(3 * n, np.uint32), np.zeros(n, np.uint32)
        ls, qt = np.zeros(3 * n, np.uint32), np.zeros(4 * n, np.uint32)
        lo, hi = np.zeros(3), np.zeros(3)
        c = spec.to_c()
        check(N.lib.gpk_quantize(self._h, C.byref(c), 1 if morton_order else 0, N.u32ptr(pos), N.u32ptr(opa),
                                 N.u32ptr(ls), N.u32ptr(qt), N.dptr(lo), N.dptr(hi)))
        return QuantizedStreams(pos, opa, ls, qt, tuple(lo), tuple(hi))

    def encode_streams(self, spec: QuantSpec | None = None) -> QuantizedStreams:
        spec = spec or QuantSpec()
        n = self.n
        sb = N.lib.gpk_stream_bytes
        bufs = [np.zeros(sb(n, k, b), np.uint8) for k, b in
                ((3, spec.pos_bits), (1, spec.opacity_bits), (3, spec.scale_bits), (4, spec.quat_bits))]
        lo, hi = np.zeros(3), np.zeros(3)
        c = spec.to_c()
        check(N.lib.gpk_encode_streams(self._h, C.byref(c), *[b.ctypes.data_as(C.c_void_p) for b in bufs],
                                       N.dptr(lo), N.dptr(hi)))
        return QuantizedStreams(*bufs, tuple(lo), tuple(hi))

    def decode_streams(self, enc: QuantizedStreams, n: int, bbox, spec: QuantSpec | None = None,
                       load: bool = True) -> np.ndarray:
        """unpack_deltas + dequantize of encode_streams' output -> (n, 11) f32 records
        (and, with load, the session's set)."""
        spec = spec or QuantSpec()
        out = np.zeros((n, RECORD), np.float32)
        b = N.Bounds((C.c_double * 3)(*bbox[0]), (C.c_double * 3)(*bbox[1]))
        lo = np.ascontiguousarray(enc.scale_min, np.float64)
        hi = np.ascontiguousarray(enc.scale_max, np.float64)
        bufs = [np.ascontiguousarray(x, np.uint8) for x in (enc.positions, enc.opacities, enc.log_scales, enc.quats)]
        c = spec.to_c()
        st = N.lib.gpk_decode_streams(self._h, C.byref(c), int(n), C.byref(b), N.dptr(lo), N.dptr(hi),
                                      *[x.ctypes.data_as(C.c_void_p) for x in bufs], N.fptr(out), 1 if load else 0)
        check(st)
        if load:
            self._refresh_n()
        return out

    # ---- checkpoints (checkpoint.hpp:38-92) ----
    def bounds(self) -> tuple:
        b = N.Bounds()
        check(N.lib.gpk_get_bounds(self._h, C.byref(b)))
        return tuple(b.min), tuple(b.max)

    def save_checkpoint(self, path):
        check(N.lib.gpk_save_checkpoint(self._h, str(path).encode()))

    def load_checkpoint(self, path):
        st = N.lib.gpk_load_checkpoint(self._h, str(path).encode())
        check(st)
        self._refresh_n()

    # ---- adaptive density control + fit driver (optimize.hpp:228-424) ----
    def _refresh_n(self):
        v = C.c_uint64()
        check(N.lib.gpk_gaussian_count(self._h, C.byref(v)))
        self.n = int(v.value)

    def densify_accum_enable(self, on: bool = True):
        check(N.lib.gpk_densify_accum_enable(self._h, 1 if on else 0))

    def densify_accum_reset(self):
        check(N.lib.gpk_densify_accum_reset(self._h))

    def densify_accum(self) -> DensifyAccum:
        n = self.n
        a = DensifyAccum(np.zeros(n), np.zeros(n, np.int32), np.zeros((n, 3)))
        check(N.lib.gpk_get_densify_accum(self._h, N.dptr(a.grad_norm_sum), N.i32ptr(a.observations),
                                          N.dptr(a.world_grad_sum)))
        return a

    def set_densify_accum(self, a: DensifyAccum):
        n = self.n
        g = np.ascontiguousarray(a.grad_norm_sum, np.float64).reshape(n)
        o = np.ascontiguousarray(a.observations, np.int32).reshape(n)
        w = np.ascontiguousarray(a.world_grad_sum, np.float64).reshape(n, 3)
        check(N.lib.gpk_set_densify_accum(self._h, N.dptr(g), N.i32ptr(o), N.dptr(w)))

    def densify_and_prune(self, cfg: DensifyConfig, rng: Rng) -> DensifyReport:
        c = cfg.to_c()
        r = N.DensifyReportC()
        check(N.lib.gpk_densify_and_prune(self._h, C.byref(c), rng.handle, C.byref(r)))
        self._refresh_n()
        return DensifyReport(int(r.pruned), int(r.cloned), int(r.split))

    def fit(self, volume: np.ndarray, spacing, origin, psf: PsfSpec, cfg: FitConfig,
            progress=None) -> None:
        """fit (optimize.hpp:360-424) on this session; volume is (Z, Y, X). The
        fitted set stays resident (get_gaussians)."""
        vol = np.ascontiguousarray(volume, np.float32)
        if vol.ndim != 3:
            raise InvalidArgument("fit: volume must be (Z, Y, X)")
        dims = np.array([vol.shape[2], vol.shape[1], vol.shape[0]], np.int32)
        sp = np.asarray(spacing, np.float64)
        org = np.asarray(origin, np.float64)
        c = cfg.to_c()
        p = psf.to_c()
        errors = []

        def _cb(pp, _user):
            try:
                q = pp.contents
                progress(FitProgress(int(q.iteration), q.loss, int(q.count), q.psnr2d, q.monitor_loss))
            except BaseException as e:  # noqa: BLE001  (re-raised after the native call)
                errors.append(e)

        cb = N.PROGRESS_FN(_cb) if progress is not None else N.PROGRESS_FN()
        st = N.lib.gpk_fit(self._h, N.fptr(vol), N.i32ptr(dims), N.dptr(sp), N.dptr(org), C.byref(p),
                           C.byref(c), cb, None)
        self._refresh_n()
        check(st)
        if errors:
            raise errors[0]


_default: dict[int, Session] = {}
_lock = threading.Lock()


class _SliceContext(Session):
    """A slice context handle (Session.context): owned by its session."""

    def close(self):
        self._h = None


def default_session(device: int = 0) -> Session:
    """Process-wide session per device used by the stateless reference-shaped calls."""
    with _lock:
        s = _default.get(device)
        if s is None:
            s = Session(device)
            _default[device] = s
        return s


def _session_for(gs: GaussianSet, device: int) -> Session:
    s = default_session(device)
    s.set_gaussians(gs)
    return s


# ---- reference-shaped free functions -----------------------------------------
def rasterize_slice(gs: GaussianSet, pose: SlicePose, psf: PsfSpec,
                    cfg: RasterConfig | None = None, device: int = 0) -> np.ndarray:
    """rasterize_slice (render.hpp:194-199): (H, W) float32 image."""
    cfg = cfg or RasterConfig()
    s = _session_for(gs, device)
    s.prepare(pose, psf, cfg)
    return s.rasterize()


def prepare_gaussians(gs: GaussianSet, pose: SlicePose, psf: PsfSpec,
                      cfg: RasterConfig | None = None, device: int = 0) -> Prepared:
    """prepare_gaussians (render.hpp:83-138): survivors in ascending set order."""
    cfg = cfg or RasterConfig()
    s = _session_for(gs, device)
    s.prepare(pose, psf, cfg)
    return s.prepared()


def tile_lists(gs: GaussianSet, pose: SlicePose, psf: PsfSpec, cfg: RasterConfig | None = None,
               device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """detail::TileGrid (render.hpp:142-160) as (offsets[tiles+1], set indices)."""
    cfg = cfg or RasterConfig()
    s = _session_for(gs, device)
    s.prepare(pose, psf, cfg)
    return s.tile_lists()


def backward_slice(gs: GaussianSet, pose: SlicePose, psf: PsfSpec, dl_di: np.ndarray,
                   cfg: RasterConfig | None = None, stats: bool = False, device: int = 0):
    """backward_slice (backward.hpp:189-196): (n, 11) gradients [, ScreenGradStats]."""
    cfg = cfg or RasterConfig()
    dl = np.asarray(dl_di)
    if dl.shape != (pose.height, pose.width):
        raise InvalidArgument("backward_slice: gradient image shape mismatch")
    s = _session_for(gs, device)
    s.prepare(pose, psf, cfg)
    return s.backward(dl, stats=stats)


def photometric_loss(rendered: np.ndarray, target: np.ndarray, lam: float,
                     dssim_scale: float = 0.5, device: int = 0) -> tuple[float, np.ndarray]:
    """photometric_loss (loss.hpp:13-37): (loss, dL/dI)."""
    r = np.ascontiguousarray(rendered, dtype=np.float32)
    t = np.ascontiguousarray(target, dtype=np.float32)
    if r.shape != t.shape or r.ndim != 2:
        raise InvalidArgument("photometric_loss: image shape mismatch")
    s = default_session(device)
    h, w = r.shape
    loss = C.c_double()
    dl = np.zeros((h, w), np.float32)
    check(N.lib.gpk_photometric_loss_images(s.handle, w, h, N.fptr(r), N.fptr(t), lam, dssim_scale,
                                            C.byref(loss), N.fptr(dl)))
    return float(loss.value), dl


def lr_at(lr0: float, iteration: int, total: int) -> float:
    """lr_at (optimize.hpp:71-73)."""
    return float(N.lib.gpk_lr_at(lr0, int(iteration), int(total)))


def adam_step(gs: GaussianSet, grads: np.ndarray, state: AdamState, lrs: LearningRates,
              device: int = 0) -> None:
    """adam_step (optimize.hpp:195-221): updates gs.records and state in place."""
    g = np.asarray(grads)
    if g.shape != (gs.size(), RECORD) or state.size() != gs.size():
        raise InvalidArgument("adam_step: shape mismatch")
    s = _session_for(gs, device)
    s.set_adam_state(state.m, state.v, state.step)
    s.set_gradients(g)
    s.adam_step(lrs, state.beta1, state.beta2, state.eps)
    m, v, st = s.adam_state()
    gs.records = s.get_gaussians().astype(np.float64)
    state.m, state.v, state.step = m.astype(np.float64), v.astype(np.float64), st


def voxelize(gs: GaussianSet, cfg: VoxelizerConfig, device: int = 0) -> np.ndarray:
    """voxelize (voxelize.hpp:113-148): (Z, Y, X) float32 volume."""
    s = _session_for(gs, device)
    return s.voxelize(cfg)


def voxelize_backward(gs: GaussianSet, cfg: VoxelizerConfig, dl_dv: np.ndarray,
                      device: int = 0) -> np.ndarray:
    """voxelize_backward (voxelize.hpp:152-240): (n, 11) gradients."""
    s = _session_for(gs, device)
    return s.voxelize_backward(cfg, dl_dv)


def init_random(count: int, bbox_min, bbox_max, scale_base: float, seed: int) -> GaussianSet:
    """init_random (optimize.hpp:94-108), bit-identical stream."""
    rec = np.zeros((int(count), RECORD), np.float64)
    b = N.Bounds((C.c_double * 3)(*bbox_min), (C.c_double * 3)(*bbox_max))
    st = N.lib.gpk_init_random(int(count), C.byref(b), float(scale_base), int(seed), N.dptr(rec))
    if st != N.GPK_OK:
        raise InvalidArgument("init_random: count must be >= 1 and bbox non-degenerate")
    return GaussianSet(rec, tuple(bbox_min), tuple(bbox_max))


def slice_pose_for_index(dims, spacing, origin, k: int) -> SlicePose:
    """slice_pose_for_index (core.hpp:202-211)."""
    d = np.asarray(dims, np.int32)
    sp = np.asarray(spacing, np.float64)
    o = np.asarray(origin, np.float64)
    p = N.SlicePoseC()
    check(N.lib.gpk_slice_pose_for_index(N.i32ptr(d), N.dptr(sp), N.dptr(o), int(k), C.byref(p)))
    return SlicePose.from_c(p)


def init_grid(count: int, bbox_min, bbox_max, scale_base: float, seed: int) -> GaussianSet:
    """init_grid (optimize.hpp:111-133), bit-identical stream."""
    rec = np.zeros((int(count), RECORD), np.float64)
    b = N.Bounds((C.c_double * 3)(*bbox_min), (C.c_double * 3)(*bbox_max))
    st = N.lib.gpk_init_grid(int(count), C.byref(b), float(scale_base), int(seed), N.dptr(rec))
    if st != N.GPK_OK:
        raise InvalidArgument("init_grid: count must be >= 1 and bbox non-degenerate")
    return GaussianSet(rec, tuple(bbox_min), tuple(bbox_max))


def default_init_count(voxel_count: int) -> int:
    """default_init_count (optimize.hpp:64-66)."""
    v = C.c_uint64()
    check(N.lib.gpk_default_init_count(int(voxel_count), C.byref(v)))
    return int(v.value)


def fit(volume: np.ndarray, spacing, origin, psf: PsfSpec, cfg: FitConfig, progress=None,
        device: int = 0) -> GaussianSet:
    """fit(volume, psf, cfg, progress) (optimize.hpp:360-424) -> the fitted set."""
    vol = np.asarray(volume)
    dims = (vol.shape[2], vol.shape[1], vol.shape[0])
    lo = tuple(float(o) - float(s) * 0.5 for o, s in zip(origin, spacing))
    hi = tuple(float(o) + (d - 0.5) * float(s) for o, s, d in zip(origin, spacing, dims))
    with Session(device) as s:
        s.fit(vol, spacing, origin, psf, cfg, progress)
        rec = s.get_gaussians().astype(np.float64)
    return GaussianSet(rec, lo, hi)


def save_checkpoint(gs: GaussianSet, path, device: int = 0) -> None:
    """save_checkpoint (checkpoint.hpp:38-57) through a device session."""
    _session_for(gs, device).save_checkpoint(path)


def load_checkpoint(path, device: int = 0) -> GaussianSet:
    """load_checkpoint (checkpoint.hpp:60-91) -> GaussianSet (records as f64 of the f32 file)."""
    with Session(device) as s:
        s.load_checkpoint(path)
        lo, hi = s.bounds()
        rec = s.get_gaussians().astype(np.float64)
    return GaussianSet(rec, lo, hi)


def checkpoint_bytes(count: int) -> int:
    """checkpoint_bytes (checkpoint.hpp:95-97)."""
    return int(N.lib.gpk_checkpoint_bytes(int(count)))
