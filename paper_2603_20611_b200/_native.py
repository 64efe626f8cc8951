"""ctypes binding of the C-ABI in include/gpile_b200.h.

The product path loads exactly one native library, the in-tree
``paper_2603_20611_b200/_lib/libgpile_b200.so`` built for sm_100a. There is no
CPU fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libgpile_b200.so"
GPK_ABI_VERSION = 7  # include/gpile_b200.h

GPK_OK = 0
GPK_ERR_INVALID_ARGUMENT = 1
GPK_ERR_DEGENERATE_COVARIANCE = 2
GPK_ERR_NUMERIC_FAILURE = 3
GPK_ERR_CUDA = 4
GPK_ERR_NCCL = 5
GPK_ERR_OUT_OF_MEMORY = 6
GPK_ERR_STATE = 7
GPK_ERR_CORRUPT_CONTAINER = 8
GPK_ERR_LOAD = 9

GPK_BUF_PARAMS, GPK_BUF_GRADS, GPK_BUF_IMAGE, GPK_BUF_DL_DI, GPK_BUF_TARGET = 0, 1, 2, 3, 4
GPK_BUF_VOLUME, GPK_BUF_DL_DV, GPK_BUF_LOSS, GPK_BUF_UNION_ROWS = 5, 6, 7, 8
GPK_DP_RENDER, GPK_DP_EXCHANGE, GPK_DP_UPDATE, GPK_DP_ALL = 1, 2, 4, 7


class Bounds(C.Structure):
    _fields_ = [("min", C.c_double * 3), ("max", C.c_double * 3)]


class SlicePoseC(C.Structure):
    _fields_ = [
        ("rotation", C.c_double * 9),
        ("translation", C.c_double * 3),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("pixel_spacing", C.c_double * 2),
        ("principal_point", C.c_double * 2),
    ]


class PsfC(C.Structure):
    _fields_ = [("sigma_x", C.c_double), ("sigma_y", C.c_double), ("sigma_z", C.c_double)]


class RasterConfigC(C.Structure):
    _fields_ = [
        ("tau", C.c_double),
        ("tile_size", C.c_int32),
        ("footprint_sigmas", C.c_double),
        ("scale_modifier", C.c_double),
    ]


class LearningRatesC(C.Structure):
    _fields_ = [("position", C.c_double), ("opacity", C.c_double), ("scale", C.c_double),
                ("rotation", C.c_double)]


class AdamHparamsC(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class VoxelizerConfigC(C.Structure):
    _fields_ = [
        ("dims", C.c_int32 * 3),
        ("spacing", C.c_double * 3),
        ("origin", C.c_double * 3),
        ("tile_dims", C.c_int32 * 3),
        ("support_sigmas", C.c_double),
        ("scale_modifier", C.c_double),
    ]


class ScreenStatsC(C.Structure):
    _fields_ = [
        ("mu2d_grad_norm", C.POINTER(C.c_double)),
        ("observed", C.POINTER(C.c_uint8)),
        ("world_pos_grad", C.POINTER(C.c_double)),
    ]


class DensifyConfigC(C.Structure):
    _fields_ = [("tau", C.c_double), ("grad_threshold", C.c_double),
                ("split_scale_fraction", C.c_double), ("split_scale_divisor", C.c_double),
                ("scale_modifier", C.c_double)]


class DensifyReportC(C.Structure):
    _fields_ = [("pruned", C.c_uint64), ("cloned", C.c_uint64), ("split", C.c_uint64)]


class FitConfigC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("lr_position", C.c_double), ("lr_opacity", C.c_double), ("lr_scale", C.c_double),
        ("lr_rotation", C.c_double),
        ("init_count", C.c_uint64),
        ("tau", C.c_double),
        ("densify_start", C.c_int32), ("densify_end", C.c_int32),
        ("grad_threshold", C.c_double),
        ("lambda_", C.c_double),
        ("densify_interval", C.c_int32),
        ("rng_seed", C.c_uint64),
        ("init_mode", C.c_int32),
        ("scale_modifier", C.c_double),
        ("split_scale_fraction", C.c_double),
        ("split_scale_divisor", C.c_double),
        ("dssim_scale", C.c_double),
        ("progress_interval", C.c_int32),
        ("tile_size", C.c_int32),
        ("footprint_sigmas", C.c_double),
    ]


class QuantSpecC(C.Structure):
    _fields_ = [("pos_bits", C.c_int32), ("opacity_bits", C.c_int32), ("scale_bits", C.c_int32),
                ("quat_bits", C.c_int32), ("morton_bits", C.c_int32)]


class FitProgressC(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("loss", C.c_double), ("count", C.c_uint64),
                ("psnr2d", C.c_double), ("monitor_loss", C.c_double)]


PROGRESS_FN = C.CFUNCTYPE(None, C.POINTER(FitProgressC), C.c_void_p)
NORMAL_FN = C.CFUNCTYPE(C.c_double, C.c_void_p)


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python paper_2603_20611_b200/build.py or __graft_entry__.build()). "
            "There is no CPU fallback.")
    return C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))


lib = _load()

_P = C.c_void_p
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_U32 = C.POINTER(C.c_uint32)
_I32 = C.POINTER(C.c_int32)
_U64 = C.POINTER(C.c_uint64)
_I64 = C.POINTER(C.c_int64)

_PROTOS = {
    "gpk_abi_version": (C.c_int, []),
    "gpk_last_error_message": (C.c_char_p, []),
    "gpk_last_error_index": (C.c_int64, []),
    "gpk_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gpk_session_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "gpk_session_destroy": (C.c_int, [_P]),
    "gpk_session_set_stream": (C.c_int, [_P, _P]),
    "gpk_session_get_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "gpk_session_synchronize": (C.c_int, [_P]),
    "gpk_session_reserve_pairs": (C.c_int, [_P, C.c_uint64]),
    "gpk_device_buffer": (C.c_int, [_P, C.c_int, C.POINTER(_P), _U64]),
    "gpk_upload": (C.c_int, [_P, C.c_int, _P, C.c_uint64]),
    "gpk_download": (C.c_int, [_P, C.c_int, _P, C.c_uint64]),
    "gpk_stage_timing": (C.c_int, [_P, C.c_int]),
    "gpk_set_lazy_adam": (C.c_int, [_P, C.c_int]),
    "gpk_set_loss_sink": (C.c_int, [_P, C.c_void_p]),
    "gpk_set_target_slot": (C.c_int, [_P, C.c_int32]),
    "gpk_stage_times": (C.c_int, [_P, _D, _U64, C.c_int]),
    "gpk_set_gaussians": (C.c_int, [_P, C.c_uint64, _F, C.POINTER(Bounds)]),
    "gpk_set_gaussians_f64": (C.c_int, [_P, C.c_uint64, _D, C.POINTER(Bounds)]),
    "gpk_get_gaussians": (C.c_int, [_P, _F]),
    "gpk_gaussian_count": (C.c_int, [_P, _U64]),
    "gpk_set_gradients": (C.c_int, [_P, _F]),
    "gpk_get_gradients": (C.c_int, [_P, _F]),
    "gpk_photometric_loss_images": (C.c_int, [_P, C.c_int32, C.c_int32, _F, _F, C.c_double,
                                              C.c_double, _D, _F]),
    "gpk_prepare": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC), C.POINTER(RasterConfigC)]),
    "gpk_prepared_count": (C.c_int, [_P, _U64, _U64]),
    "gpk_prepare_stats": (C.c_int, [_P, _U64, _U64, _U64, _U64]),
    "gpk_get_prepared": (C.c_int, [_P, _U32, _I32, _D]),
    "gpk_get_prepared_fields": (C.c_int, [_P, _D]),
    "gpk_get_tile_lists": (C.c_int, [_P, _U32, _U32]),
    "gpk_rasterize": (C.c_int, [_P, _F]),
    "gpk_backward": (C.c_int, [_P, _F, _F, C.POINTER(ScreenStatsC)]),
    "gpk_photometric_loss": (C.c_int, [_P, _F, C.c_double, C.c_double, _D, _F]),
    "gpk_adam_step": (C.c_int, [_P, C.POINTER(LearningRatesC), C.POINTER(AdamHparamsC)]),
    "gpk_adam_step_scheduled": (C.c_int, [_P, C.POINTER(LearningRatesC), C.c_int32,
                                          C.POINTER(AdamHparamsC)]),
    "gpk_adam_reset": (C.c_int, [_P]),
    "gpk_get_adam_state": (C.c_int, [_P, _F, _F, _I64]),
    "gpk_set_adam_state": (C.c_int, [_P, _F, _F, C.c_int64]),
    "gpk_fwd_bwd_slice": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                    C.POINTER(RasterConfigC)]),
    "gpk_train_step": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC), C.POINTER(RasterConfigC),
                                 C.c_double, C.c_double, C.POINTER(LearningRatesC), C.c_int32]),
    "gpk_train_step_next": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC), C.POINTER(RasterConfigC),
                                 C.c_double, C.c_double, C.POINTER(LearningRatesC), C.c_int32, C.POINTER(SlicePoseC)]),
    "gpk_slice_context": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "gpk_train_step_dp": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                    C.POINTER(RasterConfigC), C.c_double, C.c_double, C.POINTER(LearningRatesC),
                                    C.c_int32, C.c_int32]),
    "gpk_graph_capture_train_dp": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                             C.POINTER(RasterConfigC), C.c_double, C.c_double,
                                             C.POINTER(LearningRatesC), C.c_int32, C.POINTER(C.c_int32)]),
    "gpk_dp_union_rows": (C.c_int, [_P, _U64, _U64]),
    "gpk_dp_reserve_union": (C.c_int, [_P, C.c_uint64]),
    "gpk_fwd_bwd_batch": (C.c_int, [_P, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                    C.POINTER(RasterConfigC)]),
    "gpk_train_step_batch": (C.c_int, [_P, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                       C.POINTER(RasterConfigC), C.c_double, C.c_double,
                                       C.POINTER(LearningRatesC), C.c_int32]),
    "gpk_graph_capture_fwd_bwd_batch": (C.c_int, [_P, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                                  C.POINTER(RasterConfigC), C.POINTER(C.c_int32)]),
    "gpk_graph_capture_train_batch": (C.c_int, [_P, C.c_int32, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                                C.POINTER(RasterConfigC), C.c_double, C.c_double,
                                                C.POINTER(LearningRatesC), C.c_int32, C.POINTER(C.c_int32)]),
    "gpk_graph_capture_fwd_bwd": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                            C.POINTER(RasterConfigC), C.POINTER(C.c_int32)]),
    "gpk_graph_capture_train": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                          C.POINTER(RasterConfigC), C.c_double, C.c_double,
                                          C.POINTER(LearningRatesC), C.c_int32, C.POINTER(C.c_int32)]),
    "gpk_graph_capture_train_next": (C.c_int, [_P, C.POINTER(SlicePoseC), C.POINTER(PsfC),
                                          C.POINTER(RasterConfigC), C.c_double, C.c_double,
                                          C.POINTER(LearningRatesC), C.c_int32, C.POINTER(SlicePoseC), C.POINTER(C.c_int32)]),
    "gpk_graph_launch": (C.c_int, [_P, C.c_int32]),
    "gpk_graph_destroy_all": (C.c_int, [_P]),
    "gpk_voxelize": (C.c_int, [_P, C.POINTER(VoxelizerConfigC), _F]),
    "gpk_voxel_tile_count": (C.c_int, [_P, _U64, _U64]),
    "gpk_get_voxel_tile_lists": (C.c_int, [_P, _U32, _U32]),
    "gpk_voxelize_backward": (C.c_int, [_P, C.POINTER(VoxelizerConfigC), _F, _F]),
    "gpk_init_random": (C.c_int, [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64, _D]),
    "gpk_slice_pose_for_index": (C.c_int, [_I32, _D, _D, C.c_int, C.POINTER(SlicePoseC)]),
    "gpk_lr_at": (C.c_double, [C.c_double, C.c_int, C.c_int]),
    "gpk_morton_sort": (C.c_int, [_P, C.c_int32, _U64]),
    "gpk_quantize": (C.c_int, [_P, C.POINTER(QuantSpecC), C.c_int32, _U32, _U32, _U32, _U32, _D, _D]),
    "gpk_encode_streams": (C.c_int, [_P, C.POINTER(QuantSpecC), _P, _P, _P, _P, _D, _D]),
    "gpk_stream_bytes": (C.c_uint64, [C.c_uint64, C.c_int32, C.c_int32]),
    "gpk_decode_streams": (C.c_int, [_P, C.POINTER(QuantSpecC), C.c_uint64, C.POINTER(Bounds), _D, _D, _P, _P, _P,
                                     _P, _F, C.c_int32]),
    "gpk_save_checkpoint": (C.c_int, [_P, C.c_char_p]),
    "gpk_load_checkpoint": (C.c_int, [_P, C.c_char_p]),
    "gpk_checkpoint_bytes": (C.c_uint64, [C.c_uint64]),
    "gpk_get_bounds": (C.c_int, [_P, C.POINTER(Bounds)]),
    "gpk_init_grid": (C.c_int, [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64, _D]),
    "gpk_default_init_count": (C.c_int, [C.c_uint64, _U64]),
    "gpk_rng_create": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "gpk_rng_destroy": (C.c_int, [_P]),
    "gpk_rng_uniform": (C.c_int, [_P, _D]),
    "gpk_rng_below": (C.c_int, [_P, C.c_uint64, _U64]),
    "gpk_rng_normal": (C.c_int, [_P, _D]),
    "gpk_densify_accum_enable": (C.c_int, [_P, C.c_int]),
    "gpk_densify_accum_reset": (C.c_int, [_P]),
    "gpk_get_densify_accum": (C.c_int, [_P, _D, _I32, _D]),
    "gpk_set_densify_accum": (C.c_int, [_P, _D, _I32, _D]),
    "gpk_densify_and_prune": (C.c_int, [_P, C.POINTER(DensifyConfigC), _P, C.POINTER(DensifyReportC)]),
    "gpk_densify_and_prune_draw": (C.c_int, [_P, C.POINTER(DensifyConfigC), NORMAL_FN, _P,
                                             C.POINTER(DensifyReportC)]),
    "gpk_fit": (C.c_int, [_P, _F, _I32, _D, _D, C.POINTER(PsfC), C.POINTER(FitConfigC), PROGRESS_FN, _P]),
    "gpk_nccl_get_unique_id": (C.c_int, [_P]),
    "gpk_comm_init": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "gpk_comm_destroy": (C.c_int, [_P]),
    "gpk_allreduce_grads": (C.c_int, [_P]),
}

for _name, (_res, _args) in _PROTOS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args
if lib.gpk_abi_version() != GPK_ABI_VERSION:
    raise ImportError(f"{LIB_PATH}: ABI {lib.gpk_abi_version()} != {GPK_ABI_VERSION}; rebuild the library")


# ---- error mapping (errors.hpp:9-27 + std::invalid_argument) --------------------
class GpileError(RuntimeError):
    """Base of the exceptions raised for non-OK gpk_status codes."""

    def __init__(self, msg: str, index: int = -1):
        super().__init__(msg)
        self.index = index


class DegenerateCovariance(GpileError):
    """gpile::DegenerateCovariance (errors.hpp:9)."""


class NumericFailure(GpileError):
    """gpile::NumericFailure (errors.hpp:14); .index names the first primitive."""


class InvalidArgument(GpileError, ValueError):
    """std::invalid_argument."""


class CudaError(GpileError):
    pass


class StateError(GpileError):
    pass


class CorruptContainer(GpileError):
    """gpile::CorruptContainer (errors.hpp:19)."""


class LoadError(GpileError):
    """gpile::LoadError (errors.hpp:24)."""


_EXC = {
    GPK_ERR_INVALID_ARGUMENT: InvalidArgument,
    GPK_ERR_DEGENERATE_COVARIANCE: DegenerateCovariance,
    GPK_ERR_NUMERIC_FAILURE: NumericFailure,
    GPK_ERR_CUDA: CudaError,
    GPK_ERR_NCCL: CudaError,
    GPK_ERR_OUT_OF_MEMORY: CudaError,
    GPK_ERR_STATE: StateError,
    GPK_ERR_CORRUPT_CONTAINER: CorruptContainer,
    GPK_ERR_LOAD: LoadError,
}


def check(status: int) -> None:
    if status == GPK_OK:
        return
    msg = (lib.gpk_last_error_message() or b"").decode(errors="replace")
    idx = int(lib.gpk_last_error_index())
    raise _EXC.get(status, GpileError)(msg or f"gpk status {status}", idx)


def fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_F)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_U32)


def i32ptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_I32)


def declared_symbols(header: Path | None = None) -> list[str]:
    """Every function the C header declares (used by the ABI test)."""
    import re

    header = header or (Path(__file__).resolve().parent.parent / "include" / "gpile_b200.h")
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gpk_[a-z0-9_]+)\s*\(", text)))
