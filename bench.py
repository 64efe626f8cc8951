#!/usr/bin/env python
"""bench.py — slices/s of the B200 slice renderer's training step (BASELINE.json metric).

Workload (BASELINE.json configs[1] "light-sheet-like synthetic 512x512x128 stack,
1M Gaussians, fwd+bwd training step on 1 B200"): a 512x512x128
unit-spacing volume, 1M Gaussians from the reference's init_random(seed 1)
(bit-identical stream), PSF sigma_z = 1, RasterConfig defaults, targets U(0, 0.1)
(seed 7). One step = one slice of the reference's fit loop (optimize.hpp:385-402):

  --unit u2 (default): prepare_gaussians + tile binning + rasterize +
      photometric_loss(lambda = 0.2, SSIM) + backward + scheduled Adam;
  --unit u1: prepare + binning + rasterize + backward for a given dL/dI,
      producing the dense (N x 11) gradient.

Slices cycle over 16 mid-stack indices (one CUDA graph per pose). Parameters,
moments and the target are resident in HBM; L2 (126 MB) is flushed by a 256 MiB
read before every timed step, outside the per-step CUDA-event window.
`e2e` is the same step through the C-ABI with host buffers: u2 uploads the
step's target from pinned memory and reads the loss back; u1 uploads dL/dI and
reads the image and the dense gradient back.

Multi-GPU (torchrun): slices are sharded across ranks (rank r renders its own
slice of the step's world poses). u2 exchanges the gradient union-compacted
(gpk_train_step_dp): every rank derives the union of the step's candidates in
its own cull pass, one grouped NCCL all-reduce sums the union rows, every rank
runs the same Adam. The value is all ranks' slices / max-over-ranks device
time (weak scaling).

--impl reference: the reference CPU implementation (oracle/_ref: the unmodified
reference headers compiled here) on this host's cores, same unit, config and
metric, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+bwd slices/s (1/8 GPU) at 512²×128 vol, 1M Gaussians; % HBM roofline"
CONFIGS = {
    "c1": dict(dims=(128, 128, 32), n=20_000, sigma_z=1.0,
               name="synthetic 128x128x32 volume, 20k Gaussians, sigma_z=1"),
    "c2": dict(dims=(512, 512, 128), n=1_000_000, sigma_z=1.0,
               name="light-sheet-like synthetic 512x512x128 stack, 1M Gaussians, sigma_z=1"),
    "c3": dict(dims=(256, 256, 320), n=500_000, sigma_z=3.0,
               name="ABUS-like 256x256x320 volume, thick-slice PSF sigma_z=3, 500k Gaussians"),
    "c5": dict(dims=(2048, 2048, 256), n=8_000_000, sigma_z=1.0,
               name="large microscopy 2048x2048x256 stack, 8M Gaussians, sigma_z=1"),
    "c4": dict(dims=(512, 512, 512), n=1_000_000, sigma_z=1.0,
               name="3D voxelization of a 1M-Gaussian set to a 512^3 grid (8^3 tiles, support 3 sigma)"),
}
VOXEL_METRIC = "voxelizations/s of 1M Gaussians to 512^3 (bit-exact tile binning); % MUFU ex2 roofline"
UNITS = {
    "u2": "U2 training step: prepare + bin + rasterize + photometric loss (lambda 0.2, SSIM) + backward "
          "+ scheduled Adam, one slice",
    "u1": "U1 fwd+bwd slice: prepare + bin + rasterize + backward for a given dL/dI, dense gradients",
}
LAMBDA = 0.2
LR0 = (6e-4, 0.02, 2e-3, 1e-3)      # optimize.hpp:23-26
TOTAL_ITERS = 30000
E2E_WARMUP = 32  # untimed end-to-end steps before the e2e window
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--unit", default="u2", choices=sorted(UNITS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pipeline", action="store_true",
                    help="u2: fuse each step's Adam with the cull of the rank's next slice "
                         "(gpk_graph_capture_train_next); measured slower than the separate kernels on B200")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="submit the step kernel by kernel instead of as a CUDA graph")
    ap.add_argument("--batch", type=int, default=1,
                    help="slices per step (1..8): B slices rendered concurrently on slice contexts; u2: one "
                         "Adam on their summed gradient (gpk_train_step_batch), u1: the summed dense gradient")
    ap.add_argument("--no-batched", action="store_true",
                    help="skip the extra B = 8 measurement reported beside a B = 1 run")
    ap.add_argument("--cpu-1thread-seconds", type=float, default=5.0)
    return ap.parse_args()


def geometry(cfg):
    X, Y, Z = cfg["dims"]
    lo = (-0.5, -0.5, -0.5)
    hi = (X - 0.5, Y - 0.5, Z - 0.5)
    return lo, hi


def slice_indices(Z):
    return [Z // 2 - 8 + i for i in range(16)]


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_field(config, kernel, field):
    """A per-kernel field of the committed ncu capture (profiles/ncu_summary.json)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(config, {}).get(kernel, {}).get(field)
    except Exception:
        return None


def ncu_traffic(config, kernel):
    """dram__bytes_read+write per launch of `kernel` from the committed ncu capture."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(config, {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """Polls NVML during the timed region (SM clock + throttle reasons)."""

    REASONS = {
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sync_boost": 0x10,
        "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    @staticmethod
    def peak_mhz(index: int) -> float:
        try:
            import pynvml

            pynvml.nvmlInit()
            return float(pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(index),
                                                           pynvml.NVML_CLOCK_SM))
        except Exception:
            return 1965.0

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------
def cpu_reference_rate(cfg, rec, unit, seconds_budget, max_reps=None, warmup=1, threads=0):
    """The reference's own CPU implementation (oracle/_ref: its headers compiled
    unmodified) of the same unit on this host's cores. Its slice poses come from
    the reference's slice_pose_for_index (core.hpp:202-211); `rec` is the same
    synthetic set the GPU arm uses."""
    import ctypes as C

    from oracle.bindings import Bounds, CfgC, PoseC, PsfC, load

    ref = load("ref")
    L = ref.lib
    cores = os.cpu_count() or 1
    L.gref_set_threads(threads)  # worker_cap() = 0 -> hardware_concurrency (parallel.hpp:14-20)
    workers = L.gref_effective_workers()
    X, Y, Z = cfg["dims"]
    lo, hi = geometry(cfg)
    b = Bounds((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
    L.gref_set_new.restype = C.c_void_p
    h = L.gref_set_new(C.c_uint64(rec.shape[0]), rec.ctypes.data_as(C.POINTER(C.c_double)), C.byref(b))
    ks = slice_indices(Z)
    poses = (PoseC * len(ks))()
    dims = (C.c_int32 * 3)(X, Y, Z)
    sp = (C.c_double * 3)(1.0, 1.0, 1.0)
    org = (C.c_double * 3)(0.0, 0.0, 0.0)
    L.gref_slice_pose_for_index.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                            C.c_int, C.POINTER(PoseC)]
    for i, k in enumerate(ks):
        if L.gref_slice_pose_for_index(dims, sp, org, k, C.byref(poses[i])) != 0:
            raise RuntimeError("reference slice_pose_for_index failed")
    psf = PsfC(1.0, 1.0, cfg["sigma_z"])
    rc = CfgC(0.02, 16, 3.0, 1.0)
    if unit == "u2":
        img_in = synthetic_target(cfg).astype(np.float64)
        secs = np.zeros(5)
        names = ("prepare", "rasterize", "loss", "backward", "adam")
    else:
        img_in = synthetic_dl_di(cfg).astype(np.float64)
        secs = np.zeros(3)
        names = ("prepare", "rasterize", "backward")

    def run(reps):
        if unit == "u2":
            st = L.gref_time_u2(C.c_void_p(h), poses, len(ks), C.byref(psf), C.byref(rc),
                                img_in.ctypes.data_as(C.POINTER(C.c_double)), C.c_double(LAMBDA), reps,
                                secs.ctypes.data_as(C.POINTER(C.c_double)))
        else:
            st = L.gref_time_u1(C.c_void_p(h), poses, len(ks), C.byref(psf), C.byref(rc),
                                img_in.ctypes.data_as(C.POINTER(C.c_double)), reps,
                                secs.ctypes.data_as(C.POINTER(C.c_double)))
        if st != 0:
            raise RuntimeError("reference step failed")
        return secs.sum(), secs.copy()

    t1, _ = run(max(1, warmup))  # warm (page-in, allocator)
    t1 /= max(1, warmup)
    reps = max(1, int(seconds_budget / max(t1, 1e-6)))
    if max_reps:
        reps = min(reps, max_reps)
    t, parts = run(reps)
    L.gref_set_free(C.c_void_p(h))
    calls = ("prepare_gaussians+rasterize_prepared+photometric_loss+backward_prepared+adam_step" if unit == "u2"
             else "prepare_gaussians+rasterize_prepared+backward_prepared")
    return {
        "value": reps / t, "unit": "slices/s", "cores": int(workers), "host_cpus": cores,
        "kind": "reference", "reps": reps, "seconds": t,
        "stage_seconds_per_slice": {n: float(parts[i] / reps) for i, n in enumerate(names)},
        "sample": f"{reps} {unit.upper()} slices ({calls}) of {cfg['name']}, oracle/_ref with {workers} threads",
    }


def synthetic_target(cfg):
    X, Y, _ = cfg["dims"]
    return np.random.default_rng(7).uniform(0.0, 0.1, (Y, X)).astype(np.float32)


def synthetic_dl_di(cfg):
    X, Y, _ = cfg["dims"]
    rng = np.random.default_rng(7)
    return (rng.uniform(-1.0, 1.0, (Y, X)) / (X * Y)).astype(np.float32)


def make_records(cfg, via_reference=False):
    """init_random(N, world bounds, 1.5, seed 1) (optimize.hpp:94-108), rounded
    to f32 so both arms see identical values. The reference arm draws it with
    the reference's own Rng (oracle/_ref); the GPU arm with the bit-identical
    host port in the C-ABI (tests/test_abi.py pins the equality)."""
    import ctypes as C

    lo, hi = geometry(cfg)
    if via_reference:
        from oracle.bindings import Bounds, load

        L = load("ref").lib
        rec = np.zeros((cfg["n"], 11), np.float64)
        bnd = Bounds((C.c_double * 3)(*lo), (C.c_double * 3)(*hi))
        L.gref_init_random.argtypes = [C.c_uint64, C.POINTER(Bounds), C.c_double, C.c_uint64,
                                       C.POINTER(C.c_double)]
        if L.gref_init_random(cfg["n"], C.byref(bnd), 1.5, 1, rec.ctypes.data_as(C.POINTER(C.c_double))) != 0:
            raise RuntimeError("reference init_random failed")
        return rec.astype(np.float32).astype(np.float64)
    import paper_2603_20611_b200 as gp

    gs = gp.init_random(cfg["n"], lo, hi, 1.5, 1)
    return gp.GaussianSet(gs.records.astype(np.float32).astype(np.float64), lo, hi)


def config_json(args, cfg, world):
    X, Y, Z = cfg["dims"]
    B = getattr(args, "batch", 1)
    unit = UNITS[args.unit] + (
        " (Adam fused with the next slice's cull)" if args.unit == "u2" and getattr(args, "pipeline", False) else "")
    if B > 1:
        unit += (f"; {B} slices per step on slice contexts, " +
                 ("one Adam on their summed gradient" if args.unit == "u2" else "their gradients summed"))
    return {"workload": cfg["name"], "unit_of_work": unit,
            "volume": [X, Y, Z], "gaussians": cfg["n"], "sigma_z": cfg["sigma_z"],
            "slices": f"{len(slice_indices(Z))} mid-stack indices, cycled, {B} per step",
            "slices_per_step": B,
            "parallelism": f"slice-sharded dp{world}",
            "l2": "flushed (256 MiB read) before each timed step, outside the event window; "
                  "steady_state = the same steps back to back without the flush",
            "config_id": args.config,
            "state": "every measured section (timed, steady state, batched, stages, e2e) starts from the "
                     "initial parameters and Adam moments"}


def data_note(unit):
    return ("synthetic (init_random seed 1; targets U(0,0.1) seed 7)" if unit == "u2"
            else "synthetic (init_random seed 1; dL/dI U(-1,1)/P seed 7)")


# ---------------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    rec = make_records(cfg, via_reference=True)
    budget = min(150.0, max(10.0, 1.0 * args.steps))
    res = cpu_reference_rate(cfg, rec, args.unit, budget, max_reps=args.steps, warmup=min(args.warmup, 10))
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "slices/s",
        "n_gpus": args.gpus, "steps": res["reps"], "warmup": min(args.warmup, 10), "ms_per_step": 1000.0 / res["value"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": data_note(args.unit), "config": config_json(args, cfg, world),
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stage_seconds_per_slice": res["stage_seconds_per_slice"],
    }
    print(json.dumps(line), flush=True)
    return 0


def sort_passes(X, Y):
    tiles = ((X + 15) // 16) * ((Y + 15) // 16)
    bits = max(1, (tiles - 1).bit_length())
    return (bits + 9) // 10


def run_voxel(args, impl):
    """C4: voxelize (voxelize.hpp:113-148) of the 1M init_random
    set on a 512^3 unit grid. One step = one voxelize call (primitive prep +
    8^3-tile binning + per-tile evaluation of every voxel of every touched tile,
    the reference's loop). The evaluation is MUFU-bound: one ex2 per (voxel,
    primitive) of a touched tile; its roofline is the ex2 rate."""
    import ctypes as C

    cfg = CONFIGS["c4"]
    X, Y, Z = cfg["dims"]
    V = X * Y * Z
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    base = {"metric": VOXEL_METRIC, "unit": "voxelizations/s", "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "data": "synthetic (init_random seed 1 over the grid's world bounds)",
            "config": {"workload": cfg["name"], "dims": [X, Y, Z], "gaussians": cfg["n"], "tile": [8, 8, 8],
                       "support_sigmas": 3.0, "config_id": "c4",
                       "parallelism": "replicas only (one voxelization per GPU)"}}

    def ref_rate(threads, seconds):
        from oracle.bindings import VcfgC, load

        ref = load("ref")
        L = ref.lib
        L.gref_set_threads(threads)
        workers = L.gref_effective_workers()
        rec = make_records(cfg, via_reference=True)
        h = ref._set(rec, geometry(cfg))
        vc = VcfgC((C.c_int32 * 3)(X, Y, Z), (C.c_double * 3)(1, 1, 1), (C.c_double * 3)(0, 0, 0),
                   (C.c_int32 * 3)(8, 8, 8), 3.0, 1.0)
        secs = C.c_double()
        L.gref_time_voxelize.argtypes = [C.c_void_p, C.POINTER(VcfgC), C.c_int, C.POINTER(C.c_double)]
        if L.gref_time_voxelize(C.c_void_p(h.h), C.byref(vc), 1, C.byref(secs)) != 0:
            raise RuntimeError("reference voxelize failed")
        reps = max(1, min(int(seconds / max(secs.value, 1e-6)), 20))
        if L.gref_time_voxelize(C.c_void_p(h.h), C.byref(vc), reps, C.byref(secs)) != 0:
            raise RuntimeError("reference voxelize failed")
        return {"value": reps / secs.value, "unit": "voxelizations/s", "cores": int(workers), "kind": "reference",
                "sample": f"{reps} voxelize calls of {cfg['name']}, oracle/_ref with {workers} threads"}

    if impl == "reference":
        if rank != 0:
            return 0
        r = ref_rate(0, min(150.0, max(20.0, 2.0 * args.steps)))
        line = dict(base, impl="reference", value=r["value"], n_gpus=args.gpus, steps=args.steps,
                    warmup=args.warmup, ms_per_step=1000.0 / r["value"], dtype="f64",
                    cpu_baseline=r, e2e={"value": r["value"], "unit": "voxelizations/s",
                                         "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return 0

    import torch

    import paper_2603_20611_b200 as gp
    from paper_2603_20611_b200 import dp

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    s = gp.Session(local, stream=stream.cuda_stream)
    gs = make_records(cfg)
    s.set_gaussians(gs)
    vcfg = gp.VoxelizerConfig(dims=(X, Y, Z))
    s.voxelize(vcfg, to_host=False)
    off, ent = s.voxel_tile_lists()
    inst = len(ent)
    del off, ent
    evals = inst * 512.0  # every voxel of every touched 8^3 tile (voxelize.hpp:137-143)
    for _ in range(max(args.warmup, 2)):
        s.voxelize(vcfg, to_host=False)
    s.synchronize()
    steps = max(3, min(args.steps, 30))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    s.stage_timing(True)
    s.stage_times(reset=True)
    with ClockSampler(local) as clk:
        for i in range(steps):
            ev[i][0].record(stream)
            s.voxelize(vcfg, to_host=False)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    st = s.stage_times(reset=True)
    s.stage_timing(False)
    ms = dp.max_over_ranks([sum(a.elapsed_time(b) for a, b in ev) / steps], device="cuda")[0]
    eval_ms = st["voxel_eval"][0] / max(st["voxel_eval"][1], 1)
    prep_ms = st["voxel"][0] / max(st["voxel"][1], 1)
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clk_mhz = ClockSampler.peak_mhz(local)
    ex2_peak = 16.0 * sm_count * clk_mhz * 1e6
    peak, peak_src = load_peaks()
    # e2e: the public call with the volume copied to host memory (pinned)
    vol = torch.empty(V, dtype=torch.float32).pin_memory()
    e_steps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_2603_20611_b200 import _native as N

    e0.record(stream)
    for _ in range(e_steps):
        s.voxelize(vcfg, to_host=False)
        s.download(N.GPK_BUF_VOLUME, vol.data_ptr(), V * 4)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1) / e_steps
    line = dict(base, value=world * 1000.0 / ms, n_gpus=world, steps=steps, warmup=args.warmup, ms_per_step=ms,
                dtype="f32 (fp64 support bounds)")
    line["roofline"] = {"kernel": "k_veval", "bound": "mufu", "achieved": evals / (eval_ms * 1e-3),
                        "peak": ex2_peak, "unit": "ex2/s", "frac": evals / (eval_ms * 1e-3) / ex2_peak,
                        "traffic": None, "launch_ms": eval_ms, "evals_per_launch": evals,
                        "basis": f"one ex2 per (voxel, primitive) of a touched tile: 512 x {inst} tile "
                                 f"instances; 16 ex2/clk/SM x {sm_count} SMs x {clk_mhz:.0f} MHz"}
    line["hbm_roofline"] = {"bytes_per_step": 44 * cfg["n"] + 4 * V,
                            "achieved_gbs": (44 * cfg["n"] + 4 * V) / (ms * 1e-3) / 1e9, "peak": peak,
                            "frac": (44 * cfg["n"] + 4 * V) / (ms * 1e-3) / 1e9 / peak, "peak_source": peak_src,
                            "formula": "44N params + 4V volume"}
    line["stage_ms"] = {"prims_and_tile_lists": prep_ms, "evaluation": eval_ms}
    line["tile_instances"] = inst
    line["e2e"] = {"value": 1000.0 / e_ms, "unit": "voxelizations/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": V * 4, "path": "C-ABI: gpk_voxelize + gpk_download(volume, pinned)"}
    line["gpu_launches"] = (1 + 2 + 1) * steps  # k_vprep, 2 radix passes, k_veval
    line["clocks"] = clk.result()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = ref_rate(0, args.cpu_seconds)
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    s.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import ctypes as C

    import torch

    import paper_2603_20611_b200 as gp
    from paper_2603_20611_b200 import _native as N
    from paper_2603_20611_b200 import dp

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    u2 = args.unit == "u2"
    cfg = CONFIGS[args.config]
    X, Y, Z = cfg["dims"]
    P = X * Y
    gs = make_records(cfg)
    n = gs.size()
    # A dedicated (non-default) stream shared by the session and the timing events.
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    sess = gp.Session(local, stream=stream.cuda_stream)
    sess.set_gaussians(gs)
    # Training moves the Gaussians (the synthetic target is noise: scales and
    # opacities drift and slices get more pairs), so every measured section
    # below starts from the same initial parameters and moments (restored from
    # this snapshot) and all of them time the same workload.
    p_bytes = sess.device_buffer(N.GPK_BUF_PARAMS)[1]
    init_params = torch.empty(p_bytes // 4, dtype=torch.float32).pin_memory()
    sess.download(N.GPK_BUF_PARAMS, init_params.data_ptr(), p_bytes)
    sess.synchronize()
    init_adam = sess.adam_state()

    def restore_initial_state():
        sess.synchronize()
        sess.upload(N.GPK_BUF_PARAMS, init_params.data_ptr(), p_bytes)
        sess.set_adam_state(*init_adam)
        sess.synchronize()
    sess.reserve_pairs(max(1 << 20, n))
    psf = gp.PsfSpec(sigma_z=cfg["sigma_z"])
    rcfg = gp.RasterConfig()
    lr0 = gp.LearningRates(*LR0)
    ks = slice_indices(Z)
    poses = [gp.slice_pose_for_index(cfg["dims"], (1, 1, 1), (0, 0, 0), k) for k in ks]
    if world > 1:
        dp.init_grad_comm(sess, rank, world)

    B = args.batch
    if not 1 <= B <= 8 or 16 % B:
        raise SystemExit("--batch must be 1, 2, 4 or 8")
    if B > 1 and world > 1:
        raise SystemExit("--batch > 1 is single-GPU (the batched step has no collective)")
    tgt = synthetic_target(cfg)
    dl = synthetic_dl_di(cfg)
    batch_ctx = 8 if (B == 1 and world == 1 and not args.no_batched) else B
    for k in range(batch_ctx):  # slice k of a batched step reads context k's target / dL/dI
        c = sess.context(k)
        c.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        c.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    # u2, one slice per step: two target slots (gpk_set_target_slot), graph k
    # reading slot k mod 2 (the poses cycle with an even period), so a step's
    # target upload never waits for the previous step's last target reader
    slots = u2 and B == 1
    if slots:
        for k in (1, 0):
            sess.set_target_slot(k)
            sess.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    # u2: every slice context's loss kernel writes its loss straight into this
    # pinned host array (gpk_set_loss_sink): the step's result reaches the host
    # inside the step, no separate read-back copy (set before any capture)
    loss_sink = torch.zeros(max(batch_ctx, 1), dtype=torch.float64).pin_memory()
    if u2:
        for k in range(batch_ctx):
            sess.context(k).set_loss_sink(loss_sink.data_ptr() + 8 * k)
    sess.synchronize()
    # per-slice counters (algorithmic bytes of the prepare kernels) and the
    # reference's pixel-pair evaluation count (render.hpp:179-181: every pixel of
    # tile x bounds; the tiles partition the image, so sum of bound areas)
    counts, evals = [], []
    for p in poses:
        sess.prepare(p, psf, rcfg)
        counts.append(sess.prepare_stats())
        b = sess.prepared().bounds.astype(np.int64)
        evals.append(float(((b[:, 1] - b[:, 0] + 1) * (b[:, 3] - b[:, 2] + 1)).sum()))
    S_mean = float(np.mean([c["survivors"] for c in counts]))
    T_mean = float(np.mean([c["pairs"] for c in counts]))
    C_mean = float(np.mean([c["candidates"] for c in counts]))
    X64_mean = float(np.mean([c["fp64_decided"] for c in counts]))
    E_mean = float(np.mean(evals))

    # L2 flush by READING 256 MiB (> 126 MB L2): evicts the step's working set
    # without leaving dirty lines whose write-back would bill the next kernel.
    flush_src = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    flush_dst = torch.empty((), dtype=torch.float32, device="cuda")

    def flush():
        torch.sum(flush_src, dim=0, out=flush_dst)

    def host_ahead(ms=25.0):
        # hold the stream for `ms` so the host queues the whole timed loop
        # before the GPU reaches it: the event windows then time the device
        # work of each step, not the Python loop's submission jitter
        torch.cuda._sleep(int(ms * 1e-3 * ClockSampler.peak_mhz(local) * 1e6))

    # step i renders group i mod n_groups (B consecutive poses); data-parallel
    # u2: step i's world poses (dp.step_slices), rank r renders the r-th
    dp_union = u2 and world > 1
    n_groups = len(poses) // (world if dp_union else B)

    def step_poses(k):
        return [poses[j] for j in dp.step_slices(k, world, len(poses))]

    def group(k, nb=None):
        nb = nb or B
        return [poses[(k * nb + b) % len(poses)] for b in range(nb)]

    def capture(k, nb=None):
        nb = nb or B
        if slots and (nb or B) == 1:
            sess.set_target_slot(k % 2)
        if dp_union:
            return sess.capture_train_dp(world, rank, step_poses(k), psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS)
        if nb > 1:
            return (sess.capture_train_batch(group(k, nb), psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS) if u2
                    else sess.capture_fwd_bwd_batch(group(k, nb), psf, rcfg))
        # u2 --pipeline: the step's Adam is fused with the cull of this rank's
        # next slice (gpk_graph_capture_train_next), so each step starts at K_decide
        if u2:
            return sess.capture_train(poses[k], psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS,
                                      next_pose=poses[(k + world) % len(poses)] if args.pipeline else None)
        return sess.capture_fwd_bwd(poses[k], psf, rcfg)

    union_rows = [(0, 0)]
    if dp_union:
        # the union row capacity (the all-reduce count, baked into the graphs)
        # grows on direct steps; every rank runs the same steps, so every rank
        # ends with the same capacity
        for k in range(n_groups):
            sess.train_step_dp(world, rank, step_poses(k), psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS)
        sess.synchronize()
        union_rows = [sess.dp_union_rows()]

    # one CUDA graph per slice pose (group of B poses): the whole step is one submission
    graphs = [capture(k) for k in range(n_groups)] if args.graphs else None

    def step(i):
        k = i % n_groups if dp_union else dp.slice_for(i, rank, world, n_groups)
        if graphs is not None:
            sess.graph_launch(graphs[k])
        elif dp_union:
            sess.train_step_dp(world, rank, step_poses(k), psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS)
        elif B > 1:
            if u2:
                sess.train_step_batch(group(k), psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS)
            else:
                sess.fwd_bwd_batch(group(k), psf, rcfg)
        elif u2:  # all-reduce inside
            sess.train_step(poses[k], psf, rcfg, LAMBDA, 0.5, lr0, TOTAL_ITERS,
                            next_pose=poses[(k + world) % len(poses)] if args.pipeline else None)
        else:
            sess.fwd_bwd_slice(poses[k], psf, rcfg)
        if world > 1 and not u2:
            dp.allreduce_grads(sess)

    restore_initial_state()
    for i in range(args.warmup):
        step(i)
    sess.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        host_ahead()
        for i in range(args.steps):
            flush()
            starts[i].record(stream)
            step(args.warmup + i)
            ends[i].record(stream)
        torch.cuda.synchronize()
    sess.synchronize()
    if dist:
        dist.barrier()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    total_ms = dp.max_over_ranks([total_ms], device="cuda")[0]
    ms_per_step = total_ms / args.steps
    value = world * B * 1000.0 / ms_per_step

    # steady state: the same steps back to back, no flush (a training loop's
    # regime: the previous step's dirty lines are written back inside this one)
    ss_steps = min(args.steps, 100)
    restore_initial_state()
    for i in range(3):
        step(i)
    ss0, ss1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ss0.record(stream)
    for i in range(ss_steps):
        step(args.warmup + args.steps + i)
    ss1.record(stream)
    torch.cuda.synchronize()
    ss_ms = dp.max_over_ranks([ss0.elapsed_time(ss1) / ss_steps], device="cuda")[0]

    # the same workload B = 8 slices per step (batched step, single GPU), beside a B = 1 run
    batched = None
    if B == 1 and world == 1 and not args.no_batched and args.graphs:
        bg = [capture(k, 8) for k in range(len(poses) // 8)]
        restore_initial_state()
        for i in range(3):
            sess.graph_launch(bg[i % len(bg)])
        torch.cuda.synchronize()
        nb_steps = max(10, min(args.steps // 4, 50))
        bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(nb_steps)]
        for i in range(nb_steps):
            flush()
            bev[i][0].record(stream)
            sess.graph_launch(bg[i % len(bg)])
            bev[i][1].record(stream)
        torch.cuda.synchronize()
        b_ms = sum(a.elapsed_time(b) for a, b in bev) / nb_steps
        batched = {"slices_per_step": 8, "ms_per_step": b_ms, "value": 8 * 1000.0 / b_ms, "unit": "slices/s",
                   "steps": nb_steps, "unit_of_work": ("8 slices rendered concurrently on slice contexts, "
                                                       + ("one Adam on their summed gradient" if u2
                                                          else "their gradients summed")),
                   "l2": "flushed before each step"}
        sess.graph_destroy_all()
        graphs = [capture(k) for k in range(n_groups)]

    # per-kernel device time: the same steps through graphs captured with an
    # event-record node around every stage (device-side timestamps; the nodes
    # themselves add ~2-4 us per stage, so these over-state each stage a little)
    # (B > 1: only the session's own stream is bracketed: slice 0's kernels and Adam)
    prof_steps = min(args.steps, 100)
    restore_initial_state()
    sess.stage_timing(True)
    prof_graphs = [capture(k) for k in range(n_groups)]
    sess.stage_times(reset=True)
    for i in range(prof_steps):
        flush()
        j = args.warmup + i
        sess.graph_launch(prof_graphs[j % n_groups if dp_union else dp.slice_for(j, rank, world, n_groups)])
    sess.stage_timing(False)
    stages = sess.stage_times(reset=True)

    # ---- e2e through the public C-ABI with host buffers ---------------------------
    e2e_steps = max(5, min(args.steps, 50))
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps)]
    e_e = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_steps)]
    ctxs = [sess.context(b) for b in range(B)]
    restore_initial_state()
    if u2:
        # the step's B targets (one per slice context) up, its B losses down
        pin_tgt = [torch.from_numpy(tgt).pin_memory() for _ in range(B)]
        pin_loss = torch.empty(B, dtype=torch.float64).pin_memory()

        def e2e_step(i, down=False):
            if slots:  # the slot graph k reads (k = the step's pose group)
                k = i % n_groups if dp_union else dp.slice_for(i, rank, world, n_groups)
                sess.set_target_slot(k % 2)
            for b in range(B):
                ctxs[b].upload(N.GPK_BUF_TARGET, pin_tgt[b].data_ptr(), P * 4)
            step(i)
            if down:  # (the loss sink already holds them; debug comparison only)
                for b in range(B):
                    ctxs[b].download(N.GPK_BUF_LOSS, pin_loss.data_ptr() + 8 * b, 8)

        # warm-up of the copy path: the first transfers from freshly pinned
        # pages are slow on the box's host (measured: a pinned 1 MB upload
        # settles after tens of transfers, tests/_h2d_probe.py)
        for i in range(E2E_WARMUP):
            flush()
            e2e_step(i)
        sess.synchronize()
        # ... and the timed loop's own regime (queued behind a device sleep,
        # events recorded), untimed: measured on the box, the first such queued
        # run of uploads is slower than every later one
        for _ in range(2):
            torch.cuda.synchronize()
            host_ahead()
            for i in range(e2e_steps):
                flush()
                e_s[i].record(stream)
                e2e_step(i)
                e_e[i].record(stream)
            torch.cuda.synchronize()
        restore_initial_state()
        # the steps are queued back to back, the host never waits inside the
        # loop (a training loop's regime: copies and launches run ahead of the
        # GPU); each step's window — its target upload, the step, its loss
        # read-back — is bracketed by events, the L2 flush stays outside it
        torch.cuda.synchronize()
        host_ahead()
        for i in range(e2e_steps):
            flush()
            e_s[i].record(stream)
            e2e_step(i)
            e_e[i].record(stream)
        torch.cuda.synchronize()
        # the sink holds the last step's losses: the device's own values
        for b in range(B):
            ctxs[b].download(N.GPK_BUF_LOSS, pin_loss.data_ptr() + 8 * b, 8)
        torch.cuda.synchronize()
        assert np.isfinite(pin_loss.numpy()).all()
        assert np.array_equal(pin_loss.numpy(), loss_sink.numpy()[:B]), "loss sink != device loss"
        if os.environ.get("GPK_BENCH_E2E_DEBUG"):  # where the window's time goes (stderr)
            for name, up, down in (("graph", 0, 0), ("up+graph", 1, 0), ("+download", 1, 1)):
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(e2e_steps)]
                host_ahead()
                for i in range(e2e_steps):
                    flush()
                    ev[i][0].record(stream)
                    if up:
                        for b in range(B):
                            ctxs[b].upload(N.GPK_BUF_TARGET, pin_tgt[b].data_ptr(), P * 4)
                    step(i)
                    if down:
                        for b in range(B):
                            ctxs[b].download(N.GPK_BUF_LOSS, pin_loss.data_ptr() + 8 * b, 8)
                    # (up only: the loss still reaches the host through the sink)
                    ev[i][1].record(stream)
                torch.cuda.synchronize()
                t = sorted(a.elapsed_time(b) for a, b in ev)
                print(f"e2e debug {name:10s} median {t[len(t) // 2] * 1e3:7.1f} us  min {t[0] * 1e3:7.1f}",
                      file=sys.stderr, flush=True)
        h2d, d2h = B * P * 4, B * 8
        e2e_path = (f"C-ABI: gpk_upload(target, pinned) x {B} + train step (graph); the loss kernel writes "
                    f"each f64 loss into pinned host memory (gpk_set_loss_sink) x {B}")
    else:
        pin_dl = [torch.from_numpy(dl).pin_memory() for _ in range(B)]
        pin_img = torch.empty(B * P, dtype=torch.float32).pin_memory()
        _, gbytes = sess.device_buffer(N.GPK_BUF_GRADS)
        pin_grads = torch.empty(gbytes // 4, dtype=torch.float32).pin_memory()

        def e2e_step(i):
            for b in range(B):
                ctxs[b].upload(N.GPK_BUF_DL_DI, pin_dl[b].data_ptr(), P * 4)
            step(i)
            for b in range(B):
                ctxs[b].download(N.GPK_BUF_IMAGE, pin_img.data_ptr() + 4 * P * b, P * 4)
            sess.download(N.GPK_BUF_GRADS, pin_grads.data_ptr(), gbytes)  # dense gradient planes

        for i in range(E2E_WARMUP):  # warm-up of the copy path (as above)
            flush()
            e2e_step(i)
        sess.synchronize()
        torch.cuda.synchronize()
        host_ahead()
        for i in range(e2e_steps):
            flush()
            e_s[i].record(stream)
            e2e_step(i)
            e_e[i].record(stream)
        torch.cuda.synchronize()
        assert np.isfinite(pin_grads.numpy()[:1000]).all()
        h2d, d2h = B * P * 4, B * P * 4 + gbytes
        e2e_path = (f"C-ABI: gpk_upload(dL/dI) x {B} + fwd_bwd (graph) + gpk_download(image) x {B} "
                    "+ gpk_download(dense gradients)")
    e2e_each = sorted(s.elapsed_time(e) for s, e in zip(e_s, e_e))
    e2e_ms = sum(e2e_each) / e2e_steps
    e2e_ms = dp.max_over_ranks([e2e_ms], device="cuda")[0]
    # the box's pinned host->device copy time of one step's input (the e2e
    # window waits for it when it exceeds the step's time to the loss; it
    # varies between boxes and over time on this pool)
    probe_src = torch.from_numpy(np.ascontiguousarray(tgt if u2 else dl)).pin_memory()
    probe_dst = torch.empty(probe_src.numel(), dtype=torch.float32, device="cuda")
    probe_stream = torch.cuda.Stream(device=local)
    h2d_us = []
    for i in range(21):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(probe_stream):
            a0.record(probe_stream)
            probe_dst.copy_(probe_src.view(-1), non_blocking=True)
            a1.record(probe_stream)
        probe_stream.synchronize()
        if i:
            h2d_us.append(a0.elapsed_time(a1) * 1e3)
    h2d_us.sort()

    # ---- roofline of the dominant kernel -------------------------------------------
    # Algorithmic bytes per launch (each logical tensor read or written once at its
    # stored width): N Gaussians, C candidates, S survivors, T pairs, P px.
    S, T, Cc = S_mean, T_mean, C_mean
    passes = sort_passes(X, Y)
    kernel_bytes = {
        "prepare": ("k_filter", 44 * n + 48 * Cc + 4 * (n / 128),
                    "44N params + 48C candidate records + 4N/128 counts"),
        "bin": ("k_decide", 48 * Cc + 48 * S + 48 * S + 4 * S + 4 * T + 4 * 1025 * (n / 4096),
                "48C candidates + 48S records + 48S survivor params + 4S set indices + 4T slots + bucket table"),
        "sort": ("k_gather" if passes == 1 else "k_sort_pass x passes",
                 8 * T if passes == 1 else 16 * T * passes,
                 "8T (bucketed slots in, tile lists out)" if passes == 1 else "16T per radix pass"),
        "raster": ("k_raster_fwd", 52 * T + 4 * P + (8 * T if u2 and passes == 1 else 0),
                   "52T (slot + 48 B record per pair) + 4P image"
                   + (" + 8T fused gather (bucketed slots in, tile lists out)" if u2 and passes == 1 else "")),
        "backward": ("k_raster_bwd", 52 * T + 4 * P + 24 * T + (20 * P if u2 else 0),
                     "52T + 4P dL/dI + 24T partials" + (" + 20P fused SSIM backward" if u2 else "")),
        "chain": ("k_chain", 48 * S + 48 * S + 24 * T + 44 * S + (2 * S if u2 else 4 * S),
                  "48S records + 48S params + 24T partials + 44S gradients"
                  + (" (by survivor slot) + 2S slot map" if u2 else " + 4S dirty list")),
        "loss": ("k_ssim_fwd", 20 * P, "8P images + 12P SSIM partials (the backward half runs in k_raster_bwd)"),
        # slot-gradient Adam (single-GPU step): the survivors' gradients by slot
        # + a 2 B map per primitive instead of 44 B dense gradient planes
        "adam": ("k_adam_cull", 266 * n + 44 * S + 48 * Cc,
                 "266N + 44S: read params, m, v, 2 B slot map; write params, m, v; survivor gradients "
                 "+ 48C next-slice candidates")
        if (u2 and args.pipeline and world == 1 and os.environ.get("GPK_LAZY_ADAM") != "1") else
        ("k_lazy_survivors + k_lazy_window", 322 * S + (n / 16) * 272,
         "322S + 272N/16: the survivors' params, m, v read and written, their slot gradients, t_done, set "
         "index, map; the step's 1/16 window of params, m, v, t_done read and written (lazy mode)")
        if (u2 and world == 1 and B == 1 and os.environ.get("GPK_LAZY_ADAM") == "1") else
        ("k_adam_final", 264 * S + 44 * S + 6 * S,
         "264S + 44S + 6S: the survivors' params, m, v read and written, their slot gradients, set index, map")
        if (world == 1 and B == 1 and "adam_rest" in stages and stages["adam_rest"][1]) else
        ("k_adam", 266 * n + 44 * S,
         "266N + 44S: read params, m, v, 2 B slot map; write params, m, v; survivor gradients")
        if world == 1 else
        ("k_adam", 268 * n + 44 * union_rows[0][0],
         "268N + 44M: read params, m, v, 4 B union map; write params, m, v; the M summed union rows"),
        # the non-survivors' Adam, on a side stream beside the render (split step)
        "adam_rest": ("k_adam_rest", 264 * (n - S) + n / 8,
                      "264(N-S): the non-survivors' params, m, v read and written + N/8 survivor bits"),
    }
    measured = {k: v for k, v in stages.items() if v[1] > 0 and k in kernel_bytes}
    dom = max(measured, key=lambda k: measured[k][0])
    peak, peak_src = load_peaks()
    launch_ms = measured[dom][0] / measured[dom][1]
    kname, kbytes, kformula = kernel_bytes[dom]
    achieved = kbytes / (launch_ms * 1e-3) / 1e9
    roof = {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": ncu_traffic(args.config, kname.split(" ")[0]),
            "peak_source": peak_src, "bytes_per_launch": kbytes, "launch_ms": launch_ms,
            "bytes_formula": kformula}
    per_kernel = {}
    for k, (ms_tot, cnt) in measured.items():
        kn, kb, _ = kernel_bytes[k]
        ms = ms_tot / cnt
        per_kernel[kn] = {"ms": ms, "gbs": kb / (ms * 1e-3) / 1e9, "frac": kb / (ms * 1e-3) / 1e9 / peak}
    # The pixel kernels are not HBM-bound: their work is one exp per pixel and
    # (tile, Gaussian) pair of the reference's loops (render.hpp:179-181,
    # backward.hpp:120-137): E = sum over survivors of the bound area. Their
    # roofline is the MUFU ex2 rate (16 per SM per clock).
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    clk_mhz = ClockSampler.peak_mhz(local)
    ex2_peak = 16.0 * sm_count * clk_mhz * 1e6
    compute_roof = {"ex2_peak_per_s": ex2_peak, "evals_per_slice": E_mean,
                    "basis": f"16 ex2/clk/SM x {sm_count} SMs x {clk_mhz:.0f} MHz; E = sum of survivor bound areas"}
    for stg, kn in (("raster", "k_raster_fwd"), ("backward", "k_raster_bwd")):
        if stg in measured:
            ms = measured[stg][0] / measured[stg][1]
            compute_roof[kn] = {"ms": ms, "evals_per_s": E_mean / (ms * 1e-3),
                                "frac": E_mean / (ms * 1e-3) / ex2_peak}
            # the bound these kernels actually meet is instruction issue: the
            # committed ncu capture's warp instructions per SM cycle / 4
            # (profiles/ncu_summary.json; cold, serialised)
            ipc = ncu_field(args.config, kn, "ipc_per_sm")
            if ipc is not None:
                compute_roof[kn]["issue"] = {"ipc_per_sm": ipc, "peak_ipc": 4.0, "frac": ipc / 4.0,
                                             "source": "ncu --set full (profiles/ncu_summary.json)"}
    # U2 floor with slot gradients: 44N cull read + 264N Adam (p, m, v read and
    # written) + 2N slot map (SURVEY.md §8d's 396N assumed dense gradient
    # planes: +44N Adam read, +44N clear)
    step_bytes = ((310 * n + 8 * P) if world == 1 else (44 * n + 4 * n + 268 * n + 88 * union_rows[0][0] + 8 * P)) \
        if u2 else (88 * n + 8 * P)
    step_gbs = step_bytes / (ms_per_step * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": "slices/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 cull/bounds decisions and chain)",
        "data": data_note(args.unit), "config": config_json(args, cfg, world),
        "roofline": roof,
        "step_roofline": {"bytes_per_step": step_bytes, "achieved_gbs": step_gbs, "frac": step_gbs / peak,
                          "formula": (("310N + 8P (U2 with slot gradients; SURVEY.md §8d: 396N dense)" if world == 1
                                       else "44N cull + 4N union map + 268N Adam + 88M union rows + 8P per rank "
                                            "(U2, union-compacted exchange; the all-reduce excluded)")
                                      if u2 else "88N + 8P (U1, SURVEY.md §8d)")},
        "steady_state": {"ms_per_step": ss_ms, "value": world * B * 1000.0 / ss_ms, "steps": ss_steps,
                         "note": "no L2 flush between steps (back-to-back training loop)"},
        "stage_ms_per_step": {k: v[0] / max(v[1], 1) for k, v in stages.items() if v[1]},
        "compute_roofline": compute_roof,
        "kernels": per_kernel,
        "submission": "CUDA graph per slice pose" if graphs is not None else "kernel by kernel",
        "survivors_mean": S_mean, "pairs_mean": T_mean, "candidates_mean": C_mean,
        "fp64_decided_mean": X64_mean,
        "e2e": {"value": world * B * 1000.0 / e2e_ms, "unit": "slices/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "path": e2e_path,
                "ms_min": e2e_each[0], "ms_median": e2e_each[len(e2e_each) // 2], "ms_max": e2e_each[-1],
                "h2d_probe_us": {"bytes": probe_src.numel() * 4, "median": h2d_us[len(h2d_us) // 2],
                                 "min": h2d_us[0], "max": h2d_us[-1]}},
        "gpu_launches": None,
        "clocks": clk.result(),
    }
    if dp_union:
        line["exchange"] = {"kind": "union-compacted: one grouped ncclAllReduce of the step's union rows",
                            "union_rows": union_rows[0][0], "row_capacity": union_rows[0][1],
                            "bytes_per_rank": 44 * union_rows[0][1], "dense_bytes": 44 * n}
    if batched:
        line["batched"] = batched
    # per slice: filter + decide + (gather | radix passes) + forward + backward + chain + chain_exact;
    # u2: the gather runs inside the forward, + SSIM forward (its backward runs in the raster
    # backward), + Adam constants + Adam once per step (--pipeline: the filter is fused into
    # Adam); u1 x B: + one gradient scatter per slice. Memsets are not kernels.
    sort_k = passes if passes > 1 else (0 if u2 else 1)
    per_slice = 2 + sort_k + 4 + (1 if u2 else 0)
    split = "adam_rest" in stages and stages["adam_rest"][1] > 0  # Adam in two kernels (rest + final)
    launches = B * per_slice + (2 if u2 else (B if B > 1 else 0)) + (2 if dp_union else 0) + (1 if split else 0)
    if u2 and args.pipeline:
        launches -= 1
    line["gpu_launches"] = launches * args.steps
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = {k: v for k, v in cpu_reference_rate(cfg, gs.records, args.unit,
                                                                        args.cpu_seconds).items()
                                    if k in ("value", "unit", "cores", "kind", "sample",
                                             "stage_seconds_per_slice")}
            one = cpu_reference_rate(cfg, gs.records, args.unit, args.cpu_1thread_seconds, threads=1)
            line["cpu_baseline"]["one_thread"] = {k: one[k] for k in ("value", "unit", "cores", "sample")}
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    sess.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.config == "c4":
        return run_voxel(args, args.impl)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
