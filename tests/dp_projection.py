"""Per-rank cost of the union-compacted data-parallel step at world W, measured
on ONE GPU, and the scaling it implies (a projection, not a scaling run).

This container's runs have one B200, so `bench.py --gpus N` (torchrun, one rank
per GPU, the real NCCL all-reduce) cannot run here. What one rank of a W-GPU
job does on its own GPU can: rank 0's whole training step for the step's W
poses — the cull of all W poses with the candidate union (k_filter_multi),
union numbering, its own slice's render / loss / backward / chain into the
union rows, the exchange, and the scheduled Adam from the summed rows — is
captured as the same CUDA graph `bench.py --gpus W` replays (capture_train_dp),
under a world-size-1 NCCL communicator, so the captured all-reduce is an
identity over one rank. The measured per-rank time therefore excludes only the
cross-GPU transfer; that part is modelled from the measured union size:

    t_ar(W) = alpha + 2 (W - 1) / W * bytes / busbw,   bytes = 44 B x row capacity

(NCCL ring all-reduce; busbw and alpha are stated assumptions, printed with
the result, swept over a range). Projected scaling = W * t_1 / (t_W + t_ar(W)),
t_1 = the single-GPU U2 step (no union, bench.py's headline path).

    python tests/dp_projection.py [--config c5] [--steps 20] [--worlds 1,2,4,8]

Prints one JSON object (profiles/r02_dp_projection.json)."""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2603_20611_b200 as gp  # noqa: E402
from paper_2603_20611_b200 import _native as N  # noqa: E402
from paper_2603_20611_b200 import dp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5", choices=["c2", "c3", "c5"])
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    X, Y, Z = cfg["dims"]
    gs = bench.make_records(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush_src = torch.ones(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    flush_dst = torch.empty((), dtype=torch.float32, device="cuda")
    psf, rcfg, lr0 = gp.PsfSpec(sigma_z=cfg["sigma_z"]), gp.RasterConfig(), gp.LearningRates(*bench.LR0)
    poses = [gp.slice_pose_for_index(cfg["dims"], (1, 1, 1), (0, 0, 0), k) for k in bench.slice_indices(Z)]
    tgt = bench.synthetic_target(cfg)
    out = {"config": cfg["name"], "steps": args.steps, "l2": "flushed (256 MiB read) before each step, outside its window",
           "what": "rank 0 of a W-GPU union-compacted DP step, one GPU, world-1 NCCL communicator "
                   "(captured all-reduce = identity); cross-GPU transfer modelled", "worlds": {}}

    def timed(sess, launch, n_groups):
        for i in range(args.warmup):
            launch(i % n_groups)
        sess.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize()
        torch.cuda._sleep(int(25e-3 * 1.965e9))  # the host queues the loop before the GPU reaches it
        for i in range(args.steps):
            torch.sum(flush_src, dim=0, out=flush_dst)
            ev[i][0].record(stream)
            launch(i % n_groups)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in ev)
        return sum(t) / len(t), t[len(t) // 2]

    def new_session(comm):
        s = gp.Session(0, stream=stream.cuda_stream)
        if comm:
            uid = dp.native_unique_id()
            N.check(N.lib.gpk_comm_init(s.handle, 1, 0, (C.c_char * dp.NCCL_ID_BYTES).from_buffer_copy(uid)))
        s.set_gaussians(gs)
        s.reserve_pairs(max(1 << 20, gs.size()))
        s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        s.synchronize()
        return s

    # t_1: the single-GPU U2 step (bench.py's path: one graph per pose);
    # measured twice (the first run also warms the GPU up), the faster kept
    def single():
        s = new_session(False)
        graphs = [s.capture_train(p, psf, rcfg, bench.LAMBDA, 0.5, lr0, bench.TOTAL_ITERS) for p in poses]
        t, _ = timed(s, lambda k: s.graph_launch(graphs[k]), len(poses))
        s.graph_destroy_all()
        s.close()
        return t

    t1 = min(single(), single())
    out["single_gpu_u2_ms"] = t1
    for W in [int(w) for w in args.worlds.split(",")]:
        s = new_session(True)
        n_groups = len(poses) // W

        def step_poses(k):
            return [poses[j] for j in dp.step_slices(k, W, len(poses))]

        for k in range(n_groups):  # direct steps size the union row capacity (baked into the graphs)
            s.train_step_dp(W, 0, step_poses(k), psf, rcfg, bench.LAMBDA, 0.5, lr0, bench.TOTAL_ITERS)
        s.synchronize()
        rows, cap = s.dp_union_rows()
        g = [s.capture_train_dp(W, 0, step_poses(k), psf, rcfg, bench.LAMBDA, 0.5, lr0, bench.TOTAL_ITERS)
             for k in range(n_groups)]
        tw, tw_med = timed(s, lambda k: s.graph_launch(g[k]), n_groups)
        rows, cap = s.dp_union_rows()
        s.graph_destroy_all()
        s.close()
        nbytes = 44 * cap
        proj = {}
        for busbw in (400.0, 600.0, 800.0):  # GB/s, NCCL all-reduce bus bandwidth over NVLink 5 (assumed)
            for alpha in (10.0, 25.0):  # us, launch + synchronisation latency (assumed)
                tar = 0.0 if W == 1 else (alpha * 1e-3 + 2 * (W - 1) / W * nbytes / (busbw * 1e9) * 1e3)
                proj[f"busbw{int(busbw)}_alpha{int(alpha)}"] = {
                    "allreduce_ms": tar, "step_ms": tw + tar, "slices_per_s": W * 1000.0 / (tw + tar),
                    "scaling_vs_1gpu": W * t1 / (tw + tar)}
        out["worlds"][W] = {"per_rank_ms_no_transfer": tw, "per_rank_ms_median": tw_med, "union_rows": rows,
                            "row_capacity": cap, "exchange_bytes": nbytes, "dense_bytes": 44 * gs.size(),
                            "projection": proj}
        print(f"W={W}: per-rank {tw:.4f} ms (median {tw_med:.4f}), union rows {rows} / cap {cap}, "
              f"{nbytes / 1e6:.1f} MB exchanged; scaling @600GB/s,25us: "
              f"{proj['busbw600_alpha25']['scaling_vs_1gpu']:.2f}x", file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
