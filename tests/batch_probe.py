"""Probe (not a test): device time per slice of the batched steps at a config,
CUDA graphs, CUDA events on the session stream, with and without an L2 flush
between steps. Usage: python tests/batch_probe.py [c2|c3|c5] [steps]."""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2603_20611_b200 as gp
    from paper_2603_20611_b200 import _native as N

    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    X, Y, Z = cfg["dims"]
    gs = bench.make_records(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s = gp.Session(0, stream=stream.cuda_stream)
    s.set_gaussians(gs)
    s.reserve_pairs(max(1 << 20, gs.size()))
    psf, rc, lr0 = gp.PsfSpec(sigma_z=cfg["sigma_z"]), gp.RasterConfig(), gp.LearningRates(*bench.LR0)
    ks = bench.slice_indices(Z)
    poses = [gp.slice_pose_for_index(cfg["dims"], (1, 1, 1), (0, 0, 0), k) for k in ks]
    tgt, dl = bench.synthetic_target(cfg), bench.synthetic_dl_di(cfg)
    for k in range(8):
        c = s.context(k)
        c.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        c.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    s.synchronize()
    flush_src = torch.ones((256 << 20) // 4, device="cuda")
    flush_dst = torch.empty((), device="cuda")
    out = {}
    for unit in ("u2", "u1"):
        for B in (1, 2, 4, 8):
            groups = [poses[(g * B) % 16:(g * B) % 16 + B] for g in range(16 // B)]
            if unit == "u2":
                gids = [s.capture_train_batch(g, psf, rc, 0.2, 0.5, lr0, 30000) if B > 1
                        else s.capture_train(g[0], psf, rc, 0.2, 0.5, lr0, 30000) for g in groups]
            else:
                gids = [s.capture_fwd_bwd_batch(g, psf, rc) if B > 1 else s.capture_fwd_bwd(g[0], psf, rc)
                        for g in groups]
            for i in range(5):
                s.graph_launch(gids[i % len(gids)])
            s.synchronize()
            res = {}
            for flush in (True, False):
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(steps)]
                torch.cuda.synchronize()
                for i in range(steps):
                    if flush:
                        torch.sum(flush_src, dim=0, out=flush_dst)
                    ev[i][0].record(stream)
                    s.graph_launch(gids[i % len(gids)])
                    ev[i][1].record(stream)
                torch.cuda.synchronize()
                ms = sum(a.elapsed_time(b) for a, b in ev) / steps
                res["flushed" if flush else "steady"] = {"ms_per_step": ms, "slices_per_s": B * 1000.0 / ms}
            out[f"{unit}_B{B}"] = res
            s.graph_destroy_all()
            print(unit, B, json.dumps(res), flush=True)
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
