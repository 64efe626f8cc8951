"""Probe (not a test): U2 step time on a uniform vs a spatially ordered
(Morton-sorted, what gpk_decode_streams loads) vs a clustered 1M set at C2 —
the per-tile list build must not fall off a cliff when one K_decide group's
survivors crowd into one tile. CUDA graphs, events on the session stream."""
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

    cfg = bench.CONFIGS["c2"]
    base = bench.make_records(cfg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s = gp.Session(0, stream=stream.cuda_stream)
    s.set_gaussians(base)
    perm = s.morton_sort(10)
    rec = base.records
    # clustered: the 1M Gaussians squeezed into 64 blobs of radius ~12 px
    rng = np.random.default_rng(3)
    centres = rng.uniform([40, 40, 8], [472, 472, 120], (64, 3))
    clus = rec.copy()
    which = rng.integers(0, 64, rec.shape[0])
    clus[:, 0:3] = centres[which] + rng.normal(0, 6.0, (rec.shape[0], 3))
    clus[:, 0:3] = np.clip(clus[:, 0:3], -0.5, [511.5, 511.5, 127.5])
    clus[:, 10] = np.log(0.02 / 0.98)  # faint: survivors stay a few per pixel
    sets = {"uniform": rec, "morton": rec[perm], "clustered": clus.astype(np.float32).astype(np.float64)}
    psf, rc, lr0 = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*bench.LR0)
    poses = [gp.slice_pose_for_index(cfg["dims"], (1, 1, 1), (0, 0, 0), k) for k in bench.slice_indices(128)]
    tgt = bench.synthetic_target(cfg)
    out = {}
    for name, r in sets.items():
        s.graph_destroy_all()
        s.set_gaussians(gp.GaussianSet(r, base.bbox_min, base.bbox_max))
        s.reserve_pairs(1 << 22)
        s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        for p in poses:
            s.train_step(p, psf, rc, 0.2, 0.5, lr0, 30000)
        s.synchronize()
        st = [s.prepared_count()]
        gids = [s.capture_train(p, psf, rc, 0.2, 0.5, lr0, 30000) for p in poses]
        for i in range(5):
            s.graph_launch(gids[i % 16])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(64):
            s.graph_launch(gids[i % 16])
        e1.record(stream)
        torch.cuda.synchronize()
        s.prepare(poses[8], psf, rc)
        off, _ = s.tile_lists()
        per_tile = np.diff(off.astype(np.int64))
        out[name] = {"ms_per_step": e0.elapsed_time(e1) / 64, "survivors_pairs": s.prepared_count(),
                     "max_pairs_per_tile": int(per_tile.max()), "mean_pairs_per_tile": float(per_tile.mean())}
        print(name, json.dumps(out[name]), flush=True)
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
