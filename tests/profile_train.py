"""ncu driver for the training step (C2): a few steps of gpk_train_step_next
(argv[2] == "plain": gpk_train_step, Adam as its own kernel) through the
C-ABI, no timing."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2603_20611_b200 as gp  # noqa: E402
from paper_2603_20611_b200 import _native as N  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    pipelined = not (len(sys.argv) > 2 and sys.argv[2] == "plain")
    big = len(sys.argv) > 3 and sys.argv[3] == "c5"  # 2048^2 x 256, 8M Gaussians
    dims = (2048, 2048, 256) if big else (512, 512, 128)
    lo, hi = (-0.5, -0.5, -0.5), tuple(d - 0.5 for d in dims)
    gs = gp.init_random(8_000_000 if big else 1_000_000, lo, hi, 1.5, 1)
    s = gp.Session(0)
    s.set_gaussians(gp.GaussianSet(gs.records.astype(np.float32).astype(np.float64), lo, hi))
    s.reserve_pairs(1 << 21 if big else 1 << 20)
    psf, cfg = gp.PsfSpec(), gp.RasterConfig()
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), dims[2] // 2 + i) for i in range(4)]
    tgt = np.random.default_rng(7).uniform(0, 0.1, (dims[1], dims[0])).astype(np.float32)
    s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    lr = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    flush = None
    mode = sys.argv[4] if len(sys.argv) > 4 else ""
    if mode in ("flush", "flushw"):  # an L2 flush between steps: read (bench) or write 256 MiB
        import torch

        src = torch.ones((256 << 20) // 4, dtype=torch.float32, device="cuda")
        dst = torch.empty((), dtype=torch.float32, device="cuda")

        def flush():
            torch.cuda.synchronize()
            if mode == "flush":
                torch.sum(src, dim=0, out=dst)
            else:
                src.fill_(float(np.random.rand()))
            torch.cuda.synchronize()
    for i in range(steps):
        if flush:
            s.synchronize()
            flush()
        s.train_step(poses[i % 4], psf, cfg, 0.2, 0.5, lr, 30000, next_pose=poses[(i + 1) % 4] if pipelined else None)
    s.synchronize()
    print("ok", s.prepared_count())


if __name__ == "__main__":
    main()
