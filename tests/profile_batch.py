"""ncu driver (not a test): C2 batched training steps (gpk_train_step_batch,
B slices on slice contexts) through the C-ABI, no timing.
Usage: python tests/profile_batch.py [steps] [B]"""
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
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dims = (512, 512, 128)
    lo, hi = (-0.5, -0.5, -0.5), tuple(d - 0.5 for d in dims)
    gs = gp.init_random(1_000_000, lo, hi, 1.5, 1)
    s = gp.Session(0)
    s.set_gaussians(gp.GaussianSet(gs.records.astype(np.float32).astype(np.float64), lo, hi))
    s.reserve_pairs(1 << 20)
    psf, cfg = gp.PsfSpec(), gp.RasterConfig()
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 56 + i) for i in range(16)]
    tgt = np.random.default_rng(7).uniform(0, 0.1, (dims[1], dims[0])).astype(np.float32)
    for k in range(B):
        s.context(k).upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    lr = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    for i in range(steps):
        g = [poses[(i * B + b) % 16] for b in range(B)]
        s.train_step_batch(g, psf, cfg, 0.2, 0.5, lr, 30000)
    s.synchronize()
    print("ok", s.prepared_count())


if __name__ == "__main__":
    main()
