"""Minimal driver for ncu captures: C2 fwd+bwd slices through the C-ABI.

    python tests/profile_step.py [--steps N] [--config c2] [--train]
No torch, no timing: just the kernel sequence of the step (for ncu/sanitizers).
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2603_20611_b200 as gp  # noqa: E402
from paper_2603_20611_b200 import _native as N  # noqa: E402

DIMS = {"c1": ((128, 128, 32), 20000, 1.0), "c2": ((512, 512, 128), 1_000_000, 1.0),
        "c3": ((256, 256, 320), 500_000, 3.0), "c5": ((2048, 2048, 256), 8_000_000, 1.0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--train", action="store_true")
    args = ap.parse_args()
    dims, n, sz = DIMS[args.config]
    lo = (-0.5, -0.5, -0.5)
    hi = (dims[0] - 0.5, dims[1] - 0.5, dims[2] - 0.5)
    gs = gp.init_random(n, lo, hi, 1.5, 1)
    s = gp.Session(0)
    s.set_gaussians(gs)
    psf, cfg = gp.PsfSpec(sigma_z=sz), gp.RasterConfig()
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), dims[2] // 2 + i) for i in range(4)]
    s.fwd_bwd_slice(poses[0], psf, cfg)
    rng = np.random.default_rng(7)
    dl = (rng.uniform(-1, 1, (dims[1], dims[0])) / (dims[0] * dims[1])).astype(np.float32)
    s.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    tgt = rng.uniform(0, 0.1, (dims[1], dims[0])).astype(np.float32)
    s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    lr = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    for i in range(args.steps):
        if args.train:
            s.train_step(poses[i % 4], psf, cfg, 0.2, 0.5, lr, 30000)
        else:
            s.fwd_bwd_slice(poses[i % 4], psf, cfg)
    s.synchronize()
    print("ok", s.prepared_count())


if __name__ == "__main__":
    main()
