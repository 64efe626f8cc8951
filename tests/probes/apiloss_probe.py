"""ncu driver: the stand-alone photometric_loss (k_ssim_fwd + k_ssim_bwd) on a 2048^2 render."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_20611_b200 as gp  # noqa: E402

dims = (2048, 2048, 16)
lo, hi = (-0.5,) * 3, tuple(d - 0.5 for d in dims)
gs = gp.GaussianSet(gp.init_random(400_000, lo, hi, 1.5, 3).records.astype(np.float32).astype(np.float64), lo, hi)
s = gp.Session(0)
s.set_gaussians(gs)
s.prepare(gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 8), gp.PsfSpec(), gp.RasterConfig())
s.rasterize()
tgt = np.random.default_rng(1).uniform(0, 0.1, (2048, 2048)).astype(np.float32)
for _ in range(4):
    s.photometric_loss(tgt, 0.2, 0.5)
s.synchronize()
print("ok")
