"""The union-compacted data-parallel step (gpk_train_step_dp, csrc/dp.cu) with
two ranks simulated on one GPU: two sessions (the replicas) run the render
phase for their own pose of the step, the host sums their union rows (what the
NCCL all-reduce does), and both run the update phase. Two-rank sums are
order-free in fp32 (a + b = b + a), so both replicas must equal, bitwise, the
batched step that renders the same two slices on one session and sums their
gradients (gpk_train_step_batch) — parameters, moments and the gradient."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu

DIMS = (96, 80, 24)
LR0 = (6e-4, 0.02, 2e-3, 1e-3)


def test_two_ranks_simulated_equal_the_batched_step(gp):
    from paper_2603_20611_b200 import _native as N

    lo, hi = (-0.5,) * 3, (95.5, 79.5, 23.5)
    gs = gp.GaussianSet(f32(gp.init_random(6000, lo, hi, 1.5, 31).records), lo, hi)
    psf, rc, lr0 = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    rng = np.random.default_rng(32)
    tgts = [rng.uniform(0, 0.1, (80, 96)).astype(np.float32) for _ in range(2)]
    schedule = [[gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in ks]
                for ks in ((7, 12), (9, 15), (11, 4))]
    with gp.Session(0) as r0, gp.Session(0) as r1, gp.Session(0) as bat:
        ranks = (r0, r1)
        for s in (r0, r1, bat):
            s.set_gaussians(gs)
        for r, s in enumerate(ranks):
            s.upload(N.GPK_BUF_TARGET, tgts[r].ctypes.data, tgts[r].nbytes)
        for k in range(2):
            bat.context(k).upload(N.GPK_BUF_TARGET, tgts[k].ctypes.data, tgts[k].nbytes)
        for step, poses in enumerate(schedule):
            for r, s in enumerate(ranks):
                s.train_step_dp(2, r, poses, psf, rc, 0.2, 0.5, lr0, 50, phases=N.GPK_DP_RENDER)
            M0, cap0 = r0.dp_union_rows()
            M1, cap1 = r1.dp_union_rows()
            assert (M0, cap0) == (M1, cap1) and 0 < M0 <= cap0, "every rank numbers the same union"
            # the exchange: rows summed on the host, in place on both ranks
            _, nbytes = r0.device_buffer(N.GPK_BUF_UNION_ROWS)
            rows = [np.zeros(nbytes // 4, np.float32) for _ in ranks]
            for s, buf in zip(ranks, rows):
                s.download(N.GPK_BUF_UNION_ROWS, buf.ctypes.data, nbytes)
                s.synchronize()
            total = (rows[0] + rows[1]).astype(np.float32)
            for s in ranks:
                s.upload(N.GPK_BUF_UNION_ROWS, total.ctypes.data, nbytes)
                s.train_step_dp(2, ranks.index(s), poses, psf, rc, 0.2, 0.5, lr0, 50, phases=N.GPK_DP_UPDATE)
            bat.train_step_batch(poses, psf, rc, 0.2, 0.5, lr0, 50)
            want = bat.get_gaussians()
            for s in ranks:
                assert np.array_equal(s.get_gaussians(), want), step
                assert np.array_equal(s.get_gradients(), bat.get_gradients()), step
            m0, v0, st0 = r0.adam_state()
            mb, vb, stb = bat.adam_state()
            assert st0 == stb == step + 1
            assert np.array_equal(m0, mb) and np.array_equal(v0, vb)


def test_dp_phase_errors(gp, session):
    lo, hi = (-0.5,) * 3, (95.5, 79.5, 23.5)
    session.set_gaussians(gp.GaussianSet(f32(gp.init_random(500, lo, hi, 1.5, 1).records), lo, hi))
    poses = [gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in (3, 4)]
    lr0 = gp.LearningRates(*LR0)
    with pytest.raises(gp.StateError):  # no communicator for the exchange
        session.train_step_dp(2, 0, poses, gp.PsfSpec(), gp.RasterConfig(), 0.2, 0.5, lr0, 10)
    with pytest.raises(gp.InvalidArgument):
        session.train_step_dp(2, 2, poses, gp.PsfSpec(), gp.RasterConfig(), 0.2, 0.5, lr0, 10, phases=1)


def test_union_holds_every_rank_survivor_at_scale(gp):
    """The union of W = 8 poses (consecutive mid-stack slices, the shape a
    data-parallel step gives every rank) is computed by one interval test per
    Gaussian (cull.cu union_candidate), not per pose. It must contain every
    rank's survivors, or that rank's gradient would silently lose rows: for
    each simulated rank, the gradient its render phase writes into the union
    rows (read back densely) equals, bitwise, the plain single-session
    gradient of the same slice (same loss, same kernels)."""
    from paper_2603_20611_b200 import _native as N

    dims = (192, 160, 64)
    lo, hi = (-0.5,) * 3, tuple(d - 0.5 for d in dims)
    gs = gp.GaussianSet(f32(gp.init_random(120000, lo, hi, 1.5, 41).records), lo, hi)
    psf, rc, lr0 = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    rng = np.random.default_rng(42)
    tgt = rng.uniform(0, 0.1, (dims[1], dims[0])).astype(np.float32)
    W = 8
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in range(28, 28 + W)]
    with gp.Session(0) as rank, gp.Session(0) as plain:
        for s in (rank, plain):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        union_rows = None
        for r in (0, 3, 7):
            rank.train_step_dp(W, r, poses, psf, rc, 0.2, 0.5, lr0, 50, phases=N.GPK_DP_RENDER)
            got = rank.get_gradients()
            rows, cap = rank.dp_union_rows()
            union_rows = union_rows or rows
            assert rows == union_rows and rows <= cap, "every rank numbers the same union"
            plain.prepare(poses[r], psf, rc)
            plain.rasterize()
            _, dl = plain.photometric_loss(tgt, 0.2, 0.5)
            want = plain.backward(dl)
            nz = np.count_nonzero(np.any(want != 0, axis=1))
            assert nz > 1000, nz  # the slice has survivors
            assert np.array_equal(got, want), r
