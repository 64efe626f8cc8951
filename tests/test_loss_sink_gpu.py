"""gpk_set_loss_sink: the loss kernel writes each loss into page-locked host
memory itself (the end-to-end loop's device-to-host result without a copy).
The value must be the device loss (GPK_BUF_LOSS) of the same step, bitwise,
for direct steps, graphs and the slice contexts of a batched step."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import f32

pytestmark = pytest.mark.gpu

DIMS = (96, 80, 24)
LR0 = (6e-4, 0.02, 2e-3, 1e-3)


def setup(gp, s, nctx=1):
    from paper_2603_20611_b200 import _native as N

    lo, hi = (-0.5, -0.5, -0.5), (DIMS[0] - 0.5, DIMS[1] - 0.5, DIMS[2] - 0.5)
    s.set_gaussians(gp.GaussianSet(f32(gp.init_random(6000, lo, hi, 1.5, 21).records), lo, hi))
    rng = np.random.default_rng(4)
    for k in range(nctx):
        t = rng.uniform(0, 0.1, (DIMS[1], DIMS[0])).astype(np.float32)
        s.context(k).upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
    s.synchronize()


def device_loss(s):
    from paper_2603_20611_b200 import _native as N

    L = np.zeros(1)
    s.download(N.GPK_BUF_LOSS, L.ctypes.data, 8)
    s.synchronize()
    return L[0]


def test_loss_sink_direct_and_graph(gp, session):
    setup(gp, session)
    sink = torch.zeros(1, dtype=torch.float64).pin_memory()
    session.set_loss_sink(sink.data_ptr())
    psf, rc, lr = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    poses = [gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in (4, 11, 17)]
    for p in poses:
        session.train_step(p, psf, rc, 0.2, 0.5, lr, 100)
        session.synchronize()
        assert sink[0].item() == device_loss(session) and sink[0].item() > 0
    gids = [session.capture_train(p, psf, rc, 0.2, 0.5, lr, 100) for p in poses]
    for g in gids:
        sink.zero_()
        session.graph_launch(g)
        session.synchronize()
        assert sink[0].item() == device_loss(session) and sink[0].item() > 0
    # lambda = 0: the L1-only loss kernel
    session.set_loss_sink(None)
    sink.zero_()
    session.train_step(poses[0], psf, rc, 0.0, 0.5, lr, 100)
    session.synchronize()
    assert sink[0].item() == 0.0
    session.graph_destroy_all()


def test_loss_sink_batched_contexts(gp, session):
    setup(gp, session, nctx=3)
    sink = torch.zeros(3, dtype=torch.float64).pin_memory()
    for k in range(3):
        session.context(k).set_loss_sink(sink.data_ptr() + 8 * k)
    psf, rc, lr = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    poses = [gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in (5, 12, 19)]
    session.train_step_batch(poses, psf, rc, 0.2, 0.5, lr, 100)
    session.synchronize()
    for k in range(3):
        assert sink[k].item() == device_loss(session.context(k)) and sink[k].item() > 0


def test_loss_sink_rejects_pageable_memory(gp, session):
    setup(gp, session)
    buf = np.zeros(1)
    with pytest.raises(gp.InvalidArgument):
        session.set_loss_sink(buf.ctypes.data)


def test_queued_uploads_keep_step_order(gp):
    """The next target's upload starts once the current step's last target
    reader (the raster backward) is queued before it, not after the whole
    step: with every step queued ahead (the device held by a sleep) and a
    different target per step, the losses and the final state equal a run that
    waits for each step."""
    from paper_2603_20611_b200 import _native as N

    psf, rc, lr = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    ks = [3, 9, 14, 20, 6, 11, 17, 2, 8, 15, 21, 5]
    poses = [gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in ks]
    rng = np.random.default_rng(9)
    tgts = [torch.from_numpy(rng.uniform(0, 0.1, (DIMS[1], DIMS[0])).astype(np.float32)).pin_memory()
            for _ in ks]
    nb = DIMS[0] * DIMS[1] * 4
    out = []
    for queued in (False, True):
        stream = torch.cuda.Stream()
        with gp.Session(0, stream=stream.cuda_stream) as s:
            setup(gp, s)
            losses = torch.zeros(len(ks), dtype=torch.float64).pin_memory()
            gids = [s.capture_train(p, psf, rc, 0.2, 0.5, lr, 100) for p in poses]
            if queued:
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(40_000_000)
            for j, g in enumerate(gids):
                s.upload(N.GPK_BUF_TARGET, tgts[j].data_ptr(), nb)
                s.graph_launch(g)
                s.download(N.GPK_BUF_LOSS, losses.data_ptr() + 8 * j, 8)
                if not queued:
                    s.synchronize()
            s.synchronize()
            out.append((losses.numpy().copy(), s.get_gaussians()))
            s.graph_destroy_all()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
