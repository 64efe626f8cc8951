"""Batched slices (gpk_slice_context, gpk_fwd_bwd_batch, gpk_train_step_batch):
B slices of one resident set rendered concurrently on slice contexts, their
gradients summed per primitive in slice order.

There is no reference function for a B-slice step (the reference does one slice
per Adam step, optimize.hpp:383-402); the contract is that a batched step equals
the composition of B single-slice steps with the gradients summed in slice
order in fp32, bitwise: images and losses per slice, the summed gradient, and
the one Adam step on it (whose single-slice form is pinned against the
reference in test_configs_gpu.py / test_train_gpu.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu

DIMS = (96, 80, 24)
LR0 = (6e-4, 0.02, 2e-3, 1e-3)


def scene(gp, n=5000, seed=3):
    lo, hi = (-0.5, -0.5, -0.5), (DIMS[0] - 0.5, DIMS[1] - 0.5, DIMS[2] - 0.5)
    return gp.GaussianSet(f32(gp.init_random(n, lo, hi, 1.5, seed).records), lo, hi)


def poses(gp, ks):
    return [gp.slice_pose_for_index(DIMS, (1, 1, 1), (0, 0, 0), k) for k in ks]


def host_sum(gs_list):
    acc = gs_list[0].astype(np.float32).copy()
    for g in gs_list[1:]:
        acc = (acc + g.astype(np.float32)).astype(np.float32)
    return acc


def test_fwd_bwd_batch_equals_sum_of_slices(gp, session):
    from paper_2603_20611_b200 import _native as N

    gs = scene(gp)
    ps = poses(gp, (4, 9, 12, 17, 20))
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    rng = np.random.default_rng(1)
    dls = [(rng.uniform(-1, 1, (80, 96)) / 7680).astype(np.float32) for _ in ps]
    want_g, want_img = [], []
    with gp.Session(0) as s1:
        s1.set_gaussians(gs)
        for p, dl in zip(ps, dls):
            s1.prepare(p, psf, rc)
            want_img.append(s1.rasterize())
            want_g.append(s1.backward(dl))
    session.set_gaussians(gs)
    for k, dl in enumerate(dls):
        session.context(k).upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    for rep in range(2):
        session.fwd_bwd_batch(ps, psf, rc)
        assert np.array_equal(session.get_gradients(), host_sum(want_g)), rep
        for k in range(len(ps)):
            ctx = session.context(k)
            ctx.shape = (80, 96)
            img = np.zeros((80, 96), np.float32)
            ctx.download(N.GPK_BUF_IMAGE, img.ctypes.data, img.nbytes)
            ctx.synchronize()
            assert np.array_equal(img, want_img[k]), k
    # the same as a graph
    gid = session.capture_fwd_bwd_batch(ps, psf, rc)
    session.graph_launch(gid)
    assert np.array_equal(session.get_gradients(), host_sum(want_g))
    session.graph_destroy_all()


def test_train_step_batch_equals_composition(gp, session):
    """B = 3 slices, lambda 0.2: per-slice losses, the summed gradient and the
    Adam step on it equal three single-slice losses/backwards + one Adam."""
    from paper_2603_20611_b200 import _native as N

    gs = scene(gp, seed=4)
    ks = (5, 11, 18)
    ps = poses(gp, ks)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    rng = np.random.default_rng(2)
    tgts = [rng.uniform(0, 0.1, (80, 96)).astype(np.float32) for _ in ks]
    total = 100
    lr1 = gp.LearningRates(*[gp.lr_at(x, 1, total) for x in LR0])
    losses, grads = [], []
    with gp.Session(0) as s1:
        s1.set_gaussians(gs)
        for p, t in zip(ps, tgts):
            s1.prepare(p, psf, rc)
            s1.rasterize()
            L, dl = s1.photometric_loss(t, 0.2, 0.5)
            losses.append(L)
            grads.append(s1.backward(dl))
        gsum = host_sum(grads)
        s1.set_gradients(gsum)
        s1.adam_step(lr1)
        want_p = s1.get_gaussians()
        want_m, want_v, _ = s1.adam_state()
    session.set_gaussians(gs)
    for k, t in enumerate(tgts):
        session.context(k).upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
    session.train_step_batch(ps, psf, rc, 0.2, 0.5, gp.LearningRates(*LR0), total)
    session.synchronize()
    for k in range(len(ks)):
        L = np.zeros(1)
        ctx = session.context(k)
        ctx.download(N.GPK_BUF_LOSS, L.ctypes.data, 8)
        ctx.synchronize()
        assert L[0] == losses[k], k
    assert np.array_equal(session.get_gaussians(), want_p)
    m, v, step = session.adam_state()
    assert step == 1 and np.array_equal(m, want_m) and np.array_equal(v, want_v)
    assert np.array_equal(session.get_gradients(), gsum)


def test_train_batch_graph_replay_equals_direct(gp, session):
    from paper_2603_20611_b200 import _native as N

    gs = scene(gp, seed=6)
    groups = [poses(gp, (3, 8, 13, 19)), poses(gp, (6, 10, 15, 21))]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    rng = np.random.default_rng(5)
    tgts = [rng.uniform(0, 0.1, (80, 96)).astype(np.float32) for _ in range(4)]
    lr0 = gp.LearningRates(*LR0)
    with gp.Session(0) as s2:
        for s in (session, s2):
            s.set_gaussians(gs)
            for k, t in enumerate(tgts):
                s.context(k).upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
        gids = [s2.capture_train_batch(g, psf, rc, 0.2, 0.5, lr0, 50) for g in groups]
        for it in range(4):
            session.train_step_batch(groups[it % 2], psf, rc, 0.2, 0.5, lr0, 50)
            s2.graph_launch(gids[it % 2])
            assert np.array_equal(session.get_gaussians(), s2.get_gaussians()), it
        assert np.array_equal(session.get_gradients(), s2.get_gradients())
        s2.graph_destroy_all()


def test_batch_of_one_equals_train_step(gp, session):
    from paper_2603_20611_b200 import _native as N

    gs = scene(gp, seed=7)
    p = poses(gp, (12,))
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    t = np.random.default_rng(3).uniform(0, 0.1, (80, 96)).astype(np.float32)
    lr0 = gp.LearningRates(*LR0)
    with gp.Session(0) as s2:
        for s in (session, s2):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
        session.train_step_batch(p, psf, rc, 0.2, 0.5, lr0, 10)
        s2.train_step(p[0], psf, rc, 0.2, 0.5, lr0, 10)
        assert np.array_equal(session.get_gaussians(), s2.get_gaussians())
        assert np.array_equal(session.get_gradients(), s2.get_gradients())


def test_batch_errors_and_context_guards(gp, session):
    gs = scene(gp, n=500)
    session.set_gaussians(gs)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    with pytest.raises(gp.InvalidArgument):
        session.fwd_bwd_batch(poses(gp, range(9)), psf, rc)
    ctx = session.context(2)
    with pytest.raises(gp.StateError):
        ctx.set_gaussians(gs)
    with pytest.raises(gp.StateError):
        ctx.adam_step(gp.LearningRates(*LR0))
    with pytest.raises(gp.StateError):
        ctx.train_step_batch(poses(gp, (1, 2)), psf, rc, 0.2, 0.5, gp.LearningRates(*LR0), 10)
    # per-slice calls work on a context and see the session's set
    ctx.prepare(poses(gp, (7,))[0], psf, rc)
    session.prepare(poses(gp, (7,))[0], psf, rc)
    assert ctx.prepared_count() == session.prepared_count()
