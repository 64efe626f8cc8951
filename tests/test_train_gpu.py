"""GPU parity of the rest of the step — the photometric loss (loss.hpp:13-37,
metrics.hpp:187-225), the fused Adam update (optimize.hpp:195-221, lr_at
:71-73) and the fused training step — plus the golden fixtures the reference
produced (tests/golden/), all through the C-ABI.

Tolerances (tests/tolerances.py): images 1e-4 relative, gradients (dL/dI is
one) 1e-3 relative with the per-plane floor, scalars 1e-5 relative; Adam's
parameters / moments are fp32 on the device: 2e-6 relative + 1e-7 absolute.
"""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

from conftest import f32
from tolerances import grads_ok, image_ok

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def golden_case(gp, name):
    d = np.load(GOLD / f"{name}.npz")
    meta = json.loads(str(d["meta"]))
    pm = meta["pose"]
    pose = gp.SlicePose(np.array(pm["rotation"]).reshape(3, 3), tuple(pm["translation"]), pm["width"],
                        pm["height"], tuple(pm["pixel_spacing"]), tuple(pm["principal_point"]))
    psf = gp.PsfSpec(*meta["psf"])
    cfg = gp.RasterConfig(tau=meta["cfg"][0], tile_size=meta["cfg"][1], footprint_sigmas=meta["cfg"][2],
                          scale_modifier=meta["cfg"][3])
    gs = gp.GaussianSet(d["records"], tuple(meta["bbox"][0]), tuple(meta["bbox"][1]))
    return d, gs, pose, psf, cfg


@pytest.mark.parametrize("name", ["render_stack_k3", "render_stack_k6", "render_random_pose",
                                  "render_thick_psf"])
def test_golden_render(gp, session, name):
    """Vectors produced by the reference itself (no /root/reference needed here)."""
    d, gs, pose, psf, cfg = golden_case(gp, name)
    session.set_gaussians(gs)
    session.prepare(pose, psf, cfg)
    prep = session.prepared()
    assert np.array_equal(prep.index, d["index"]) and np.array_equal(prep.bounds, d["bounds"])
    off, ent = session.tile_lists()
    assert np.array_equal(off, d["offsets"]) and np.array_equal(ent, d["entries"])
    ok, worst = image_ok(session.rasterize(), d["image"])
    assert ok, worst
    g, stats = session.backward(d["dl_di"].astype(np.float32), stats=True)
    ok, worst = grads_ok(g, d["grads"])
    assert ok, worst
    assert np.array_equal(stats.observed, d["stat_observed"])


def test_golden_voxel(gp, session):
    d = np.load(GOLD / "voxel.npz")
    meta = json.loads(str(d["meta"]))
    cfg = gp.VoxelizerConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in meta.items()})
    session.set_gaussians(gp.GaussianSet(d["records"], (0, 0, 0), (24, 20, 16)))
    vol = session.voxelize(cfg)
    off, ent = session.voxel_tile_lists()
    assert np.array_equal(off, d["offsets"]) and np.array_equal(ent, d["entries"])
    ok, worst = image_ok(vol, d["volume"])
    assert ok, worst
    ok, worst = grads_ok(session.voxelize_backward(cfg, d["dl_dv"].astype(np.float32)), d["grads"])
    assert ok, worst


@pytest.mark.parametrize("lam", [0.0, 0.2, 1.0])
def test_loss_matches_reference(gp, lam):
    d = np.load(GOLD / "loss.npz")
    L, dl = gp.photometric_loss(d["rendered"], d["target"], lam, 0.5)
    assert L == pytest.approx(float(d[f"loss_{lam}"]), rel=1e-5)
    ok, worst = grads_ok(dl, d[f"dl_{lam}"])
    assert ok, worst


def test_loss_identical_images_is_zero(gp):
    """test_loss.cpp:20-35: L(I, I) = 0 and dL/dI = 0 (SSIM(I, I) = 1)."""
    img = np.random.default_rng(1).uniform(0, 1, (40, 52)).astype(np.float32)
    L, dl = gp.photometric_loss(img, img, 0.2, 0.5)
    assert abs(L) < 1e-6 and np.abs(dl).max() < 1e-6


def test_loss_l1_only(gp):
    """test_loss.cpp:37-50: lambda = 0 -> mean |I - T|, dL/dI = sign(I - T) / N."""
    r = np.random.default_rng(2)
    a = r.uniform(0, 1, (33, 47)).astype(np.float32)
    b = r.uniform(0, 1, (33, 47)).astype(np.float32)
    L, dl = gp.photometric_loss(a, b, 0.0, 0.5)
    assert L == pytest.approx(np.abs(a.astype(np.float64) - b).mean(), rel=1e-6)
    assert np.array_equal(dl, (np.sign(a - b) / a.size).astype(np.float32))


def test_loss_shape_mismatch(gp):
    with pytest.raises(gp.InvalidArgument):
        gp.photometric_loss(np.zeros((4, 5), np.float32), np.zeros((5, 4), np.float32), 0.2)


def adam_close(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= 2e-6 * np.abs(b) + 1e-7))


def test_adam_matches_reference(gp, session):
    d = np.load(GOLD / "adam.npz")
    bbox = (tuple(d["bbox"][0]), tuple(d["bbox"][1]))
    session.set_gaussians(gp.GaussianSet(d["records"], *bbox))
    lrs = gp.LearningRates(*d["lrs"])
    for s in range(3):
        session.set_gradients(d["grads"][s].astype(np.float32))
        session.adam_step(lrs)
        m, v, step = session.adam_state()
        assert step == s + 1
        assert adam_close(session.get_gaussians(), d[f"rec_{s}"]), f"params after step {s + 1}"
        assert adam_close(m, d[f"m_{s}"]) and adam_close(v, d[f"v_{s}"])


def test_adam_zero_grad_and_first_step(gp, session):
    """test_optim.cpp:121-146: zero gradients leave (normalized) parameters unchanged;
    the first step moves every parameter by ~lr against the gradient sign."""
    gs = gp.init_random(300, (0, 0, 0), (10, 10, 10), 1.0, 3)
    rec = f32(gs.records)
    q = rec[:, 6:10]
    rec[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    session.set_gaussians(gp.GaussianSet(f32(rec), (0, 0, 0), (10, 10, 10)))
    before = session.get_gaussians().astype(np.float64)
    lrs = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    session.set_gradients(np.zeros((300, 11), np.float32))
    session.adam_step(lrs)
    assert np.allclose(session.get_gaussians(), before, rtol=0, atol=1e-6)
    g = np.random.default_rng(4).normal(0, 1, (300, 11)).astype(np.float32)
    session.adam_reset()
    session.set_gaussians(gp.GaussianSet(f32(rec), (0, 0, 0), (10, 10, 10)))
    session.set_gradients(g)
    session.adam_step(lrs)
    delta = session.get_gaussians().astype(np.float64) - before
    want = -np.sign(g) * np.array([6e-4] * 3 + [2e-3] * 3 + [1e-3] * 4 + [0.02])
    sl = np.r_[0:6, 10]  # quaternion is renormalized after the step
    assert np.allclose(delta[:, sl], want[:, sl], rtol=1e-3, atol=1e-6)


def test_scheduled_adam_uses_lr_schedule(gp, session):
    """gpk_adam_step_scheduled: lr = lr_at(lr0, step, total) (optimize.hpp:71-73)."""
    from paper_2603_20611_b200 import _native as N
    import ctypes as C

    d = np.load(GOLD / "adam.npz")
    bbox = (tuple(d["bbox"][0]), tuple(d["bbox"][1]))
    lr0 = gp.LearningRates(*d["lrs"])
    total = 4
    with gp.Session(0) as s2:
        session.set_gaussians(gp.GaussianSet(d["records"], *bbox))
        s2.set_gaussians(gp.GaussianSet(d["records"], *bbox))
        for s in range(3):
            g = d["grads"][s].astype(np.float32)
            session.set_gradients(g)
            l = lr0.to_c()
            N.check(N.lib.gpk_adam_step_scheduled(session.handle, C.byref(l), total, None))
            s2.set_gradients(g)
            s2.adam_step(gp.LearningRates(*[gp.lr_at(x, s + 1, total) for x in d["lrs"]]))
            assert np.array_equal(session.get_gaussians(), s2.get_gaussians())


def test_train_step_equals_composition(gp, session):
    """gpk_train_step == prepare + rasterize + photometric_loss + backward +
    scheduled Adam, bitwise on the device; its image, loss and gradients match
    the reference within the north-star tolerances."""
    from paper_2603_20611_b200 import _native as N

    ref = pytest.importorskip("oracle.bindings").load("ref")
    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 1).records), lo, hi)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 5)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(7).uniform(0, 0.1, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    session.set_gaussians(gs)
    session.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    session.train_step(pose, psf, rc, 0.2, 0.5, lr0, 100)
    grads = session.get_gradients()
    loss = np.zeros(1)
    session.download(N.GPK_BUF_LOSS, loss.ctypes.data, 8)
    after = session.get_gaussians()

    # the same step, staged, on a second session
    with gp.Session(0) as s2:
        s2.set_gaussians(gs)
        s2.prepare(pose, psf, rc)
        img2 = s2.rasterize()
        L2, dl2 = s2.photometric_loss(tgt, 0.2, 0.5)
        g2 = s2.backward(dl2)
        s2.adam_step(gp.LearningRates(*[gp.lr_at(x, 1, 100) for x in (6e-4, 0.02, 2e-3, 1e-3)]))
        assert np.array_equal(grads, g2)
        assert loss[0] == L2
        assert np.array_equal(after, s2.get_gaussians())
    # against the reference
    rimg = ref.rasterize(gs.records, pose, psf, rc, (lo, hi))
    ok, worst = image_ok(img2, rimg)
    assert ok, worst
    rL, rdl = ref.loss(rimg, tgt.astype(np.float64), 0.2, 0.5)
    assert L2 == pytest.approx(rL, rel=1e-4)
    rg, _ = ref.backward(gs.records, pose, psf, rc, rdl, (lo, hi))
    ok, worst = grads_ok(grads, rg)
    assert ok, worst


def test_train_graph_replay_equals_direct(gp, session):
    from paper_2603_20611_b200 import _native as N

    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 2).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (4, 7)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(8).uniform(0, 0.1, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    with gp.Session(0) as s2:
        for s in (session, s2):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        gids = [s2.capture_train(p, psf, rc, 0.2, 0.5, lr0, 50) for p in poses]
        for it in range(4):
            session.train_step(poses[it % 2], psf, rc, 0.2, 0.5, lr0, 50)
            s2.graph_launch(gids[it % 2])
            assert np.array_equal(session.get_gaussians(), s2.get_gaussians()), it
        s2.graph_destroy_all()


def test_pipelined_train_step_bitwise_equals_plain(gp, session):
    """gpk_train_step_next (Adam fused with the next slice's cull) leaves exactly
    the parameters, moments and gradients of gpk_train_step, also when other
    calls in between force the next step to cull again, and through graphs."""
    from paper_2603_20611_b200 import _native as N

    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 4).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (3, 6, 8, 5)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(9).uniform(0, 0.1, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    with gp.Session(0) as s2:
        for s in (session, s2):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        for it in range(8):
            k, nk = it % 4, (it + 1) % 4
            session.train_step(poses[k], psf, rc, 0.2, 0.5, lr0, 40)
            s2.train_step(poses[k], psf, rc, 0.2, 0.5, lr0, 40, next_pose=poses[nk])
            if it == 3:  # anything touching the gradients in between: the next step culls again
                g = s2.get_gradients()
                s2.set_gradients(g)
                session.set_gradients(g)
            assert np.array_equal(session.get_gaussians(), s2.get_gaussians()), it
            m1, v1, st1 = session.adam_state()
            m2, v2, st2 = s2.adam_state()
            assert st1 == st2 and np.array_equal(m1, m2) and np.array_equal(v1, v2), it
        # graphs: each pose's graph culls the next one
        gids = [s2.capture_train(poses[k], psf, rc, 0.2, 0.5, lr0, 40, next_pose=poses[(k + 1) % 4])
                for k in range(4)]
        for it in range(8, 14):
            k = it % 4
            session.train_step(poses[k], psf, rc, 0.2, 0.5, lr0, 40)
            s2.graph_launch(gids[k])
            assert np.array_equal(session.get_gaussians(), s2.get_gaussians()), it
        s2.graph_launch(gids[1])  # out of order: the graph culls its own slice first
        session.train_step(poses[1], psf, rc, 0.2, 0.5, lr0, 40)
        assert np.array_equal(session.get_gaussians(), s2.get_gaussians())
        s2.graph_destroy_all()


def test_gradient_layouts_interleave(gp, session):
    """The dense gradient planes stay exact across mixed calls: a dense backward
    after training steps (plain and pipelined, the latter skipping K_filter),
    training steps after a dense backward (the stale entries are cleared), and
    gpk_get_gradients after a plain step equals the staged composition's."""
    from paper_2603_20611_b200 import _native as N

    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 5).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (2, 9, 5)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(11).uniform(0, 0.1, (48, 64)).astype(np.float32)
    dl = np.random.default_rng(12).normal(0, 1e-3, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)

    def fresh_backward(params, pose):
        with gp.Session(0) as f:
            f.set_gaussians(gp.GaussianSet(params.astype(np.float64), lo, hi))
            f.prepare(pose, psf, rc)
            return f.backward(dl)

    session.set_gaussians(gs)
    session.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    session.prepare(poses[0], psf, rc)
    session.backward(dl)  # dense gradients of slice 0 pending a clear
    session.train_step(poses[1], psf, rc, 0.2, 0.5, lr0, 40, next_pose=poses[2])
    session.train_step(poses[2], psf, rc, 0.2, 0.5, lr0, 40)  # prefiltered: no K_filter
    # the staged step on the same parameters gives the same dense gradient
    before = session.get_gaussians()
    session.prepare(poses[0], psf, rc)
    g = session.backward(dl)
    assert np.array_equal(g, fresh_backward(before, poses[0]))
    # gradients read after a step equal the staged composition's
    with gp.Session(0) as s2:
        s2.set_gaussians(gp.GaussianSet(before.astype(np.float64), lo, hi))
        s2.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        s2.adam_reset()
        session.adam_reset()
        session.train_step(poses[1], psf, rc, 0.2, 0.5, lr0, 40)
        s2.prepare(poses[1], psf, rc)
        s2.rasterize()
        _, dl2 = s2.photometric_loss(tgt, 0.2, 0.5)
        assert np.array_equal(session.get_gradients(), s2.backward(dl2))


def test_target_upload_overlaps_but_is_ordered(gp, session):
    """gpk_upload(GPK_BUF_TARGET) runs on the session's copy stream and overlaps
    the next step's prepare + forward; the loss (direct or in a replayed graph)
    must still see the new target: both equal a session that synchronizes after
    every upload. A large slice (16 MB target) and a small set make the copy
    outlast the kernels before the loss."""
    from paper_2603_20611_b200 import _native as N

    dims = (2048, 2048, 8)
    lo, hi = (-0.5, -0.5, -0.5), (2047.5, 2047.5, 7.5)
    gs = gp.GaussianSet(f32(gp.init_random(2000, lo, hi, 1.5, 6).records), lo, hi)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 3)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    rng = np.random.default_rng(13)
    targets = [rng.uniform(0, 0.1 * (k + 1), (2048, 2048)).astype(np.float32) for k in range(3)]
    with gp.Session(0) as s2, gp.Session(0) as s3:
        for s in (session, s2, s3):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, targets[0].ctypes.data, targets[0].nbytes)
        gid = s2.capture_train(pose, psf, rc, 0.2, 0.5, lr0, 20)
        for k in range(3):
            for s in (session, s2, s3):
                s.upload(N.GPK_BUF_TARGET, targets[k].ctypes.data, targets[k].nbytes)
            s3.synchronize()
            session.train_step(pose, psf, rc, 0.2, 0.5, lr0, 20)
            s2.graph_launch(gid)
            s3.train_step(pose, psf, rc, 0.2, 0.5, lr0, 20)
            loss = []
            for s in (session, s2, s3):
                v = np.zeros(1)
                s.download(N.GPK_BUF_LOSS, v.ctypes.data, 8)
                s.synchronize()
                loss.append(v[0])
            assert loss[0] == loss[2] and loss[1] == loss[2], (k, loss)
            ref = s3.get_gaussians()
            assert np.array_equal(session.get_gaussians(), ref), k
            assert np.array_equal(s2.get_gaussians(), ref), k
        s2.graph_destroy_all()


def test_target_slots_alternating_equal_single_slot(gp, session):
    """gpk_set_target_slot: a session that alternates two target slots step by
    step (graphs captured per slot, uploads into the slot of the step they
    feed, queued without waiting) trains exactly like a session that
    synchronizes after every upload into the one default slot."""
    from paper_2603_20611_b200 import _native as N

    dims = (256, 192, 8)
    lo, hi = (-0.5, -0.5, -0.5), (255.5, 191.5, 7.5)
    gs = gp.GaussianSet(f32(gp.init_random(20000, lo, hi, 1.5, 16).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (2, 5)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    rng = np.random.default_rng(17)
    targets = [rng.uniform(0, 0.1 * (k + 1), (192, 256)).astype(np.float32) for k in range(6)]
    with gp.Session(0) as ref:
        for s in (session, ref):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, targets[0].ctypes.data, targets[0].nbytes)
        ref.synchronize()
        session.synchronize()
        gids = []
        for k in range(2):  # graph k reads slot k
            session.set_target_slot(k)
            session.upload(N.GPK_BUF_TARGET, targets[0].ctypes.data, targets[0].nbytes)
            gids.append(session.capture_train(poses[k], psf, rc, 0.2, 0.5, lr0, 20))
        losses = []
        for i, t in enumerate(targets):
            session.set_target_slot(i % 2)
            session.upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
            session.graph_launch(gids[i % 2])
            ref.upload(N.GPK_BUF_TARGET, t.ctypes.data, t.nbytes)
            ref.synchronize()
            ref.train_step(poses[i % 2], psf, rc, 0.2, 0.5, lr0, 20)
            v = np.zeros(1)
            ref.download(N.GPK_BUF_LOSS, v.ctypes.data, 8)
            ref.synchronize()
            losses.append(v[0])
        v = np.zeros(1)
        session.download(N.GPK_BUF_LOSS, v.ctypes.data, 8)
        session.synchronize()
        assert v[0] == losses[-1]
        assert np.array_equal(session.get_gaussians(), ref.get_gaussians())
        m1, v1, s1 = session.adam_state()
        m2, v2, s2 = ref.adam_state()
        assert s1 == s2 == len(targets) and np.array_equal(m1, m2) and np.array_equal(v1, v2)
        # downloads read the selected slot
        got = np.zeros_like(targets[0])
        session.set_target_slot(0)
        session.download(N.GPK_BUF_TARGET, got.ctypes.data, got.nbytes)
        session.synchronize()
        assert np.array_equal(got, targets[4])
        with pytest.raises(gp.InvalidArgument):
            session.set_target_slot(2)
        session.graph_destroy_all()
