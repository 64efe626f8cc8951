"""Adaptive density control and the fit driver on the device, against the
reference (oracle/_ref: optimize.hpp compiled unmodified).

* densify_and_prune (optimize.hpp:255-344): the same set, moments and
  accumulator in, the same generator seed: identical report, set size and
  order; parameters equal to the reference's rounded to the stored fp32
  (born primitives' positions within fp32 rounding of the fp64 arithmetic);
  moments carried bitwise, zero for the born; the step counter kept. Plus the
  reference's own cases (test_optim.cpp:153-209).
* DensifyAccum (optimize.hpp:228-249): the chain's on-device accumulation
  equals the sum of the per-backward ScreenGradStats.
* fit (optimize.hpp:360-424): progress (count, loss, monitor loss, PSNR)
  tracks the reference's run on the same volume and seed (counts exact; losses
  within FIT_LOSS_REL: the fp32 step vs the fp64 reference, compounded over
  the iterations); determinism; the reference's fit tests
  (test_optim.cpp:211-369) restated.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu

FIT_LOSS_REL = 2e-3   # per-iteration loss, fp32 device vs fp64 reference, over <= 400 iterations
FIT_PSNR_ABS = 0.05   # dB


def blob_volume(dims, center, scale, amplitude, quat=(1.0, 0.0, 0.0, 0.0)):
    """A single anisotropic Gaussian blob sampled at voxel centres, (Z, Y, X)."""
    X, Y, Z = dims
    w, x, y, z = np.asarray(quat, np.float64) / np.linalg.norm(quat)
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    cov = R @ np.diag(np.square(scale)) @ R.T
    inv = np.linalg.inv(cov)
    k, j, i = np.meshgrid(np.arange(Z), np.arange(Y), np.arange(X), indexing="ij")
    d = np.stack([i - center[0], j - center[1], k - center[2]], -1).astype(np.float64)
    q = np.einsum("...a,ab,...b->...", d, inv, d)
    return (amplitude * np.exp(-0.5 * q)).astype(np.float32)


def fit_fields(cfg):
    c = cfg.to_c()
    return {f: getattr(c, f) for f, _ in type(c)._fields_}


# ---- densify_and_prune -------------------------------------------------------
def random_densify_case(seed, n=3000, ext=64.0):
    rng = np.random.default_rng(seed)
    lo, hi = (0.0, 0.0, 0.0), (ext, ext, ext)
    rec = np.zeros((n, 11))
    rec[:, 0:3] = rng.uniform(0, ext, (n, 3))
    rec[:, 3:6] = np.log(rng.uniform(0.1, 1.0, (n, 3)))    # split threshold 0.01 * 64 = 0.64
    q = rng.normal(size=(n, 4))
    rec[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    alpha = rng.uniform(0.005, 0.3, n)                      # some below tau = 0.02
    rec[:, 10] = np.log(alpha / (1 - alpha))
    rec = f32(rec)
    m = f32(rng.normal(0, 1e-3, (n, 11)))
    v = f32(rng.uniform(0, 1e-6, (n, 11)))
    obs = rng.integers(0, 4, n).astype(np.int32)            # 0 -> pruned (never observed)
    gsum = rng.uniform(0, 1e-4, n) * obs                    # mean straddles 5e-5
    world = rng.normal(size=(n, 3)) * obs[:, None]
    world[::97] = 0.0                                       # zero direction: clone in place
    return rec, (lo, hi), m, v, gsum, obs, world


def run_device_densify(gp, session, rec, bbox, m, v, step, gsum, obs, world, dcfg, seed):
    session.set_gaussians(gp.GaussianSet(rec, bbox[0], bbox[1]))
    session.set_adam_state(m.astype(np.float32), v.astype(np.float32), step)
    session.densify_accum_enable(True)
    session.set_densify_accum(gp.DensifyAccum(gsum, obs, world))
    rep = session.densify_and_prune(dcfg, gp.Rng(seed))
    got = session.get_gaussians().astype(np.float64)
    gm, gv, gstep = session.adam_state()
    return rep, got, gm, gv, gstep


@pytest.mark.parametrize("seed", [1, 2])
def test_densify_matches_reference(gp, ref, session, seed):
    from oracle.bindings import RefRng

    rec, bbox, m, v, gsum, obs, world = random_densify_case(seed)
    dcfg = gp.DensifyConfig()
    rep, got, gm, gv, gstep = run_device_densify(gp, session, rec, bbox, m, v, 17, gsum, obs, world, dcfg, 40 + seed)
    want, wm, wv, wrep = ref.densify_and_prune(
        rec, bbox, m, v, 17, gsum, obs, world,
        (dcfg.tau, dcfg.grad_threshold, dcfg.split_scale_fraction, dcfg.split_scale_divisor,
         dcfg.scale_modifier), RefRng(40 + seed))
    assert (rep.pruned, rep.cloned, rep.split) == wrep
    assert min(wrep) > 50, wrep  # every branch exercised
    assert got.shape == want.shape
    kept = want.shape[0] - rep.cloned - 2 * rep.split
    # kept primitives and all quaternions / alphas: bitwise copies
    assert np.array_equal(got[:kept], f32(want[:kept]))
    assert np.array_equal(got[:, 6:], f32(want[:, 6:]))
    # born positions / log-scales: fp64 arithmetic on both sides, fp32 store
    np.testing.assert_allclose(got[kept:, :6], want[kept:, :6], rtol=2e-7, atol=1e-6)
    assert np.array_equal(gm.astype(np.float64), f32(wm)) and np.array_equal(gv.astype(np.float64), f32(wv))
    assert np.all(gm[kept:] == 0) and np.all(gv[kept:] == 0)
    assert gstep == 17
    # the accumulator restarts for the new set
    acc = session.densify_accum()
    assert acc.grad_norm_sum.shape == (got.shape[0],)
    assert not acc.observations.any() and not acc.grad_norm_sum.any() and not acc.world_grad_sum.any()


def test_densify_prunes_low_alpha(gp, session, ref):
    """test_optim.cpp:153-168."""
    from oracle.bindings import RefRng

    gs = gp.init_random(10, (0, 0, 0), (8, 8, 8), 1.0, 17)
    rec = f32(gs.records)
    rec[3, 10] = math.log(0.01 / 0.99)
    rec[7, 10] = math.log(0.019 / 0.981)
    rec = f32(rec)
    z = np.zeros((10, 11))
    rep, got, gm, gv, _ = run_device_densify(gp, session, rec, ((0, 0, 0), (8, 8, 8)), z, z, 0,
                                             np.zeros(10), np.ones(10, np.int32), np.zeros((10, 3)),
                                             gp.DensifyConfig(), 1)
    assert (rep.pruned, rep.cloned, rep.split) == (2, 0, 0)
    assert got.shape[0] == 8 and gm.shape[0] == 8
    assert np.array_equal(got, np.delete(rec, [3, 7], axis=0))


def test_densify_clones_small_and_splits_large(gp, session):
    """test_optim.cpp:170-209."""
    small = [10, 10, 10, math.log(0.5), math.log(0.5), math.log(0.5), 1, 0, 0, 0, 0.0]
    large = [50, 50, 50, math.log(5.0), math.log(5.0), math.log(5.0), 1, 0, 0, 0, 0.0]
    rec = f32(np.array([small, large]))
    m = np.zeros((2, 11))
    m[0, 10] = 0.5
    rep, got, gm, gv, _ = run_device_densify(
        gp, session, rec, ((0, 0, 0), (100, 100, 100)), m, np.zeros((2, 11)), 3,
        np.array([1.0, 1.0]), np.array([1, 1], np.int32), np.array([[1.0, 0, 0], [0, 1.0, 0]]),
        gp.DensifyConfig(grad_threshold=1e-6), 23)
    assert (rep.cloned, rep.split) == (1, 1)
    assert got.shape[0] == 4 and gm.shape[0] == 4
    assert gm[0, 10] == 0.5 and gm[2, 10] == 0.0 and gm[3, 10] == 0.0
    assert got[1, 0] == pytest.approx(10.5, rel=1e-6)
    assert math.exp(got[2, 3]) == pytest.approx(5.0 / 1.6, rel=1e-6)


def test_densify_accumulates_screen_stats(gp, session):
    """DensifyAccum::add (optimize.hpp:238-245) on the device = sum of the per-backward stats."""
    dims = (48, 40, 12)
    gs = gp.init_random(4000, (-0.5, -0.5, -0.5), (47.5, 39.5, 11.5), 1.5, 3)
    session.set_gaussians(gp.GaussianSet(f32(gs.records), gs.bbox_min, gs.bbox_max))
    session.densify_accum_enable(True)
    psf, cfg = gp.PsfSpec(), gp.RasterConfig()
    rng = np.random.default_rng(0)
    norm = np.zeros(4000)
    obs = np.zeros(4000, np.int64)
    world = np.zeros((4000, 3))
    for k in (3, 4, 4, 9):
        session.prepare(gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k), psf, cfg)
        dl = (rng.uniform(-1, 1, (dims[1], dims[0])) / 1000).astype(np.float32)
        _, st = session.backward(dl, stats=True)
        norm += st.mu2d_grad_norm
        obs += st.observed
        world += st.world_pos_grad
    acc = session.densify_accum()
    assert np.array_equal(acc.observations, obs)
    assert obs.max() >= 3
    np.testing.assert_allclose(acc.grad_norm_sum, norm, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(acc.world_grad_sum, world, rtol=1e-6, atol=1e-12)


# ---- fit ---------------------------------------------------------------------
def run_fit_both(gp, ref, vol, cfg, psf=None):
    psf = psf or gp.PsfSpec()
    rows = []
    with gp.Session(0) as s:
        s.fit(vol, (1, 1, 1), (0, 0, 0), psf, cfg,
              lambda p: rows.append((p.iteration, p.loss, p.count, p.psnr2d, p.monitor_loss)))
        got = s.get_gaussians().astype(np.float64)
    want, wrows = ref.fit(vol.astype(np.float64), (1, 1, 1), (0, 0, 0), psf, fit_fields(cfg))
    return got, np.array(rows), want, wrows


def test_fit_tracks_reference_with_densification(gp, ref):
    """test_optim.cpp:279-304 config (under-covered blob), progress every 20."""
    vol = blob_volume((24, 24, 8), (12.0, 12.0, 3.0), (3.0, 3.0, 1.5), 0.9)
    cfg = gp.FitConfig(iterations=200, init_count=16, densify_start=100, densify_end=200,
                       densify_interval=100, rng_seed=11, progress_interval=20)
    got, rows, want, wrows = run_fit_both(gp, ref, vol, cfg)
    assert rows.shape == wrows.shape == (10, 5)
    assert np.array_equal(rows[:, 0], wrows[:, 0])
    assert np.array_equal(rows[:, 2], wrows[:, 2]), (rows[:, 2], wrows[:, 2])
    assert rows[-1, 2] > 16  # densification triggered (test_optim.cpp:303)
    np.testing.assert_allclose(rows[:, 1], wrows[:, 1], rtol=FIT_LOSS_REL)
    np.testing.assert_allclose(rows[:, 4], wrows[:, 4], rtol=FIT_LOSS_REL)
    np.testing.assert_allclose(rows[:, 3], wrows[:, 3], atol=FIT_PSNR_ABS)
    assert got.shape == want.shape


def test_fit_count_never_grows_outside_window(gp, ref):
    """test_optim.cpp:306-332, against the reference's own trajectory."""
    vol = blob_volume((16, 16, 16), (8.0, 8.0, 8.0), (2.5, 2.5, 2.5), 0.8)
    cfg = gp.FitConfig(iterations=400, init_count=32, densify_start=100, densify_end=200,
                       rng_seed=13, progress_interval=10)
    got, rows, want, wrows = run_fit_both(gp, ref, vol, cfg)
    for a, b in zip(rows[:-1], rows[1:]):
        if a[0] >= 200:
            assert b[2] <= a[2]
    assert np.array_equal(rows[:, 2], wrows[:, 2])
    np.testing.assert_allclose(rows[:, 1], wrows[:, 1], rtol=FIT_LOSS_REL)


def test_fit_deterministic_for_fixed_seed(gp):
    """test_optim.cpp:334-369: bitwise on the device."""
    vol = blob_volume((16, 16, 16), (8.0, 8.0, 8.0), (2.0, 2.0, 2.0), 0.7)
    cfg = gp.FitConfig(iterations=300, init_count=48, rng_seed=21, progress_interval=300)
    out = []
    for seed in (21, 21, 22):
        cfg.rng_seed = seed
        losses = []
        gs = gp.fit(vol, (1, 1, 1), (0, 0, 0), gp.PsfSpec(), cfg, lambda p: losses.append(p.loss))
        out.append((gs.records, losses[-1]))
    assert out[0][0].shape == out[1][0].shape and np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    assert out[2][0].shape != out[0][0].shape or out[2][1] != out[0][1]


def test_fit_zero_volume_prunes_to_near_empty(gp):
    """test_optim.cpp:211-229."""
    vol = np.zeros((16, 16, 16), np.float32)
    cfg = gp.FitConfig(iterations=2000, init_count=64, rng_seed=3, progress_interval=2000)
    counts = []
    gs = gp.fit(vol, (1, 1, 1), (0, 0, 0), gp.PsfSpec(), cfg, lambda p: counts.append(p.count))
    assert gs.size() == counts[-1]
    assert gs.size() <= 64 // 5
    if gs.size():
        img = gp.rasterize_slice(gs, gp.slice_pose_for_index((16, 16, 16), (1, 1, 1), (0, 0, 0), 8),
                                 gp.PsfSpec(), gp.RasterConfig())
        assert np.all(img < 0.02)


def test_fit_graph_replay_equals_direct_steps(gp, monkeypatch):
    """After the densify window gpk_fit replays one CUDA graph per slice; the
    result is bitwise that of direct launches (GPK_FIT_NO_GRAPHS=1)."""
    vol = blob_volume((20, 16, 12), (9.0, 8.0, 6.0), (2.5, 2.0, 2.0), 0.8)
    cfg = gp.FitConfig(iterations=300, init_count=40, densify_start=50, densify_end=100,
                       densify_interval=50, rng_seed=4, progress_interval=50)
    runs = []
    for direct in (False, True):
        if direct:
            monkeypatch.setenv("GPK_FIT_NO_GRAPHS", "1")
        rows = []
        gs = gp.fit(vol, (1, 1, 1), (0, 0, 0), gp.PsfSpec(), cfg,
                    lambda p: rows.append((p.iteration, p.loss, p.count, p.psnr2d, p.monitor_loss)))
        runs.append((gs.records, rows))
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])
