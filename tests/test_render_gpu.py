"""GPU parity of the slice renderer (prepare + binning + forward + backward)
against the reference (oracle/_ref) / the C oracle, through the C-ABI.

Mirrors the reference's own pins (proj/tests/test_render.cpp, test_grad.cpp)
with the north-star tolerances (tests/tolerances.py).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import f32
from tolerances import grads_ok, image_ok

pytestmark = pytest.mark.gpu


def plain_pose(gp, w, h):
    """test_render.cpp:17-26"""
    return gp.SlicePose(np.eye(3), (0.0, 0.0, 0.0), w, h, (1.0, 1.0), (0.0, 0.0))


def stack_scene(gp, n, dims, seed=1):
    lo = (-0.5, -0.5, -0.5)
    hi = (dims[0] - 0.5, dims[1] - 0.5, dims[2] - 0.5)
    gs = gp.init_random(n, lo, hi, 1.5, seed)
    return gp.GaussianSet(f32(gs.records), lo, hi)


def run_all(gp, session, gs, pose, psf, cfg, dl):
    session.set_gaussians(gs)
    session.prepare(pose, psf, cfg)
    img = session.rasterize()
    grads, stats = session.backward(dl, stats=True)
    prep = session.prepared()
    off, ent = session.tile_lists()
    return img, grads, stats, prep, off, ent


def check_against(ck, gp, session, gs, pose, psf, cfg, dl):
    img, grads, stats, prep, off, ent = run_all(gp, session, gs, pose, psf, cfg, dl)
    bbox = (gs.bbox_min, gs.bbox_max)
    idx, bnd, _ = ck.prepare(gs.records, pose, psf, cfg, bbox)
    roff, rent = ck.tile_lists(gs.records, pose, psf, cfg, bbox)
    rimg = ck.rasterize(gs.records, pose, psf, cfg, bbox)
    rg, (rn, ro, rw) = ck.backward(gs.records, pose, psf, cfg, dl.astype(np.float64), bbox)
    assert np.array_equal(prep.index, idx), "survivor set (render.hpp:107,127)"
    assert np.array_equal(prep.bounds, bnd), "pixel bounds (render.hpp:123-126)"
    assert np.array_equal(off, roff), "tile list offsets (render.hpp:146-159)"
    assert np.array_equal(ent, rent), "tile list entries / order (render.hpp:146-159)"
    ok, worst = image_ok(img, rimg)
    assert ok, f"image beyond tolerance (worst {worst:.2f} x bound)"
    ok, worst = grads_ok(grads, rg)
    assert ok, f"gradients beyond tolerance (worst {worst:.2f} x bound)"
    assert np.array_equal(stats.observed, ro), "observed flags (backward.hpp:168-172)"
    return len(idx), len(rent)


@pytest.mark.parametrize("k", [0, 5, 16, 31])
def test_c1_slices_match_reference(gp, session, ref, k):
    dims = (128, 128, 32)
    gs = stack_scene(gp, 20000, dims)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k)
    dl = (np.random.default_rng(k).uniform(-1, 1, (128, 128)) / 128 ** 2).astype(np.float32)
    S, T = check_against(ref, gp, session, gs, pose, gp.PsfSpec(), gp.RasterConfig(), dl)
    assert S > 1000 and T > S


def test_tau0_thick_psf_matches(gp, session, ref):
    dims = (96, 80, 24)
    gs = stack_scene(gp, 6000, dims, seed=4)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 11)
    dl = (np.random.default_rng(2).uniform(-1, 1, (80, 96)) / 7680).astype(np.float32)
    check_against(ref, gp, session, gs, pose, gp.PsfSpec(sigma_z=3.0),
                  gp.RasterConfig(tau=0.0, footprint_sigmas=4.0), dl)


def test_random_poses_match(gp, session, ref):
    """The FD-suite scenes (test_grad.cpp:128-177): random rotations, tau 0, 8 sigma."""
    from oracle.bindings import RefRng

    rng = RefRng(7)
    for scene in range(12):
        pc = rng.random_pose_c(24, 24)
        pose = gp.SlicePose(np.array(list(pc.rotation)).reshape(3, 3), tuple(pc.translation), 24, 24,
                            (1.0, 1.0), tuple(pc.principal_point))
        bbox = ((-2, -2, -2), (2, 2, 2))
        count = 1 + int(rng.below(5))
        rec = np.stack([rng.random_primitive(bbox, 0.6, 1.8) for _ in range(count)])
        gs = gp.GaussianSet(f32(rec), bbox[0], bbox[1])
        dl = (np.random.default_rng(scene).uniform(-1, 1, (24, 24))).astype(np.float32)
        check_against(ref, gp, session, gs, pose, gp.PsfSpec(),
                      gp.RasterConfig(tau=0.0, footprint_sigmas=8.0), dl)


def test_unit_primitive_spot_values(gp, session):
    """test_render.cpp:245-262"""
    g = [8.0, 8.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, math.log((1 - 1e-13) / 1e-13)]
    gs = gp.GaussianSet(np.array([g]), (-100, -100, -100), (100, 100, 100))
    session.set_gaussians(gs)
    session.prepare(plain_pose(gp, 16, 16), gp.PsfSpec(sigma_z=1.0), gp.RasterConfig())
    img = session.rasterize()
    assert abs(img[8, 8] - 1.0) < 1e-6
    assert abs(img[8, 9] - math.exp(-0.5)) < 1e-6
    assert abs(img[7, 8] - math.exp(-0.5)) < 1e-6


def test_empty_set_is_black(gp, session):
    """test_render.cpp:238-243"""
    session.set_gaussians(gp.GaussianSet(np.zeros((0, 11)), (0, 0, 0), (1, 1, 1)))
    session.prepare(plain_pose(gp, 8, 8), gp.PsfSpec(), gp.RasterConfig())
    assert not session.rasterize().any()


def test_tiled_equals_naive_reference_scene(gp, session, ref):
    """test_render.cpp:286-299 scene: 60 primitives, 40x40."""
    from oracle.bindings import RefRng

    rng = RefRng(19)
    bbox = ((0, 0, -4), (40, 40, 4))
    rec = np.stack([rng.random_primitive(bbox, 0.5, 3.0) for _ in range(60)])
    gs = gp.GaussianSet(f32(rec), bbox[0], bbox[1])
    pose = plain_pose(gp, 40, 40)
    session.set_gaussians(gs)
    session.prepare(pose, gp.PsfSpec(), gp.RasterConfig())
    img = session.rasterize()
    naive = ref.rasterize(gs.records, pose, gp.PsfSpec(), gp.RasterConfig(), naive=True)
    ok, worst = image_ok(img, naive)
    assert ok, worst


def test_culled_primitive_gets_exact_zero_gradient(gp, session):
    """test_grad.cpp:179-205"""
    vis = [8.0, 8.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, math.log(0.6 / 0.4)]
    cul = list(vis)
    cul[2] = 9.5
    gs = gp.GaussianSet(np.array([vis, cul]), (0, 0, -10), (16, 16, 10))
    session.set_gaussians(gs)
    session.prepare(plain_pose(gp, 16, 16), gp.PsfSpec(sigma_z=1.0), gp.RasterConfig())
    grads, stats = session.backward(np.ones((16, 16), np.float32), stats=True)
    assert np.linalg.norm(grads[0, :3]) > 0
    assert stats.observed[0] == 1 and stats.observed[1] == 0
    assert not grads[1].any()


def test_center_pixel_alpha_gradient(gp, session):
    """test_grad.cpp:102-126: d alpha_raw = alpha (1 - alpha) at the centre pixel."""
    g = [8.0, 8.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, math.log(0.6 / 0.4)]
    session.set_gaussians(gp.GaussianSet(np.array([g]), (-100,) * 3, (100,) * 3))
    session.prepare(plain_pose(gp, 16, 16), gp.PsfSpec(sigma_z=1.0), gp.RasterConfig(tau=0.0))
    dl = np.zeros((16, 16), np.float32)
    dl[8, 8] = 1.0
    grads = session.backward(dl)
    assert abs(grads[0, 10] - 0.6 * 0.4) < 1e-6


def test_zero_upstream_gives_zero_gradients(gp, session, ref):
    """test_grad.cpp:89-100"""
    from oracle.bindings import RefRng

    rng = RefRng(3)
    bbox = ((4, 4, -2), (20, 20, 2))
    rec = np.stack([rng.random_primitive(bbox) for _ in range(3)])
    session.set_gaussians(gp.GaussianSet(f32(rec), *bbox))
    session.prepare(plain_pose(gp, 24, 24), gp.PsfSpec(), gp.RasterConfig())
    assert not session.backward(np.zeros((24, 24), np.float32)).any()


def test_backward_error_paths(gp, session):
    """test_grad.cpp:257-281: shape mismatch and a NaN upstream gradient."""
    g = [4.0, 4.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0]
    session.set_gaussians(gp.GaussianSet(np.array([g]), (0, 0, -1), (8, 8, 1)))
    session.prepare(plain_pose(gp, 8, 8), gp.PsfSpec(), gp.RasterConfig(tau=0.0))
    with pytest.raises(gp.InvalidArgument):
        session.backward(np.zeros((4, 4), np.float32))
    dl = np.zeros((8, 8), np.float32)
    dl[4, 4] = np.nan
    with pytest.raises(gp.NumericFailure) as ei:
        session.backward(dl)
    assert ei.value.index == 0


def test_invalid_psf_and_quaternion(gp, session):
    g = [4.0, 4.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]  # zero quaternion
    session.set_gaussians(gp.GaussianSet(np.array([g]), (0, 0, -1), (8, 8, 1)))
    with pytest.raises(gp.InvalidArgument):
        session.prepare(plain_pose(gp, 8, 8), gp.PsfSpec(sigma_z=0.0), gp.RasterConfig())
    session.prepare(plain_pose(gp, 8, 8), gp.PsfSpec(), gp.RasterConfig())
    with pytest.raises(gp.InvalidArgument):
        session.rasterize()


def test_backward_bitwise_deterministic(gp, session):
    """test_grad.cpp:232-255 (thread-count determinism -> run-to-run on the GPU)."""
    dims = (128, 128, 32)
    gs = stack_scene(gp, 20000, dims, seed=17)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 12)
    dl = (np.random.default_rng(9).uniform(-1, 1, (128, 128))).astype(np.float32)
    session.set_gaussians(gs)
    outs = []
    for _ in range(3):
        session.prepare(pose, gp.PsfSpec(), gp.RasterConfig())
        outs.append((session.rasterize(), session.backward(dl)))
    for img, g in outs[1:]:
        assert np.array_equal(img, outs[0][0]) and np.array_equal(g, outs[0][1])


def test_fused_u1_equals_staged(gp, session):
    dims = (128, 128, 32)
    gs = stack_scene(gp, 20000, dims, seed=2)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 20)
    dl = (np.random.default_rng(1).uniform(-1, 1, (128, 128)) / 16384).astype(np.float32)
    session.set_gaussians(gs)
    session.prepare(pose, gp.PsfSpec(), gp.RasterConfig())
    img = session.rasterize()
    g = session.backward(dl)
    from paper_2603_20611_b200 import _native as N

    session.fwd_bwd_slice(pose, gp.PsfSpec(), gp.RasterConfig())
    session.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    session.fwd_bwd_slice(pose, gp.PsfSpec(), gp.RasterConfig())
    assert np.array_equal(session.get_gradients(), g)
    assert np.array_equal(session.rasterize(), img)


def test_graph_replay_equals_direct(gp, session):
    """A captured CUDA graph of the U1 step reproduces the direct submission bitwise."""
    from paper_2603_20611_b200 import _native as N

    dims = (128, 128, 32)
    gs = stack_scene(gp, 20000, dims, seed=5)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (9, 10)]
    dl = (np.random.default_rng(4).uniform(-1, 1, (128, 128)) / 16384).astype(np.float32)
    session.set_gaussians(gs)
    session.fwd_bwd_slice(poses[0], gp.PsfSpec(), gp.RasterConfig())
    session.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    direct = []
    for p in poses:
        session.fwd_bwd_slice(p, gp.PsfSpec(), gp.RasterConfig())
        direct.append((session.rasterize(), session.get_gradients()))
    gids = [session.capture_fwd_bwd(p, gp.PsfSpec(), gp.RasterConfig()) for p in poses]
    for _ in range(2):
        for gid, (img, g) in zip(gids, direct):
            session.graph_launch(gid)
            assert np.array_equal(session.get_gradients(), g)
            assert np.array_equal(session.rasterize(), img)
    session.graph_destroy_all()


def test_dense_gradients_after_sparse_clear(gp, session):
    """The gradient planes are cleared sparsely (previous survivors only) between
    fused steps: every step must still leave the exact dense gradient, whatever
    wrote the planes before (another slice, set_gradients, voxelize_backward,
    a graph replay)."""
    from paper_2603_20611_b200 import _native as N

    dims = (128, 128, 32)
    gs = stack_scene(gp, 20000, dims, seed=8)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (3, 28, 15)]
    dl = (np.random.default_rng(6).uniform(-1, 1, (128, 128)) / 16384).astype(np.float32)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    # expected: staged path (dense memset + backward) on a fresh session
    want = []
    with gp.Session(0) as fresh:
        fresh.set_gaussians(gs)
        for p in poses:
            fresh.prepare(p, psf, rc)
            fresh.rasterize()
            want.append(fresh.backward(dl))
    session.set_gaussians(gs)
    session.fwd_bwd_slice(poses[0], psf, rc)
    session.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
    for k in (0, 1, 2, 0, 2, 1):
        session.fwd_bwd_slice(poses[k], psf, rc)
        assert np.array_equal(session.get_gradients(), want[k]), k
    session.set_gradients(np.full((gs.size(), 11), 7.0, np.float32))
    session.fwd_bwd_slice(poses[1], psf, rc)
    assert np.array_equal(session.get_gradients(), want[1])
    session.voxelize_backward(gp.VoxelizerConfig(dims=(32, 32, 8)), np.ones((8, 32, 32), np.float32))
    session.fwd_bwd_slice(poses[2], psf, rc)
    assert np.array_equal(session.get_gradients(), want[2])
    gids = [session.capture_fwd_bwd(p, psf, rc) for p in poses]
    for k in (2, 0, 1, 1, 0):
        session.graph_launch(gids[k])
        assert np.array_equal(session.get_gradients(), want[k]), k
    session.graph_destroy_all()


def test_c2_full_size_bitexact_binning(gp, session, ref):
    """C2 (512^2 x 128, 1M Gaussians): survivors, bounds and tile lists bit-exact;
    image and gradients within tolerance of the reference."""
    dims = (512, 512, 128)
    gs = stack_scene(gp, 1_000_000, dims)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 64)
    dl = (np.random.default_rng(7).uniform(-1, 1, (512, 512)) / 512 ** 2).astype(np.float32)
    S, T = check_against(ref, gp, session, gs, pose, gp.PsfSpec(), gp.RasterConfig(), dl)
    assert 30000 < S < 80000 and T > 2 * S
