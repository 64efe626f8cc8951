"""GPU parity of the 3-D voxelizer (voxelize / voxelize_backward,
voxelize.hpp:113-240) against the reference (oracle/_ref), through the C-ABI.

Mirrors proj/tests/test_voxelize.cpp (empty set, on-centre primitive,
additivity, monotone support, >2^31 refusal, trivial backward cases) and adds
direct comparisons with the reference: per-tile lists bit-exact, volumes and
gradients within the north-star tolerances (tests/tolerances.py).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import f32
from tolerances import grads_ok, image_ok

pytestmark = pytest.mark.gpu


def unit_cfg(gp, n, **kw):
    """test_voxelize.cpp:17-23"""
    return gp.VoxelizerConfig(dims=(n, n, n), **kw)


def random_scene(gp, n, lo, hi, scale=1.0, seed=3):
    gs = gp.init_random(n, lo, hi, scale, seed)
    return gp.GaussianSet(f32(gs.records), lo, hi)


def on_center(gp, mu, alpha, s=1.5):
    rec = np.zeros((1, 11))
    rec[0, 0:3] = mu
    rec[0, 3:6] = math.log(s)
    rec[0, 6] = 1.0
    rec[0, 10] = math.log(alpha / (1.0 - alpha))  # alpha_activation_inverse
    return gp.GaussianSet(f32(rec), (0, 0, 0), (16, 16, 16))


def check_volume(ref, session, gs, cfg):
    session.set_gaussians(gs)
    vol = session.voxelize(cfg)
    off, ent = session.voxel_tile_lists()
    rvol = ref.voxelize(gs.records, cfg)
    roff, rent = ref.voxel_tiles(gs.records, cfg)
    assert np.array_equal(off, roff), "voxel tile offsets (voxelize.hpp:86-105)"
    assert np.array_equal(ent, rent), "voxel tile entries / order (voxelize.hpp:93-103)"
    ok, worst = image_ok(vol, rvol)
    assert ok, f"volume beyond tolerance (worst {worst:.2f} x bound)"
    return vol, rvol, len(rent)


def test_empty_set_voxelizes_to_zero(gp, session):
    session.set_gaussians(gp.GaussianSet(np.zeros((0, 11)), (0, 0, 0), (8, 8, 8)))
    vol = session.voxelize(unit_cfg(gp, 8))
    assert vol.shape == (8, 8, 8) and not vol.any()


def test_isotropic_on_center_evaluates_to_alpha(gp, session):
    """test_voxelize.cpp:65-77 (fp32 device: relative 1e-6 instead of 1e-12)."""
    session.set_gaussians(on_center(gp, (5.0, 7.0, 9.0), 0.73))
    vol = session.voxelize(unit_cfg(gp, 16))
    assert vol[9, 7, 5] == pytest.approx(np.float32(0.73), rel=1e-6)


@pytest.mark.parametrize("n,count,tile", [(32, 20, (8, 8, 8)), (64, 3000, (8, 8, 8)),
                                          (48, 2000, (4, 8, 16)), (40, 500, (5, 3, 7))])
def test_matches_reference(gp, session, ref, n, count, tile):
    gs = random_scene(gp, count, (4, 4, 4), (n - 4, n - 4, n - 4), scale=1.2, seed=count)
    _, _, pairs = check_volume(ref, session, gs, unit_cfg(gp, n, tile_dims=tile))
    assert pairs >= count // 2


def test_anisotropic_grid_matches_reference(gp, session, ref):
    """Non-unit spacing, shifted origin, non-cubic grid, tiles larger than one axis."""
    cfg = gp.VoxelizerConfig(dims=(72, 40, 24), spacing=(0.5, 0.75, 1.25), origin=(-3.0, 1.0, 2.5),
                             tile_dims=(8, 8, 32), support_sigmas=2.5, scale_modifier=1.3)
    lo = (-3.0, 1.0, 2.5)
    hi = (-3.0 + 36.0, 1.0 + 30.0, 2.5 + 30.0)
    gs = random_scene(gp, 4000, lo, hi, scale=0.8, seed=17)
    check_volume(ref, session, gs, cfg)


def test_additivity_over_disjoint_subsets(gp, session):
    """test_voxelize.cpp:113-127 (fp32 accumulation: 1e-5 instead of 1e-9)."""
    gs = random_scene(gp, 8, (2, 2, 2), (14, 14, 14), seed=5)
    cfg = unit_cfg(gp, 16)
    a = gp.GaussianSet(gs.records[1::2], gs.bbox_min, gs.bbox_max)
    b = gp.GaussianSet(gs.records[0::2], gs.bbox_min, gs.bbox_max)
    session.set_gaussians(a)
    va = session.voxelize(cfg)
    session.set_gaussians(b)
    vb = session.voxelize(cfg)
    session.set_gaussians(gs)
    vall = session.voxelize(cfg)
    assert np.abs(vall.astype(np.float64) - va - vb).max() <= 1e-5


def test_larger_support_never_decreases(gp, session):
    """test_voxelize.cpp:129-138: holds exactly (same per-primitive values, extra
    non-negative terms inserted into a monotone fp32 sum)."""
    gs = random_scene(gp, 6, (2, 2, 2), (14, 14, 14), seed=7)
    session.set_gaussians(gs)
    lo = session.voxelize(unit_cfg(gp, 16, support_sigmas=2.0))
    hi = session.voxelize(unit_cfg(gp, 16, support_sigmas=4.0))
    assert (hi >= lo).all()


def test_refuses_oversized_grids(gp, session):
    """test_voxelize.cpp:140-147"""
    session.set_gaussians(gp.GaussianSet(np.zeros((0, 11)), (0, 0, 0), (1, 1, 1)))
    with pytest.raises(gp.InvalidArgument):
        session.voxelize(gp.VoxelizerConfig(dims=(2048, 2048, 1024)))


@pytest.mark.parametrize("bad", [dict(dims=(0, 4, 4)), dict(dims=(4, 4, 4), tile_dims=(8, 0, 8)),
                                 dict(dims=(4, 4, 4), support_sigmas=0.0),
                                 dict(dims=(4, 4, 4), spacing=(1.0, -1.0, 1.0))])
def test_invalid_config_rejected(gp, session, bad):
    """VoxelizerConfig::validate (voxelize.hpp:24-37)."""
    session.set_gaussians(on_center(gp, (2.0, 2.0, 2.0), 0.5))
    with pytest.raises(gp.InvalidArgument):
        session.voxelize(gp.VoxelizerConfig(**bad))


def test_backward_trivial_cases(gp, session):
    """test_voxelize.cpp:149-175"""
    session.set_gaussians(on_center(gp, (8.0, 8.0, 8.0), 0.5))
    cfg = unit_cfg(gp, 16)
    gz = session.voxelize_backward(cfg, np.zeros((16, 16, 16), np.float32))
    assert not gz.any()
    one = np.zeros((16, 16, 16), np.float32)
    one[8, 8, 8] = 1.0
    g1 = session.voxelize_backward(cfg, one)
    assert g1[0, 10] == pytest.approx(0.25, rel=1e-6)  # dL/dalpha_raw = alpha (1 - alpha)
    assert np.linalg.norm(g1[0, 0:3]) <= 1e-6           # symmetric peak


@pytest.mark.parametrize("n,count,tile", [(12, 3, (8, 8, 8)), (48, 1500, (8, 8, 8)),
                                          (40, 800, (4, 8, 16)), (64, 600, (64, 64, 8))])
def test_backward_matches_reference(gp, session, ref, n, count, tile):
    """Last case stages a 128 KB dL/dV tile: exercises the global-memory path."""
    gs = random_scene(gp, count, (3, 3, 3), (n - 3, n - 3, n - 3), scale=1.2, seed=11 + count)
    cfg = unit_cfg(gp, n, tile_dims=tile, support_sigmas=3.0 if count > 3 else 10.0)
    dl = np.random.default_rng(count).uniform(-1.0, 1.0, (n, n, n)).astype(np.float32)
    session.set_gaussians(gs)
    g = session.voxelize_backward(cfg, dl)
    rg = ref.voxelize_backward(gs.records, cfg, dl.astype(np.float64))
    ok, worst = grads_ok(g, rg)
    assert ok, f"voxel gradients beyond tolerance (worst {worst:.2f} x bound)"


def test_backward_volume_shape_mismatch(gp, session):
    session.set_gaussians(on_center(gp, (8.0, 8.0, 8.0), 0.5))
    with pytest.raises(gp.InvalidArgument):
        session.voxelize_backward(unit_cfg(gp, 16), np.zeros((16, 16, 15), np.float32))


def test_voxelize_then_render_stays_exact(gp, session, ref):
    """The voxelizer reuses the pair/sort buffers: a later slice must still bin
    bit-exactly (histogram rows cleared) and the prepared state must be dropped."""
    dims = (64, 64, 16)
    gs = random_scene(gp, 4000, (-0.5, -0.5, -0.5), (63.5, 63.5, 15.5), scale=1.5, seed=21)
    session.set_gaussians(gs)
    pose = gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 7)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    session.prepare(pose, psf, rc)
    session.voxelize(gp.VoxelizerConfig(dims=(64, 64, 16)))
    with pytest.raises(gp.StateError):
        session.prepared()
    session.prepare(pose, psf, rc)
    off, ent = session.tile_lists()
    roff, rent = ref.tile_lists(gs.records, pose, psf, rc, (gs.bbox_min, gs.bbox_max))
    assert np.array_equal(off, roff) and np.array_equal(ent, rent)
    img = session.rasterize()
    ok, worst = image_ok(img, ref.rasterize(gs.records, pose, psf, rc, (gs.bbox_min, gs.bbox_max)))
    assert ok, worst
