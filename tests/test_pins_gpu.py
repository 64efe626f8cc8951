"""The reference's own render pins restated for the device (proj/tests/
test_render.cpp), through the C-ABI, with fp32-appropriate tolerances where the
reference's are fp64 ones. Every PreparedGaussian field the device reports
(gpk_get_prepared_fields) is also compared with the reference's
prepare_gaussians (oracle/_ref) field by field.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu


def plain_pose(gp, w, h):
    """test_render.cpp:17-26"""
    return gp.SlicePose(np.eye(3), (0.0, 0.0, 0.0), w, h, (1.0, 1.0), (0.0, 0.0))


def prim(mu, log_scale=(0.0, 0.0, 0.0), quat=(1.0, 0.0, 0.0, 0.0), alpha=0.5):
    return [*mu, *log_scale, *quat, math.log(alpha / (1.0 - alpha))]


def fields_close(a, b, rel=1e-10, abs_=1e-12):
    return bool(np.all(np.abs(a - b) <= rel * np.abs(b) + abs_))


def test_identity_covariance_chain(gp, session):
    """test_render.cpp:80-93 (acceptance.cpp:206-224): Sigma_c = I, mu_c = (0,0,1),
    sigma_z = 1 -> Sigma_e = diag(1,1,1/2), mu_e = (0,0,1/2), opacity e^{-1/4}."""
    gs = gp.GaussianSet(np.array([prim((0.0, 0.0, 1.0))]), (-8, -8, -8), (8, 8, 8))
    session.set_gaussians(gs)
    session.prepare(plain_pose(gp, 16, 16), gp.PsfSpec(sigma_z=1.0), gp.RasterConfig())
    f = session.prepared_fields()
    assert len(f["alpha"]) == 1
    assert np.allclose(f["sigma_e"][0], np.diag([1.0, 1.0, 0.5]), rtol=0, atol=1e-12)
    assert np.allclose(f["mu_e"][0], [0.0, 0.0, 0.5], rtol=0, atol=1e-12)
    assert abs(f["opacity_r"][0] - math.exp(-0.25)) < 1e-12
    assert np.allclose(f["sigma_c"][0], np.eye(3), atol=1e-15)
    assert np.allclose(f["sigma_c_inv"][0], np.eye(3), atol=1e-15)
    assert abs(f["alpha_tilde"][0] - 0.5 * math.exp(-0.25)) < 1e-12  # det(Sigma_2d) = 1


def test_all_in_focus_limit(gp, session):
    """test_render.cpp:336-353: sigma_z = 1e9 -> opacity_r = 1, Sigma_2d = Sigma_c[0:2, 0:2]."""
    from oracle.bindings import RefRng

    rng = RefRng(23)
    bbox = ((0, 0, -4), (16, 16, 4))
    for trial in range(10):
        rec = f32(np.stack([rng.random_primitive(bbox)]))
        session.set_gaussians(gp.GaussianSet(rec, *bbox))
        session.prepare(plain_pose(gp, 16, 16), gp.PsfSpec(sigma_z=1e9), gp.RasterConfig(tau=0.0))
        f = session.prepared_fields()
        assert len(f["alpha"]) == 1, trial
        assert abs(f["opacity_r"][0] - 1.0) < 1e-6
        sc, cov = f["sigma_c"][0], f["cov2d"][0]
        assert abs(cov[0, 0] - sc[0, 0]) <= 1e-6 * abs(sc[0, 0])
        assert abs(cov[0, 1] - sc[0, 1]) <= 1e-6
        assert abs(cov[1, 1] - sc[1, 1]) <= 1e-6 * abs(sc[1, 1])
        # and the image is the unmodulated 2-D Gaussian the reference renders
        img = session.rasterize()
        assert img.max() > 0


def test_prepared_fields_match_reference(gp, session, ref):
    """Every PreparedGaussian field (render.hpp:68-79) vs the reference's
    prepare_gaussians: C1 mid slice, a thick PSF and random rotated poses."""
    from oracle.bindings import RefRng

    dims = (128, 128, 32)
    lo, hi = (-0.5,) * 3, (127.5, 127.5, 31.5)
    gs = gp.GaussianSet(f32(gp.init_random(20_000, lo, hi, 1.5, 1).records), lo, hi)
    cases = [(gs, gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 16), gp.PsfSpec(), gp.RasterConfig()),
             (gs, gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), 9), gp.PsfSpec(sigma_z=3.0),
              gp.RasterConfig(tau=0.0, footprint_sigmas=4.0))]
    rng = RefRng(7)
    for _ in range(4):
        pc = rng.random_pose_c(24, 24)
        pose = gp.SlicePose(np.array(list(pc.rotation)).reshape(3, 3), tuple(pc.translation), 24, 24,
                            (1.0, 1.0), tuple(pc.principal_point))
        b = ((-2, -2, -2), (2, 2, 2))
        rec = f32(np.stack([rng.random_primitive(b, 0.6, 1.8) for _ in range(5)]))
        cases.append((gp.GaussianSet(rec, *b), pose, gp.PsfSpec(), gp.RasterConfig(tau=0.0, footprint_sigmas=8.0)))
    for gset, pose, psf, rc in cases:
        session.set_gaussians(gset)
        session.prepare(pose, psf, rc)
        f = session.prepared_fields()
        raw = np.concatenate([f["alpha"][:, None], f["opacity_r"][:, None], f["alpha_tilde"][:, None],
                              f["mu_c"], f["mu_e"], f["sigma_c"].reshape(-1, 9), f["sigma_c_inv"].reshape(-1, 9),
                              f["sigma_e"].reshape(-1, 9), f["mu_2d"], f["cov2d"].reshape(-1, 4),
                              f["conic"].reshape(-1, 4), f["det2"][:, None]], axis=1)
        want = ref.prepare_full(gset.records, pose, psf, rc, (gset.bbox_min, gset.bbox_max))
        assert raw.shape == want.shape
        scale = np.maximum(np.abs(want).max(axis=0, keepdims=True), 1e-300)
        err = np.abs(raw - want) / (np.abs(want) + 1e-12 * scale)
        assert err.max() < 1e-9, f"field {int(np.argmax(err.max(axis=0)))} rel err {err.max():.3g}"


def test_linearity_over_subsets_tau0(gp, session):
    """test_render.cpp:264-284: at tau = 0, I(A u B) = I(A) + I(B) (1e-6)."""
    from oracle.bindings import RefRng

    rng = RefRng(17)
    bbox = ((0, 0, -3), (16, 16, 3))
    prims = [rng.random_primitive(bbox) for _ in range(6)]
    cfg, psf, pose = gp.RasterConfig(tau=0.0), gp.PsfSpec(), plain_pose(gp, 16, 16)

    def render(rows):
        session.set_gaussians(gp.GaussianSet(f32(np.stack(rows)), *bbox))
        session.prepare(pose, psf, cfg)
        return session.rasterize().astype(np.float64)

    a = render(prims[0::2])
    b = render(prims[1::2])
    both = render(prims)
    assert np.all(np.abs(both - (a + b)) <= 1e-6)


def test_focus_falloff_over_nine_slices(gp, session):
    """test_render.cpp:301-334: mu_z = 0.1 peaks on the nearest slice (k = 4) and
    decays monotonically on both sides."""
    g = prim((8.0, 8.0, 0.1), (math.log(1.2),) * 3, alpha=0.8)
    session.set_gaussians(gp.GaussianSet(np.array([g]), (-20, -20, -20), (20, 20, 20)))
    peaks = []
    for k in range(9):
        pose = gp.slice_pose_for_index((16, 16, 9), (1, 1, 1), (0.0, 0.0, -4.0), k)
        session.prepare(pose, gp.PsfSpec(sigma_z=1.0), gp.RasterConfig(tau=0.0))
        peaks.append(float(session.rasterize().max()))
    assert int(np.argmax(peaks)) == 4
    assert all(peaks[k] < peaks[k + 1] for k in range(3))
    assert all(peaks[k] > peaks[k + 1] for k in range(5, 8))


def test_quadrature_oracle_ratio_and_log_profile(gp, session, ref):
    """test_render.cpp:373-442 (acceptance criterion 1): the device's analytic
    slice image is proportional to the reference's adaptive-quadrature oracle
    (render_oracle, render.hpp:251-272) — ratio constant across pixels (CoV),
    same argmax, log-profiles equal up to a constant. fp32 pixels: CoV bound
    5e-6 instead of the fp64 1e-6; the log-profile bound is the reference's."""
    from oracle.bindings import RefRng

    rng = RefRng(29)
    psf, cfg, pose = gp.PsfSpec(sigma_z=1.0), gp.RasterConfig(tau=0.0), plain_pose(gp, 24, 24)
    bbox = ((4, 4, -2), (20, 20, 2))
    worst_cov = 0.0
    for trial in range(20):
        rec = f32(np.stack([rng.random_primitive(bbox, 0.8, 2.5)]))
        session.set_gaussians(gp.GaussianSet(rec, *bbox))
        session.prepare(pose, psf, cfg)
        prep = session.prepared()
        assert len(prep.index) == 1
        lo_x, hi_x, lo_y, hi_y = (int(v) for v in prep.bounds[0])
        at = session.prepared_fields()["alpha_tilde"][0]
        img = session.rasterize().astype(np.float64)
        ratios = []
        for j in range(lo_y, hi_y + 1):
            for i in range(lo_x, hi_x + 1):
                if len(ratios) >= 50:
                    break
                a = img[j, i]
                if a < 1e-4 * at:
                    continue
                ratios.append(ref.render_oracle(rec, 0, pose, psf, float(i), float(j)) / a)
        assert len(ratios) >= 10
        r = np.array(ratios)
        cov = r.std() / r.mean()
        worst_cov = max(worst_cov, cov)
        assert cov < 5e-6, (trial, cov)
        orc = np.zeros_like(img)
        for j in range(lo_y, hi_y + 1):
            for i in range(lo_x, hi_x + 1):
                orc[j, i] = ref.render_oracle(rec, 0, pose, psf, float(i), float(j))
        win = (slice(lo_y, hi_y + 1), slice(lo_x, hi_x + 1))
        pa = np.unravel_index(np.argmax(img[win]), img[win].shape)
        po = np.unravel_index(np.argmax(orc[win]), orc[win].shape)
        assert pa == po or abs(img[win][po] - img[win][pa]) <= 1e-6 * img[win][pa]
        peak, opeak = img[win].max(), orc[win].max()
        offset = math.log(opeak) - math.log(peak)
        for j in range(lo_y, hi_y + 1, 2):
            for i in range(lo_x, hi_x + 1, 2):
                if img[j, i] < 1e-3 * peak:
                    continue
                d = math.log(orc[j, i]) - math.log(img[j, i])
                assert abs(d - offset) <= 1e-4 * (1.0 + abs(offset))
    print(f"quadrature ratio: worst CoV {worst_cov:.3g}")
