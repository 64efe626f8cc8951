"""CPU: pin the checkers before trusting them.

* The C restatement (oracle/gpile_oracle.c) against the golden fixtures the
  reference itself produced (tests/golden/make_golden.py): tile lists and
  survivor sets bit-exact, floating point to ~1e-12 relative (both are fp64
  CPU implementations of the same formulas; the restatement keeps the
  reference's operation order where it matters).
* The reference build (oracle/_ref), when present, reproduces the fixtures
  bit for bit (the fixtures are not stale).
* Closed-form pins from the reference's own tests (test_render.cpp,
  test_grad.cpp, test_loss.cpp, test_optim.cpp, test_voxelize.cpp).
"""
from __future__ import annotations

import json
import math
from pathlib import Path
from types import SimpleNamespace as NS

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
RENDER_CASES = ["render_stack_k3", "render_stack_k6", "render_random_pose", "render_thick_psf"]


def load_case(name):
    d = np.load(GOLD / f"{name}.npz")
    meta = json.loads(str(d["meta"]))
    pm = meta["pose"]
    pose = NS(rotation=np.array(pm["rotation"]).reshape(3, 3), translation=tuple(pm["translation"]),
              width=pm["width"], height=pm["height"], pixel_spacing=tuple(pm["pixel_spacing"]),
              principal_point=tuple(pm["principal_point"]))
    psf = NS(sigma_x=meta["psf"][0], sigma_y=meta["psf"][1], sigma_z=meta["psf"][2])
    cfg = NS(tau=meta["cfg"][0], tile_size=meta["cfg"][1], footprint_sigmas=meta["cfg"][2],
             scale_modifier=meta["cfg"][3])
    bbox = (tuple(meta["bbox"][0]), tuple(meta["bbox"][1]))
    return d, pose, psf, cfg, bbox


def close(a, b, rel=1e-12, abs_of_max=1e-12):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.abs(b).max() if b.size else 0.0
    return np.all(np.abs(a - b) <= rel * np.abs(b) + abs_of_max * scale)


@pytest.mark.parametrize("name", RENDER_CASES)
def test_oracle_render_matches_golden(oracle, name):
    d, pose, psf, cfg, bbox = load_case(name)
    rec = d["records"]
    idx, bnd, fld = oracle.prepare(rec, pose, psf, cfg, bbox)
    assert np.array_equal(idx, d["index"]), "survivor set (render.hpp:107,127)"
    assert np.array_equal(bnd, d["bounds"]), "pixel bounds (render.hpp:116-126)"
    assert close(fld, d["fields"], 1e-10, 1e-12)
    off, ent = oracle.tile_lists(rec, pose, psf, cfg, bbox)
    assert np.array_equal(off, d["offsets"]) and np.array_equal(ent, d["entries"])
    assert close(oracle.rasterize(rec, pose, psf, cfg, bbox), d["image"], 1e-11, 1e-13)
    g, (nrm, obs, wld) = oracle.backward(rec, pose, psf, cfg, d["dl_di"], bbox)
    assert close(g, d["grads"], 1e-8, 1e-11)
    assert np.array_equal(obs, d["stat_observed"])
    assert close(nrm, d["stat_norm"], 1e-8, 1e-11)
    assert close(wld, d["stat_world"], 1e-8, 1e-11)


@pytest.mark.parametrize("name", RENDER_CASES)
def test_reference_reproduces_golden(ref, name):
    d, pose, psf, cfg, bbox = load_case(name)
    rec = d["records"]
    idx, bnd, fld = ref.prepare(rec, pose, psf, cfg, bbox)
    assert np.array_equal(idx, d["index"]) and np.array_equal(bnd, d["bounds"])
    assert np.array_equal(fld, d["fields"])
    assert np.array_equal(ref.rasterize(rec, pose, psf, cfg, bbox), d["image"])
    g, _ = ref.backward(rec, pose, psf, cfg, d["dl_di"], bbox)
    assert np.array_equal(g, d["grads"])


def test_oracle_tiled_equals_naive(oracle):
    """rasterize_prepared == rasterize_naive bitwise (test_render.cpp:286-299)."""
    d, pose, psf, cfg, bbox = load_case("render_random_pose")
    a = oracle.rasterize(d["records"], pose, psf, cfg, bbox)
    b = oracle.rasterize(d["records"], pose, psf, cfg, bbox, naive=True)
    assert np.array_equal(a, b)


def test_oracle_loss_matches_golden(oracle):
    d = np.load(GOLD / "loss.npz")
    for lam in (0.0, 0.2, 1.0):
        L, dl = oracle.loss(d["rendered"], d["target"], lam, 0.5)
        assert math.isclose(L, float(d[f"loss_{lam}"]), rel_tol=1e-12)
        assert close(dl, d[f"dl_{lam}"], 1e-10, 1e-12)


def test_oracle_adam_matches_golden(oracle):
    d = np.load(GOLD / "adam.npz")
    rec, m, v, step = d["records"], np.zeros_like(d["records"]), np.zeros_like(d["records"]), 0
    bbox = (tuple(d["bbox"][0]), tuple(d["bbox"][1]))
    for s in range(3):
        rec, m, v, step = oracle.adam_step(rec, bbox, d["grads"][s], m, v, step, tuple(d["lrs"]))
        assert close(rec, d[f"rec_{s}"], 1e-13, 0) and close(m, d[f"m_{s}"], 1e-13, 0)
        assert close(v, d[f"v_{s}"], 1e-13, 0)
    assert step == 3


def test_oracle_voxel_matches_golden(oracle):
    d = np.load(GOLD / "voxel.npz")
    meta = json.loads(str(d["meta"]))
    vc = NS(**{k: tuple(v) if isinstance(v, list) else v for k, v in meta.items()})
    off, ent = oracle.voxel_tiles(d["records"], vc)
    assert np.array_equal(off, d["offsets"]) and np.array_equal(ent, d["entries"])
    assert close(oracle.voxelize(d["records"], vc), d["volume"], 1e-11, 1e-13)
    assert close(oracle.voxelize_backward(d["records"], vc, d["dl_dv"]), d["grads"], 1e-8, 1e-11)


# ---- closed-form pins on the restatement (the reference's own unit tests) ----

def unit_primitive(alpha=0.5, mu=(8.0, 8.0, 0.0), s=1.0):
    rec = np.zeros((1, 11))
    rec[0, 0:3] = mu
    rec[0, 3:6] = math.log(s)
    rec[0, 6] = 1.0
    rec[0, 10] = math.log(alpha / (1 - alpha))
    return rec


def plain(w, h):
    return NS(rotation=np.eye(3), translation=(0.0, 0.0, 0.0), width=w, height=h, pixel_spacing=(1.0, 1.0),
              principal_point=(0.0, 0.0))


def test_oracle_unit_primitive_spot_values(oracle):
    """test_render.cpp:245-262: I(8,8) = alpha*op/sqrt(det) with sigma_z = 1e9 (all in focus)."""
    rec = unit_primitive(alpha=0.5)
    psf = NS(sigma_x=1.0, sigma_y=1.0, sigma_z=1e9)
    cfg = NS(tau=0.0, tile_size=16, footprint_sigmas=3.0, scale_modifier=1.0)
    img = oracle.rasterize(rec, plain(17, 17), psf, cfg)
    assert abs(img[8, 8] - 0.5) < 1e-9
    assert abs(img[8, 9] - 0.5 * math.exp(-0.5)) < 1e-9


def test_oracle_zero_upstream_zero_grads(oracle):
    """test_grad.cpp:89-100"""
    d, pose, psf, cfg, bbox = load_case("render_stack_k3")
    g, _ = oracle.backward(d["records"], pose, psf, cfg, np.zeros_like(d["dl_di"]), bbox)
    assert not g.any()


def test_oracle_center_pixel_alpha_grad(oracle):
    """test_grad.cpp:102-126: dL/dalpha_raw at the centre pixel = alpha(1-alpha)/sqrt(det)*op."""
    rec = unit_primitive(alpha=0.3)
    psf = NS(sigma_x=1.0, sigma_y=1.0, sigma_z=1e9)
    cfg = NS(tau=0.0, tile_size=16, footprint_sigmas=3.0, scale_modifier=1.0)
    dl = np.zeros((17, 17))
    dl[8, 8] = 1.0
    g, _ = oracle.backward(rec, plain(17, 17), psf, cfg, dl)
    assert abs(g[0, 10] - 0.3 * 0.7) < 1e-9


def test_oracle_lr_schedule(oracle):
    d = np.load(GOLD / "adam.npz")
    want = d["lr_at"][0]
    got = [lr0 * 0.1 ** ((it - 1) / tot) for lr0, it, tot in ((6e-4, 1, 30000), (6e-4, 15000, 30000),
                                                             (0.02, 30000, 30000), (1e-3, 7, 10))]
    assert np.allclose(got, want, rtol=1e-15, atol=0)


def test_oracle_error_paths(oracle):
    from oracle.bindings import CheckerError

    rec = unit_primitive()
    rec[0, 6:10] = 0.0  # zero quaternion: std::invalid_argument (vec.hpp:185-186)
    cfg = NS(tau=0.0, tile_size=16, footprint_sigmas=3.0, scale_modifier=1.0)
    with pytest.raises(CheckerError):
        oracle.rasterize(rec, plain(17, 17), NS(sigma_x=1.0, sigma_y=1.0, sigma_z=1.0), cfg)
    with pytest.raises(CheckerError):  # PsfSpec::validate (core.hpp:112-116)
        oracle.rasterize(unit_primitive(), plain(17, 17), NS(sigma_x=1.0, sigma_y=1.0, sigma_z=0.0), cfg)
