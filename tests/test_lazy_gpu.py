"""Lazy training steps (LazyAdam, csrc/common.cuh; gpk_set_lazy_adam): the
survivors and one 1/16 window of the set are updated per step, every other
Gaussian's zero-gradient Adam step (optimize.hpp:195-221 with g = 0) is
deferred and replayed in order where it is next needed.

The contract is bit-identity with the eager step (every Gaussian updated
every step, the form pinned against the reference in test_train_gpu.py and
test_configs_gpu.py): per-step losses (which see the survivors' replayed
parameters through the cull, the render and the chain) and the final
parameters, moments and step counter, after runs long enough that Gaussians
sit deferred for up to 15 steps, with the paths that replay everything
(non-identity poses, a moment state outside the drift bound), graphs, and the
API calls that read or write the state in between.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import f32

pytestmark = pytest.mark.gpu

DIMS = (96, 80, 24)
LR0 = (6e-4, 0.02, 2e-3, 1e-3)
TOTAL = 300


def scene(gp, n=9000, seed=11, dims=DIMS, scale=1.5):
    lo, hi = (-0.5, -0.5, -0.5), (dims[0] - 0.5, dims[1] - 0.5, dims[2] - 0.5)
    return gp.GaussianSet(f32(gp.init_random(n, lo, hi, scale, seed).records), lo, hi)


def slice_pose(gp, k, dims=DIMS):
    return gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k)


def order(steps, nz, seed=0):
    return list(np.random.default_rng(seed).integers(0, nz, steps))


def run(gp, s, ks, tgt, graphs=None, dims=DIMS, lr0=LR0):
    """Train steps over slice indices ks; returns the per-step losses."""
    from paper_2603_20611_b200 import _native as N

    psf, rc, lr = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*lr0)
    s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    losses = np.zeros(len(ks))
    for j, k in enumerate(ks):
        if graphs is not None:
            s.graph_launch(graphs[k])
        else:
            s.train_step(slice_pose(gp, k, dims), psf, rc, 0.2, 0.5, lr, TOTAL)
        s.download(N.GPK_BUF_LOSS, losses.ctypes.data + 8 * j, 8)
    s.synchronize()
    return losses


def state(s):
    p = s.get_gaussians()
    m, v, st = s.adam_state()
    return p, m, v, st


def assert_same_state(a, b):
    for x, y, name in zip(a, b, ("params", "m", "v", "step")):
        assert np.array_equal(x, y), name


@pytest.fixture
def pair(gp):
    with gp.Session(0) as lazy, gp.Session(0) as eager:
        lazy.set_lazy_adam(True)
        yield lazy, eager


def target(shape=(DIMS[1], DIMS[0]), seed=7):
    return np.random.default_rng(seed).uniform(0, 0.1, shape).astype(np.float32)


def test_lazy_steps_equal_eager(gp, pair):
    lazy, eager = pair
    gs, tgt = scene(gp), target()
    ks = order(60, DIMS[2])
    for s in pair:
        s.set_gaussians(gs)
    la, le = run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt)
    assert np.array_equal(la, le)
    assert_same_state(state(lazy), state(eager))
    # continue after the flush the state reads did
    ks2 = order(25, DIMS[2], seed=1)
    assert np.array_equal(run(gp, lazy, ks2, tgt), run(gp, eager, ks2, tgt))
    assert_same_state(state(lazy), state(eager))
    # lazy steps left deferred, then the mode switched off (they are replayed)
    ks3 = order(11, DIMS[2], seed=2)
    assert np.array_equal(run(gp, lazy, ks3, tgt), run(gp, eager, ks3, tgt))
    lazy.set_lazy_adam(False)
    assert np.array_equal(run(gp, lazy, ks2, tgt), run(gp, eager, ks2, tgt))
    assert_same_state(state(lazy), state(eager))


def test_lazy_graphs_equal_eager(gp, pair):
    lazy, eager = pair
    gs, tgt = scene(gp, seed=12), target(seed=8)
    psf, rc, lr = gp.PsfSpec(), gp.RasterConfig(), gp.LearningRates(*LR0)
    for s in pair:
        s.set_gaussians(gs)
    from paper_2603_20611_b200 import _native as N

    lazy.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
    graphs = [lazy.capture_train(slice_pose(gp, k), psf, rc, 0.2, 0.5, lr, TOTAL) for k in range(DIMS[2])]
    ks = order(70, DIMS[2], seed=3)
    la = run(gp, lazy, ks, tgt, graphs=graphs)
    le = run(gp, eager, ks, tgt)
    assert np.array_equal(la, le)
    assert_same_state(state(lazy), state(eager))
    lazy.graph_destroy_all()


def test_lazy_mixed_api_equal_eager(gp, pair):
    """Lazy steps interleaved with a U1 fwd+bwd (its cull replays), an eager
    Adam call (everything replayed first), a gradient read and a pose with a
    rotation (no drift test: every deferred step replayed first)."""
    from paper_2603_20611_b200 import _native as N

    lazy, eager = pair
    gs, tgt = scene(gp, seed=13), target(seed=9)
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    for s in pair:
        s.set_gaussians(gs)
    ks = order(20, DIMS[2], seed=4)
    assert np.array_equal(run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt))
    dl = (np.random.default_rng(2).uniform(-1, 1, (DIMS[1], DIMS[0])) / 7680).astype(np.float32)
    g = []
    for s in pair:
        s.upload(N.GPK_BUF_DL_DI, dl.ctypes.data, dl.nbytes)
        s.fwd_bwd_slice(slice_pose(gp, 9), psf, rc)
        g.append(s.get_gradients())
    assert np.array_equal(g[0], g[1])
    ks = order(9, DIMS[2], seed=5)
    assert np.array_equal(run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt))
    for s in pair:  # eager Adam on the dense gradient of the last backward
        s.adam_step(gp.LearningRates(*LR0))
    ks = order(18, DIMS[2], seed=6)
    assert np.array_equal(run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt))
    c, sn = np.cos(0.3), np.sin(0.3)
    rot = gp.SlicePose(np.array([[c, -sn, 0], [sn, c, 0], [0, 0, 1]]), (-40.0, -30.0, 11.0), DIMS[0], DIMS[1],
                       (1.0, 1.0), (0.0, 0.0))
    lr = gp.LearningRates(*LR0)
    ls = []
    for s in pair:
        s.train_step(rot, psf, rc, 0.2, 0.5, lr, TOTAL)
        L = np.zeros(1)
        s.download(N.GPK_BUF_LOSS, L.ctypes.data, 8)
        s.synchronize()
        ls.append(L[0])
    assert ls[0] == ls[1]
    ks = order(12, DIMS[2], seed=7)
    assert np.array_equal(run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt))
    assert_same_state(state(lazy), state(eager))


def test_lazy_state_outside_bound_replays_all(gp, pair):
    """A moment state with |m| > K sqrt(v) (set through the API) voids the
    drift bound: K_filter then replays every Gaussian; still the eager bits."""
    lazy, eager = pair
    gs, tgt = scene(gp, seed=14), target(seed=10)
    for s in pair:
        s.set_gaussians(gs)
    n = gs.size()
    rng = np.random.default_rng(3)
    v = rng.uniform(1e-8, 1e-6, (n, 11))
    m = 0.1 * np.sqrt(v) * rng.standard_normal((n, 11))
    m[::7] *= 200.0  # |m| up to ~60 sqrt(v): outside |m| <= 7.4 sqrt(v)
    m, v = m.astype(np.float32), v.astype(np.float32)
    for s in pair:
        s.set_adam_state(m, v, 5)
    ks = order(40, DIMS[2], seed=8)
    assert np.array_equal(run(gp, lazy, ks, tgt), run(gp, eager, ks, tgt))
    assert_same_state(state(lazy), state(eager))


def test_lazy_c2_scale_equal_eager(gp, pair):
    """BASELINE C2 geometry (512^2 x 128, 1M Gaussians), 40 steps over the
    central slices: losses and final state bit-identical."""
    dims = (512, 512, 128)
    lazy, eager = pair
    gs = scene(gp, n=1_000_000, seed=1, dims=dims)
    tgt = target((512, 512), seed=7)
    for s in pair:
        s.set_gaussians(gs)
        s.reserve_pairs(1 << 20)
    ks = [56 + int(k) for k in order(40, 16, seed=9)]
    la, le = run(gp, lazy, ks, tgt, dims=dims), run(gp, eager, ks, tgt, dims=dims)
    assert np.array_equal(la, le)
    assert_same_state(state(lazy), state(eager))
