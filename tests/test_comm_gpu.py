"""The NCCL path of the slice-sharded training step on one GPU: a world-size-1
communicator through the C-ABI (NCCL loaded by the library, ncclCommInitRank,
the grouped reduce-scatter / all-gather inside the training step). With one
rank the collectives are identities, so the step under a communicator — dense
gradient planes, reduce-scatter, Adam on the rank's shard (here: everything),
parameter all-gather — must equal the single-GPU step with slot gradients
bitwise."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def f32(rec):
    return rec.astype(np.float32).astype(np.float64)


def _comm_session(gp):
    from paper_2603_20611_b200 import _native as N
    from paper_2603_20611_b200 import dp

    s = gp.Session(0)
    uid = dp.native_unique_id()
    buf = (C.c_char * dp.NCCL_ID_BYTES).from_buffer_copy(uid)
    N.check(N.lib.gpk_comm_init(s.handle, 1, 0, buf))
    return s


def test_train_step_under_world1_communicator_equals_single_gpu(gp, session):
    from paper_2603_20611_b200 import _native as N

    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 21).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (3, 7, 5)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(22).uniform(0, 0.1, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    sc = _comm_session(gp)
    try:
        for s in (session, sc):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        for it in range(6):
            p = poses[it % 3]
            session.train_step(p, psf, rc, 0.2, 0.5, lr0, 30)
            sc.train_step(p, psf, rc, 0.2, 0.5, lr0, 30)
            assert np.array_equal(session.get_gaussians(), sc.get_gaussians()), it
            m1, v1, st1 = session.adam_state()
            m2, v2, st2 = sc.adam_state()
            assert st1 == st2 and np.array_equal(m1, m2) and np.array_equal(v1, v2), it
        # graphs under the communicator (the all-reduce is a captured node)
        gid = sc.capture_train(poses[0], psf, rc, 0.2, 0.5, lr0, 30)
        for it in range(2):
            session.train_step(poses[0], psf, rc, 0.2, 0.5, lr0, 30)
            sc.graph_launch(gid)
            assert np.array_equal(session.get_gaussians(), sc.get_gaussians()), it
        sc.graph_destroy_all()
        # the stand-alone all-reduce of a backward's dense gradient
        dl = np.random.default_rng(23).normal(0, 1e-3, (48, 64)).astype(np.float32)
        sc.prepare(poses[1], psf, rc)
        g = sc.backward(dl)
        N.check(N.lib.gpk_allreduce_grads(sc.handle))
        assert np.array_equal(sc.get_gradients(), g)
    finally:
        N.check(N.lib.gpk_comm_destroy(sc.handle))
        sc.close()


def test_union_exchange_world1_equals_single_gpu(gp, session):
    """gpk_train_step_dp at world size 1 (union of one pose, one all-reduce of
    the union rows, Adam from the rows) == gpk_train_step bitwise, direct and
    as a captured graph."""
    from paper_2603_20611_b200 import _native as N

    dims = (64, 48, 12)
    lo, hi = (-0.5, -0.5, -0.5), (63.5, 47.5, 11.5)
    gs = gp.GaussianSet(f32(gp.init_random(3000, lo, hi, 1.5, 23).records), lo, hi)
    poses = [gp.slice_pose_for_index(dims, (1, 1, 1), (0, 0, 0), k) for k in (4, 8, 6)]
    psf, rc = gp.PsfSpec(), gp.RasterConfig()
    tgt = np.random.default_rng(24).uniform(0, 0.1, (48, 64)).astype(np.float32)
    lr0 = gp.LearningRates(6e-4, 0.02, 2e-3, 1e-3)
    sc = _comm_session(gp)
    try:
        for s in (session, sc):
            s.set_gaussians(gs)
            s.upload(N.GPK_BUF_TARGET, tgt.ctypes.data, tgt.nbytes)
        for it in range(4):
            p = poses[it % 3]
            session.train_step(p, psf, rc, 0.2, 0.5, lr0, 30)
            sc.train_step_dp(1, 0, [p], psf, rc, 0.2, 0.5, lr0, 30)
            assert np.array_equal(session.get_gaussians(), sc.get_gaussians()), it
            assert np.array_equal(session.get_gradients(), sc.get_gradients()), it
        rows, cap = sc.dp_union_rows()
        assert 0 < rows <= cap
        gids = [sc.capture_train_dp(1, 0, [p], psf, rc, 0.2, 0.5, lr0, 30) for p in poses]
        for it in range(3):
            session.train_step(poses[it], psf, rc, 0.2, 0.5, lr0, 30)
            sc.graph_launch(gids[it])
            assert np.array_equal(session.get_gaussians(), sc.get_gaussians()), it
        sc.graph_destroy_all()
    finally:
        sc.close()
