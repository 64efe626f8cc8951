"""CPU, world_size 2 over gloo: the host side of slice-sharded data parallelism
(paper_2603_20611_b200/dp.py).

* the slice schedule deals distinct slices to the ranks of a step and covers
  the schedule;
* the NCCL unique id created on rank 0 reaches every rank intact;
* max-over-ranks timing reduction;
* the exchange algebra: each rank's dense gradient of its own slice (the C
  oracle stands in for the device backward), summed by an all-reduce, equals
  the serial sum over the step's slices — what ncclAllReduce(sum) over the
  11-plane buffer computes on the GPUs;
* the training step's ZeRO-style update: reduce the summed gradient to each
  primitive's owner, Adam on the owner's shard only, all-gather the parameter
  shards — every replica ends bitwise equal to the full all-reduce + full Adam;
* the union-compacted exchange (gpk_train_step_dp, csrc/dp.cu): each rank
  derives the union of the step's survivors itself, numbers it like the
  device (dp.union_rows), packs its gradient into those rows; one all-reduce
  of the rows, unpacked, equals the dense all-reduce.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from types import SimpleNamespace as NS

    rng = np.random.default_rng(0)
    n = 300
    rec = np.zeros((n, 11))
    rec[:, 0] = rng.uniform(0, 32, n)
    rec[:, 1] = rng.uniform(0, 24, n)
    rec[:, 2] = rng.uniform(0, 8, n)
    rec[:, 3:6] = np.log(rng.uniform(0.8, 1.6, (n, 3)))
    q = rng.normal(size=(n, 4))
    rec[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    rec[:, 10] = rng.uniform(-3, 0, n)
    poses = [NS(rotation=np.eye(3), translation=(0.0, 0.0, -float(k)), width=32, height=24,
                pixel_spacing=(1.0, 1.0), principal_point=(0.0, 0.0)) for k in range(8)]
    psf = NS(sigma_x=1.0, sigma_y=1.0, sigma_z=1.0)
    cfg = NS(tau=0.02, tile_size=16, footprint_sigmas=3.0, scale_modifier=1.0)
    dl = [np.random.default_rng(10 + k).uniform(-1, 1, (24, 32)) for k in range(8)]
    return rec, poses, psf, cfg, dl


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from oracle.bindings import load
    from paper_2603_20611_b200 import dp

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        out["uid"] = dp.exchange_unique_id(rank, make_id=lambda: bytes(range(128)))
        out["max"] = dp.max_over_ranks([float(rank), 10.0 - rank])
        oracle = load("oracle")
        rec, poses, psf, cfg, dl = _scene()
        sums = []
        for step in range(3):
            k = dp.slice_for(step, rank, world, len(poses))
            g, _ = oracle.backward(rec, poses[k], psf, cfg, dl[k])
            t = torch.from_numpy(np.ascontiguousarray(g))
            dist.all_reduce(t)  # the exchange: sum of per-slice dense gradients
            sums.append(t.numpy().copy())
        out["sums"] = sums
        # sharded Adam: owner r holds primitives [r*chunk, (r+1)*chunk)
        n = rec.shape[0]
        chunk = (n + world - 1) // world
        bbox = ((-0.5, -0.5, -0.5), (31.5, 23.5, 7.5))
        lrs = (6e-4, 0.02, 2e-3, 1e-3)
        k = dp.slice_for(0, rank, world, len(poses))
        g, _ = oracle.backward(rec, poses[k], psf, cfg, dl[k])
        full = torch.from_numpy(np.array(g, copy=True))
        for r in range(world):  # reduce-scatter: each shard summed onto its owner
            part = full[r * chunk:min(n, (r + 1) * chunk)].clone()  # (gloo may scribble on non-root inputs)
            dist.reduce(part, dst=r)
            if r == rank:
                mine = part.numpy().copy()
        lo, hi = rank * chunk, min(n, (rank + 1) * chunk)
        p = rec[lo:hi].copy()
        m = np.zeros_like(p)
        v = np.zeros_like(p)
        p, m, v = oracle.adam_step(p, bbox, mine, m, v, 0, lrs)[:3]
        shards = [torch.zeros((chunk, 11), dtype=torch.float64) for _ in range(world)]
        mine_p = torch.zeros((chunk, 11), dtype=torch.float64)
        mine_p[:hi - lo] = torch.from_numpy(np.ascontiguousarray(p))
        dist.all_gather(shards, mine_p)  # the parameter shards to every replica
        out["zero_params"] = torch.cat(shards)[:n].numpy()
        out["zero_grads"] = np.array(g, copy=True)
        # union-compacted exchange (csrc/dp.cu): every rank evaluates the cull of
        # ALL the step's poses itself — no collective for the union — numbers
        # the union identically, packs its own gradient into those rows, one
        # all-reduce of the rows, unpack; equals the dense all-reduce
        for step in range(3):
            ks = dp.step_slices(step, world, len(poses))
            union = np.zeros(n, bool)
            for kk in ks:
                idx, _, _ = oracle.prepare(rec, poses[kk], psf, cfg)
                union[idx] = True
            umap = dp.union_rows(union)
            g, _ = oracle.backward(rec, poses[ks[rank]], psf, cfg, dl[ks[rank]])
            assert not np.any(g[~union]), "a rank's gradient lives inside the union"
            rows = torch.from_numpy(dp.pack_rows(np.asarray(g, np.float32), umap))
            dist.all_reduce(rows)
            out.setdefault("union_umap", []).append(umap)
            out.setdefault("union_sum", []).append(dp.unpack_rows(rows.numpy(), umap))
            dense = torch.from_numpy(np.ascontiguousarray(g, np.float32))
            dist.all_reduce(dense)
            out.setdefault("union_dense", []).append(dense.numpy().copy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_slice_schedule_partitions_each_step():
    from paper_2603_20611_b200 import dp

    for world in (1, 2, 4, 8):
        n = 16
        seen = []
        for step in range(n // world):
            ks = dp.step_slices(step, world, n)
            assert len(set(ks)) == world
            seen += ks
        assert sorted(seen) == list(range(n))
    with pytest.raises(ValueError):
        dp.slice_for(0, 2, 2, 4)


def test_gloo_world2_exchange():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["uid"] == res[1]["uid"] == bytes(range(128))
    assert res[0]["max"] == res[1]["max"] == [1.0, 10.0]

    sys.path.insert(0, str(ROOT))
    from oracle.bindings import load
    from paper_2603_20611_b200 import dp

    oracle = load("oracle")
    rec, poses, psf, cfg, dl = _scene()
    for step in range(3):
        want = sum(oracle.backward(rec, poses[k], psf, cfg, dl[k])[0] for k in dp.step_slices(step, 2, len(poses)))
        for r in (0, 1):
            assert np.allclose(res[r]["sums"][step], want, rtol=1e-12, atol=1e-15)
        assert np.array_equal(res[0]["sums"][step], res[1]["sums"][step])  # replicas stay equal
    # sharded update == all-reduce + full Adam, bitwise, on both replicas
    g_sum = res[0]["zero_grads"] + res[1]["zero_grads"]
    bbox = ((-0.5, -0.5, -0.5), (31.5, 23.5, 7.5))
    want = oracle.adam_step(rec.copy(), bbox, g_sum, np.zeros_like(rec), np.zeros_like(rec), 0,
                            (6e-4, 0.02, 2e-3, 1e-3))[0]
    assert np.array_equal(res[0]["zero_params"], res[1]["zero_params"])
    assert np.array_equal(res[0]["zero_params"], want)
    # union-compacted exchange: same numbering on both ranks, rows' sum == dense sum
    for step in range(3):
        assert np.array_equal(res[0]["union_umap"][step], res[1]["union_umap"][step])
        for r in (0, 1):
            assert np.array_equal(res[r]["union_sum"][step], res[r]["union_dense"][step])
        assert 0 < (res[0]["union_umap"][step] > 0).sum() < rec.shape[0]
