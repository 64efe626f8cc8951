"""Slice-sharded data parallelism, host side.

One process per GPU, each holding a full Gaussian replica in its session. In
step s, rank r renders slice ``schedule[(s * world + r) % len(schedule)]``
(the fit loop's slices, optimize.hpp:385-395, dealt round-robin), so the
world renders ``world`` distinct slices per step, and every rank knows all of
the step's poses (``step_slices``).

The exchange (``gpk_train_step_dp``, csrc/dp.cu) is union-compacted:
gradients are exactly zero outside the union of the step's survivors, so each
rank evaluates the cull of every pose of the step in its own cull pass, numbers
the union of candidates identically on every rank (row = how many union
members precede the Gaussian in index order: ``union_rows``), writes its
survivors' gradients into those rows and ONE grouped ``ncclAllReduce`` sums
the rows; every rank then runs the scheduled Adam on all Gaussians from the
summed rows, so the replicas stay bitwise equal. ``pack_rows`` /
``unpack_rows`` restate the device layout for the CPU tests. The dense
all-reduce (``gpk_allreduce_grads``) and the reduce-scatter + sharded Adam +
all-gather step (``gpk_train_step`` under a communicator) remain.

The NCCL communicator is created by the C-ABI (``gpk_comm_init``) from an
``ncclUniqueId`` that rank 0 generates and the launcher's process group
(torch.distributed, any backend) broadcasts.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

NCCL_ID_BYTES = 128


def slice_for(step: int, rank: int, world: int, n_slices: int) -> int:
    """Index into the slice schedule rendered by ``rank`` in ``step``."""
    if not (0 <= rank < world) or n_slices <= 0:
        raise ValueError("slice_for: need 0 <= rank < world and a non-empty schedule")
    return (step * world + rank) % n_slices


def step_slices(step: int, world: int, n_slices: int) -> list[int]:
    """All slices the world renders in ``step`` (rank order)."""
    return [slice_for(step, r, world, n_slices) for r in range(world)]


def native_unique_id() -> bytes:
    """ncclGetUniqueId through the C-ABI (the library loads NCCL lazily)."""
    from . import _native as N

    buf = (C.c_char * NCCL_ID_BYTES)()
    N.check(N.lib.gpk_nccl_get_unique_id(buf))
    return bytes(buf)


def exchange_unique_id(rank: int, group=None, make_id: Callable[[], bytes] | None = None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist

    obj = [(make_id or native_unique_id)() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != NCCL_ID_BYTES:
        raise RuntimeError("exchange_unique_id: malformed ncclUniqueId")
    return bytes(uid)


def init_grad_comm(session, rank: int, world: int, group=None) -> None:
    """Create the session's NCCL communicator (one per session / GPU)."""
    from . import _native as N

    uid = exchange_unique_id(rank, group)
    buf = (C.c_char * NCCL_ID_BYTES).from_buffer_copy(uid)
    N.check(N.lib.gpk_comm_init(session.handle, int(world), int(rank), buf))


def allreduce_grads(session) -> None:
    """Sum the dense gradient planes over all ranks, in place, on the session stream."""
    from . import _native as N

    N.check(N.lib.gpk_allreduce_grads(session.handle))


def max_over_ranks(values: Sequence[float], device=None, group=None) -> list[float]:
    """Element-wise max across ranks (multi-GPU timings are reported as the max)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.tolist()]


def union_rows(mask):
    """Row numbering of the union (csrc/dp.cu k_union_map): umap[i] = 1 + the
    number of union members with a smaller index, 0 outside the union."""
    import numpy as np

    m = np.asarray(mask, bool)
    rows = np.cumsum(m, dtype=np.int64) - 1
    return np.where(m, rows + 1, 0).astype(np.uint32)


def pack_rows(grads, umap):
    """A rank's (n, 11) gradient as the union rows (M, 11): row umap[i]-1 holds
    Gaussian i's gradient (zero for union members that are not its survivors)."""
    import numpy as np

    umap = np.asarray(umap, np.int64)
    grads = np.asarray(grads)
    M = int((umap > 0).sum())
    rows = np.zeros((M, 11), grads.dtype)
    sel = umap > 0
    rows[umap[sel] - 1] = grads[sel]
    return rows


def unpack_rows(rows, umap):
    """The summed union rows back to an (n, 11) gradient (zero outside)."""
    import numpy as np

    umap = np.asarray(umap, np.int64)
    rows = np.asarray(rows)
    out = np.zeros((umap.size, 11), rows.dtype)
    sel = umap > 0
    out[sel] = rows[umap[sel] - 1]
    return out
