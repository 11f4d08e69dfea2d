"""Host-side plumbing of the multi-GPU path (BASELINE.json north_star s7:
"the matrix is row-partitioned by non-zero balance across the GPUs of one
8xB200 box: each GPU holds the full x, and the y slices are all-gathered with
NCCL over NVLink for iterated SpMV").

Only bookkeeping lives here -- every byte of the data path (the local SpMV and
the all-gather of the y slices) runs in libsable.so (sable_spmv_allgather /
sable_spmv_iterate).  These helpers are what the bench and the tests use to
set a run up: the NCCL unique id exchange over torch.distributed, and the row
ranges of every rank, derived from the block-row bounds that
sable_shard_bounds computes (the same function the inspector calls).
"""
from __future__ import annotations

import numpy as np

from . import sable


def block_row_weights(nbr: int, rpntr, tile_area_per_br, rem_per_row) -> np.ndarray:
    """Per block row a: W_a = sum of its dense-tile areas + the remainder
    non-zeros of its rows ("non-zero balance" read as stored entries
    streamed)."""
    rpntr = np.asarray(rpntr, np.int64)
    rem = np.asarray(rem_per_row, np.int64)
    cs = np.concatenate([[0], np.cumsum(rem)])
    rem_br = cs[rpntr[1:]] - cs[rpntr[:-1]]
    return np.asarray(tile_area_per_br, np.int64)[:nbr] + rem_br


def shard_bounds(weights, world: int) -> np.ndarray:
    """Block-row bounds of every rank: 0 = b0 <= ... <= b_world = nbr
    (sable_shard_bounds: boundary k = the first block row whose prefix weight
    reaches k * total / world)."""
    return sable.sable_shard_bounds(np.ascontiguousarray(weights, np.int64), world)


def row_ranges(rpntr, bounds) -> list[tuple[int, int]]:
    """(row_begin, row_end) of every rank for block-row bounds."""
    rpntr = np.asarray(rpntr, np.int64)
    return [(int(rpntr[bounds[q]]), int(rpntr[bounds[q + 1]])) for q in range(len(bounds) - 1)]


def broadcast_nccl_id(rank: int, group=None) -> bytes:
    """Rank 0 creates the ncclUniqueId (inside libsable.so) and broadcasts its
    128 bytes over the torch.distributed process group."""
    import torch.distributed as dist

    obj = [sable.sable_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
