"""Point-batch sharding across ranks: contiguous ranges of one global point
stream, system replicated, no collective on the data path. Host-side logic only."""
from __future__ import annotations

import numpy as np

from ._lib import check, lib


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, last) of rank's contiguous shard; sizes differ by at most one point."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    return total * rank // world, total * (rank + 1) // world


def shard_points(n: int, total: int, seed: int, world: int, rank: int) -> np.ndarray:
    """This rank's shard of random_points(n, total, seed) as complex128 [count, n], generated
    without materialising the other ranks' points."""
    a, b = shard_range(total, world, rank)
    out = np.empty((b - a, n, 2), np.float64)
    check(lib().pj_random_points_range(n, a, b - a, seed, out.ctypes.data))
    return out.view(np.complex128).reshape(b - a, n)


def gather_to_rank0(local, group=None, out=None):
    """End-of-run gather of per-rank results to rank 0 (off the hot path): rank 0
    returns the concatenation of every rank's rows in rank order, the other ranks None.

    Point to point: each rank r > 0 sends its shard once (isend), rank 0 posts one irecv per
    source straight into its slice of the output (batch_isend_irecv, so the transfers overlap) —
    the bytes that cross the links are the other ranks' shards, once (an all_gather would deliver
    every shard to every rank: N times the traffic). `local` is a torch tensor (CUDA for NCCL,
    CPU for gloo) or a numpy array (sent as a CPU tensor); shards may differ in length by any
    amount (the row counts are exchanged first). `out` (rank 0, optional): a preallocated tensor
    of the full shape, so the timed region holds no allocation."""
    import numpy as np
    import torch
    import torch.distributed as dist
    as_numpy = isinstance(local, np.ndarray)
    t = torch.from_numpy(np.ascontiguousarray(local)) if as_numpy else local.contiguous()
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(ws)]
    dist.all_gather(sizes, cnt, group=group)  # ws integers: the shard lengths
    rows = [int(x.item()) for x in sizes]
    if rank != 0:
        if rows[rank]:
            dist.batch_isend_irecv([dist.P2POp(dist.isend, t, 0, group=group)])[0].wait()
        return None
    total = sum(rows)
    full = out if out is not None else torch.empty((total,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if tuple(full.shape) != (total,) + tuple(t.shape[1:]):
        raise ValueError("gather_to_rank0: output buffer has the wrong shape")
    full[: rows[0]].copy_(t)
    ops, at = [], rows[0]
    for r in range(1, ws):
        if rows[r]:
            ops.append(dist.P2POp(dist.irecv, full[at: at + rows[r]], r, group=group))
        at += rows[r]
    for w in (dist.batch_isend_irecv(ops) if ops else []):
        w.wait()
    return full.numpy() if as_numpy else full
