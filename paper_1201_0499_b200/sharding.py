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


def gather_to_rank0(local: np.ndarray, group=None):
    """End-of-run gather of per-rank results (optional, off the hot path): rank 0 receives the
    concatenation in rank order. Uses torch.distributed (gloo on CPU tensors, NCCL on CUDA)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(local)
    ws = dist.get_world_size(group)
    sizes = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(ws)]
    dist.all_gather(sizes, torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device), group=group)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(ws)]
    dist.all_gather(parts, pad, group=group)
    if dist.get_rank(group) != 0:
        return None
    return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)]).cpu().numpy()
