"""N > 1 host logic on CPU with the gloo backend, world_size 2 (the GPU box has one GPU):
contiguous point shards of one stream, end-of-run gather to rank 0, max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1201_0499_b200.sharding import gather_to_rank0, shard_points
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = shard_points(8, 13, 11, world, rank)          # uneven split: 6 + 7
        full = gather_to_rank0(np.ascontiguousarray(pts.view(np.float64)))
        t = torch.tensor([1.5 + rank], dtype=torch.float64)  # per-rank elapsed
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((full, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_reassemble_the_single_stream():
    import paper_1201_0499_b200 as pj
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = pj.random_points(8, 13, 11).view(np.float64)
    assert np.array_equal(full.view(np.uint64), want.view(np.uint64))
    assert tmax == 2.5
