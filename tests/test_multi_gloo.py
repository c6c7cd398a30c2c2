"""world_size-2 gloo tests (CPU) of the row-sharding plumbing: head shards
scattered from rank 0, convolved independently (here by the oracle, since
there is no GPU), gathered back -- bitwise identical to the unsharded result
because rows are independent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_05908_b200.dist import gather_heads, head_shard, scatter_heads


def test_head_shard_balanced_and_covering():
    for H in (1, 5, 768, 769):
        for W in (1, 2, 3, 8):
            ranges = [head_shard(H, r, W) for r in range(W)]
            assert ranges[0][0] == 0 and ranges[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 3  # balanced in 2-head groups, the last may be short
            # shards start at even heads (k_f head pairs stay together)
            assert all(a % 2 == 0 or a == H for a, _ in ranges)
            assert [head_shard(H, r, W, align=1) for r in range(W)][-1][1] == H


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import oracle as orc
        B, H, N = 3, 5, 64
        k = synth.decay_filters(0, H, N)
        x = torch.tensor(synth.signal(0, "u", B, H, N)) if rank == 0 else None
        xs = scatter_heads(x, H, (B, N), torch.float64, "cpu")
        h0, h1 = head_shard(H, rank, world)
        ys = torch.tensor(orc.conv_fwd(xs.numpy(), k[h0:h1]))
        full = gather_heads(ys, H)
        if rank == 0:
            ref = orc.conv_fwd(synth.signal(0, "u", B, H, N), k)
            q.put(bool(np.array_equal(full.numpy(), ref)))
    finally:
        dist.destroy_process_group()


def test_scatter_conv_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
