"""Row-sharding plumbing for multi-GPU use.

Rows (b, h) are independent, so the path shards by heads: rank r of
W owns heads [h0, h1) of every batch row and only its own k_f slice; no
collective runs inside the convolution, and dk needs no reduction.  These
helpers move head shards between rank 0 and the other ranks with
torch.distributed scatter/gather (NCCL on GPUs, gloo in the CPU tests).
They contain no arithmetic of the method.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(H: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced head range of `rank` (sizes differ by at most 1)."""
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def scatter_heads(x: torch.Tensor | None, H: int, shape_bn, dtype, device, src: int = 0) -> torch.Tensor:
    """Rank `src` holds x (B, H, N); every rank returns its (B, h1-h0, N)
    contiguous shard."""
    rank, world = dist.get_rank(), dist.get_world_size()
    B, N = shape_bn
    h0, h1 = head_shard(H, rank, world)
    out = torch.empty(B, h1 - h0, N, dtype=dtype, device=device)
    if world == 1:
        out.copy_(x)
        return out
    if rank == src:
        parts = []
        for r in range(world):
            a, b = head_shard(H, r, world)
            parts.append(x[:, a:b].contiguous())
        # scatter needs equal sizes: pad to the largest shard
        hmax = max(p.shape[1] for p in parts)
        padded = [torch.nn.functional.pad(p, (0, 0, 0, hmax - p.shape[1])) for p in parts]
        buf = torch.empty(B, hmax, N, dtype=dtype, device=device)
        dist.scatter(buf, padded, src=src)
    else:
        hmax = max(head_shard(H, r, world)[1] - head_shard(H, r, world)[0] for r in range(world))
        buf = torch.empty(B, hmax, N, dtype=dtype, device=device)
        dist.scatter(buf, None, src=src)
    out.copy_(buf[:, : h1 - h0])
    return out


def gather_heads(y: torch.Tensor, H: int, dst: int = 0) -> torch.Tensor | None:
    """Inverse of scatter_heads: rank `dst` returns the full (B, H, N)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    B, hloc, N = y.shape
    if world == 1:
        return y
    hmax = max(head_shard(H, r, world)[1] - head_shard(H, r, world)[0] for r in range(world))
    buf = torch.nn.functional.pad(y, (0, 0, 0, hmax - hloc)).contiguous()
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst)
        full = torch.empty(B, H, N, dtype=y.dtype, device=y.device)
        for r in range(world):
            a, b = head_shard(H, r, world)
            full[:, a:b] = parts[r][:, : b - a]
        return full
    dist.gather(buf, None, dst=dst)
    return None
