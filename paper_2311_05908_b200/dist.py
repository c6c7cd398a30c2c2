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


def head_shard(H: int, rank: int, world: int, align: int = 2) -> tuple[int, int]:
    """Contiguous, balanced head range of `rank`, in units of `align` heads
    (shard sizes differ by at most 2 * align - 1).  The default align = 2 keeps
    the head pairs (2j, 2j + 1) the k_f precompute transforms together (two
    real filters as one complex FFT) inside one shard, so a shard's k_f --
    and hence its y, du, dw, dv and dk -- is bitwise the corresponding slice
    of the unsharded call."""
    G = (H + align - 1) // align  # groups of `align` heads (the last may be short)
    base, extra = divmod(G, world)
    g0 = rank * base + min(rank, extra)
    g1 = g0 + base + (1 if rank < extra else 0)
    return min(H, g0 * align), min(H, g1 * align)


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
