"""Contiguous-range sharding of a pair list over ranks + the final stats reduce.

Every triangle pair is independent, so rank r of W owns the
contiguous range [r*n//W, (r+1)*n//W) and computes it with no data-path
communication.  The only exchange is the final reduction of the tc_stats
record: a SUM of the six int64 tallies and a MIN of the fp64 minimum
distance, done as ONE all-gather of the 56-byte records enqueued on the
current stream (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for the
tests) followed by the sum / min on the device.  Integer sums and the
min are order-independent, so results are bit-identical for any W.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

N_COUNTS = 6  # tc_stats int64 words before min_distance


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """(start, count) of rank's contiguous share of n_total pairs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def allreduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """In-place all-reduce of a tc_stats tensor (7 x int64 words, last = fp64 bits).

    One collective: every rank's 56-byte record is all-gathered (NCCL on the
    current stream for CUDA tensors, gloo on CPU), then the six tallies are
    summed and the minimum distance taken on the device -- integer sums and
    the min are order-independent, so the result is bit-identical for any W.
    """
    if stats.dtype != torch.int64 or stats.numel() != N_COUNTS + 1:
        raise ValueError("expected the 7-word int64 tc_stats tensor")
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return stats
    world = dist.get_world_size(group)
    if stats.is_cuda and dist.get_backend(group) == "nccl":
        buf = torch.empty(world * (N_COUNTS + 1), dtype=torch.int64, device=stats.device)
        dist.all_gather_into_tensor(buf, stats, group=group)
    else:
        # gloo (CPU tests, or the one-GPU functional test of the N-rank path)
        host = stats.detach().cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        buf = torch.cat(parts)
    buf = buf.view(world, N_COUNTS + 1)
    red = torch.empty(N_COUNTS + 1, dtype=torch.int64, device=buf.device)
    red[:N_COUNTS] = buf[:, :N_COUNTS].sum(0)
    red[N_COUNTS:].view(torch.float64).copy_(buf[:, N_COUNTS:].contiguous().view(torch.float64).min().reshape(1))
    stats.copy_(red)
    return stats


def stats_dict(stats: torch.Tensor) -> dict:
    h = stats.detach().cpu()
    names = ("iterative", "comparison", "fallback", "degenerate", "contacts", "intersecting")
    d = {k: int(h[i]) for i, k in enumerate(names)}
    d["min_distance"] = float(h[N_COUNTS:].view(torch.float64)[0])
    return d
