"""Multi-GPU sharding of the PRNGD path.

Streams are independent and counter-addressed (R6), so the path shards by disjoint
stream-id ranges with NO communication on the generation path: rank r of R generates global
streams [stream_begin_r, stream_begin_r + n_r) into its own HBM; its outputs are the contiguous
slice [stream_begin_r * n_per_stream, ...) of the logical global array.  The only exchange is
the all-reduce of the fused consumer's statistics (65536-bin int64 histogram, 4 FP64 power sums,
int64 count), done with torch.distributed (NCCL over NVLink on B200, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable

WEAK, STRONG = "weak", "strong"


def shard_range(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank r's streams when N global streams are split over R ranks."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * n_global // world, (rank + 1) * n_global // world


def shard_params(p: dict, rank: int, world: int, mode: str = STRONG) -> dict:
    """Parameters of rank r's shard.

    STRONG: p["n_streams"] is the global stream count, split over the ranks.
    WEAK:   p["n_streams"] is the per-rank count; rank r starts at stream_begin + r * n_streams.
    """
    q = dict(p)
    base = p.get("stream_begin", 0)
    if mode == STRONG:
        lo, hi = shard_range(p["n_streams"], rank, world)
        q["stream_begin"], q["n_streams"] = base + lo, hi - lo
    elif mode == WEAK:
        q["stream_begin"] = base + rank * p["n_streams"]
    else:
        raise ValueError(mode)
    return q


def allreduce_stats(hist, pw, count, group=None, deterministic: bool = False):
    """Sum the consumer statistics over ranks, in place.  hist and count are int64 (exact in
    any order); the FP64 power sums are order-dependent, so `deterministic=True` all-gathers the
    per-rank partials and adds them in rank order (bit-identical for any NCCL algorithm)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return hist, pw, count
    dist.all_reduce(hist, group=group)
    dist.all_reduce(count, group=group)
    if deterministic:
        parts = [torch.empty_like(pw) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, pw, group=group)
        acc = torch.zeros_like(pw)
        for t in parts:
            acc += t
        pw.copy_(acc)
    else:
        dist.all_reduce(pw, group=group)
    return hist, pw, count


def generate_sharded(p: dict, mode: str = STRONG, consume: bool = False, write: bool = True,
                     group=None, deterministic: bool = False,
                     local: Callable | None = None):
    """Run this rank's shard and (if `consume`) all-reduce the statistics.

    Returns (local_outputs_or_None, hist, pw, count, shard_params).  `local` replaces the
    per-rank generator (the CPU tests pass the oracle; the product path is the CUDA library)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    q = shard_params(p, rank, world, mode)
    if local is not None:
        out, hist, pw, count = local(q, consume, write)
    else:
        from . import prngd as P
        g = P.Generator(**q)
        out = torch.empty(g.shape, dtype=torch.float64, device="cuda") if write else None
        if consume:
            out, hist, pw, count = g.generate_consume(out)
        else:
            g.generate(out)
            hist = pw = count = None
    if consume:
        allreduce_stats(hist, pw, count, group=group, deterministic=deterministic)
    return out, hist, pw, count, q
