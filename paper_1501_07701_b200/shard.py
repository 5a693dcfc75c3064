"""Multi-GPU sharding of independent MTGP32 streams.

Streams are independent by parameterization, so the path shards
with no data-path collective: rank r owns a contiguous range of parameter-set IDs and generates
them on its own GPU. The only collective is the final gather of per-stream checksums
{sum64, xor32, words} (16-24 B per stream) -- NCCL all_gather on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .tables import MtgpParams, sets_for

Cksum = Tuple[int, int, int]  # (sum64, xor32, words)


def set_range(rank: int, sets_per_rank: int) -> range:
    """Global parameter-set IDs owned by `rank` (weak scaling: fixed sets per rank)."""
    return range(rank * sets_per_rank, (rank + 1) * sets_per_rank)


def sets_for_rank(mexp: int, sets_per_rank: int, rank: int) -> List[MtgpParams]:
    """The rank's parameter sets: certified cuRAND sets first (11213), then synthetic ones."""
    return sets_for(mexp, sets_per_rank, first=rank * sets_per_rank)


def gather_checksums(local: Sequence[Cksum], device=None) -> List[Cksum]:
    """All-gather every rank's per-stream checksums; returns them in global set-ID order.

    sum64 is carried as two int64 halves (torch has no uint64 collectives)."""
    import torch
    import torch.distributed as dist

    rows = [[c[0] & 0xFFFFFFFF, (c[0] >> 32) & 0xFFFFFFFF, c[1] & 0xFFFFFFFF, c[2]] for c in local]
    t = torch.tensor(rows, dtype=torch.int64, device=device)
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        parts = [t]
    else:
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, t)
    out: List[Cksum] = []
    for p in parts:
        for lo, hi, x, w in p.cpu().tolist():
            out.append(((hi << 32) | lo, x, w))
    return out
