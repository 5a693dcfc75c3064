"""Multi-GPU sharding of independent MTGP32 streams and of stat-test campaigns.

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
    t = torch.tensor(rows, dtype=torch.int64, device=device).reshape(-1, 4)
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        parts = [t]
    else:
        # ranks may own different stream counts (a balanced split of n sets over any world size):
        # gather the counts, pad to the largest, gather, trim
        world = dist.get_world_size()
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
        counts = [torch.empty_like(n) for _ in range(world)]
        dist.all_gather(counts, n)
        counts = [int(c.item()) for c in counts]
        pad = torch.zeros((max(counts), 4), dtype=torch.int64, device=device)
        pad[:t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        parts = [p[:c] for p, c in zip(parts, counts)]
    out: List[Cksum] = []
    for p in parts:
        for lo, hi, x, w in p.cpu().tolist():
            out.append(((hi << 32) | lo, x, w))
    return out


def status_range(n_statuses: int, rank: int, world: int) -> range:
    """Contiguous, balanced status-index range of `rank` for a campaign over n_statuses
    (strong scaling: the campaign's cells are fixed, split across ranks)."""
    base, extra = divmod(n_statuses, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def run_grid_distributed(statuses: Sequence, seeds: Sequence[int], specs: Sequence, runner=None, **kw):
    """The sieve's campaign grid (sieve.cpp:116-183) over every rank's GPU: rank r runs the
    cells of its status range on its own device (stattests.run_grid), and rank 0 returns all
    rows in the reference's (status, seed, test) order -- the same report for any world size,
    as run_grid is for any worker count. Other ranks return []. The row gather is the only
    collective (all_gather_object: NCCL / gloo). `runner` replaces stattests.run_grid (tests)."""
    import torch.distributed as dist

    from . import stattests
    dist_on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank() if dist_on else 0
    world = dist.get_world_size() if dist_on else 1
    mine = status_range(len(statuses), rank, world)
    rows = []
    if runner is None:
        import os
        kw.setdefault("device", int(os.environ.get("LOCAL_RANK", "0")))  # each rank its own GPU
    if len(mine):
        run = runner or stattests.run_grid
        ids = kw.pop("status_ids", None) or [str(i) for i in range(len(statuses))]
        rows = run([statuses[i] for i in mine], seeds, specs, status_ids=[ids[i] for i in mine], **kw)
        for r in rows:
            r.status_index += mine.start
    if world == 1:
        return rows
    parts = [None] * world
    dist.all_gather_object(parts, rows)
    if rank != 0:
        return []
    return [r for part in parts for r in part]
