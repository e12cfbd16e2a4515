"""Multi-GPU sharding of independent planning units.

Windows of *different* scenarios / traces / overhead-sweep points are
independent, so each rank plans a contiguous block of them with no
collective on the data path. The only exchange is the final combine of the
per-shard best (objective, plan owner): an all-reduce(max) on the objective's
IEEE bits (Goodput is never negative, so the bit pattern orders like the
value), then an all-reduce(min) of the owning shard among the maxima — the
deterministic tie-break toward the lowest shard index. Over NCCL this runs on
NVLink; the same code runs over gloo for the CPU tests.
"""
from __future__ import annotations

import struct


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous block [lo, hi) of n_items owned by rank."""
    lo = n_items * rank // world
    hi = n_items * (rank + 1) // world
    return lo, hi


def objective_key(objective: float) -> int:
    """int64 whose order matches the (non-negative) objective's order."""
    if objective != objective or objective < 0:
        raise ValueError("objective must be a non-negative number")
    return struct.unpack("<q", struct.pack("<d", float(objective)))[0]


def key_objective(key: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(key)))[0]


def combine_best(objective: float, rank: int, world: int, device="cpu"):
    """Returns (best objective, owning rank) over all ranks."""
    import torch
    import torch.distributed as dist
    key = torch.tensor([objective_key(objective)], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(key, op=dist.ReduceOp.MAX)
    best = int(key.item())
    owner = torch.tensor([rank if objective_key(objective) == best else world], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(owner, op=dist.ReduceOp.MIN)
    return key_objective(best), int(owner.item())


def gather_rows(rows, world: int, device="cpu"):
    """All-gather of each rank's int64 rows (a list of equal-width lists; ranks may
    hold different row counts). Returns the rows of every rank, rank-major. Over
    NCCL this is two all_gathers on NVLink (counts, then the padded rows)."""
    import torch
    import torch.distributed as dist
    width = len(rows[0]) if rows else 0
    if world == 1:
        return [list(map(int, r)) for r in rows]
    meta = torch.tensor([len(rows), width], dtype=torch.int64, device=device)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    n_max = max(int(m[0]) for m in metas)
    width = max(int(m[1]) for m in metas)
    buf = torch.zeros((max(1, n_max), max(1, width)), dtype=torch.int64, device=device)
    if rows:
        buf[:len(rows), :len(rows[0])] = torch.tensor(rows, dtype=torch.int64, device=device)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    out = []
    for m, b in zip(metas, bufs):
        out.extend(b[:int(m[0]), :width].tolist())
    return out
