"""Sharding of the hot path across GPUs (one process per GPU).

Every (batch row, head) is independent in profiling, compaction and decode
(reference: per-head loops engine.py:182-199, 236-259, 310-349, no
cross-head reads), so the path partitions with no data-path collective:

* ``head_shard``: contiguous head blocks per rank (H/P heads x all batch
  rows), the column-parallel split a multi-layer model would use;
* ``batch_shard``: contiguous batch rows per rank (independent sessions,
  what bench.py's weak-scaling run does).

The only communication is host-side bookkeeping: gathering the per-rank
profile rows (HeadProfile CSV) and, for verification, the outputs.  The
multi-layer configs' all-gather of attention outputs is SURVEY §8(f)
'next' and is not implemented here.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def heads(self) -> list:
        """Global (b, h) pairs owned by this rank, in flattened g order."""
        return [(b, h) for b in range(self.b0, self.b1) for h in range(self.h0, self.h1)]


def _split(n: int, world: int, rank: int) -> tuple:
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def head_shard(B: int, H: int, world: int, rank: int) -> Shard:
    """Contiguous head block [h0, h1) of every batch row for ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    h0, h1 = _split(H, world, rank)
    return Shard(rank, world, 0, B, h0, h1)


def batch_shard(B: int, H: int, world: int, rank: int) -> Shard:
    """Contiguous batch rows [b0, b1) (all heads) for ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    b0, b1 = _split(B, world, rank)
    return Shard(rank, world, b0, b1, 0, H)


def profile_rows(shard: Shard, policies, recoveries, costs) -> list:
    """Per-head profile rows (b, h, policy string, recovery, cost) of a shard's
    local results, keyed by global (b, h) for gathering."""
    rows = []
    for (b, h), pol, rec, cost in zip(shard.heads, policies, recoveries, costs):
        rows.append((b, h, str(pol), float(rec), int(cost)))
    return rows


def gather_profile(rows: list, group=None) -> list:
    """All-gather the ranks' profile rows (host objects; gloo or nccl group)
    and return them sorted by (b, h): the global profile."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return sorted(rows)
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, rows, group=group)
    merged = sorted(r for part in out for r in part)
    keys = [(r[0], r[1]) for r in merged]
    if len(set(keys)) != len(keys):
        raise RuntimeError("overlapping shards: a head was profiled by two ranks")
    return merged


def profile_csv(rows: list) -> str:
    """HeadProfile-style CSV (profiler.py:206-214) with (b, h) as (layer, head)."""
    lines = ["layer,head,policy,recovery,cost_tokens"]
    lines += [f"{b},{h},{p},{rec!r},{c}" for b, h, p, rec, c in rows]
    return "\n".join(lines) + "\n"
