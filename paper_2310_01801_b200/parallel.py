"""Sharding of the hot path across GPUs (one process per GPU).

Every (batch row, head) is independent in profiling, compaction and decode
(reference: per-head loops engine.py:182-199, 236-259, 310-349, no
cross-head reads), so the path partitions with no data-path collective:

* ``head_shard``: contiguous head blocks per rank (H/P heads x all batch
  rows), the column-parallel split a multi-layer model would use;
* ``batch_shard``: contiguous batch rows per rank (independent sessions,
  what bench.py's weak-scaling run does).

For the single-layer configs the only communication is host-side
bookkeeping: gathering the per-rank profile rows (HeadProfile CSV) and, for
verification, the outputs.  The multi-layer caller (``llama.py``, configs
2/3) adds the data-path collectives below: the all-gather of head-sharded
attention outputs (``gather_head_blocks``) and, in tensor-parallel mode,
the all-reduce of row-parallel partial sums (``all_reduce_partial``); the
weight slicing both modes use is ``shard_layer_weights``.
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


def shard_layer_weights(mats: dict, h0: int, h1: int, d: int, f0: int, f1: int, mode: str):
    """Local weights of one decoder layer from its full matrices
    (``wq, wk, wv, wo`` [dm, dm], ``wg, wu`` [F, dm], ``wd`` [dm, F]):

    * wqkv [3*Hl*d, dm] - rows of heads [h0, h1) of q, k and v (column
      parallel: each rank projects only its own heads);
    * wo - full [dm, H*d] in ``gather`` mode (outputs are all-gathered
      first), the columns of the local heads [dm, Hl*d] in ``tp`` mode
      (row parallel, partial sums all-reduced);
    * wgu [2*Fl, dm] - gate rows [f0, f1) then up rows [f0, f1);
    * wdown [dm, Fl] - columns [f0, f1).
    """
    hs = slice(h0 * d, h1 * d)
    fs = slice(f0, f1)
    wqkv = _cat([mats["wq"][hs], mats["wk"][hs], mats["wv"][hs]])
    wo = mats["wo"] if mode != "tp" else mats["wo"][:, hs].contiguous()
    wgu = _cat([mats["wg"][fs], mats["wu"][fs]])
    wdown = mats["wd"][:, fs].contiguous()
    return wqkv, wo, wgu, wdown


def _cat(parts):
    import torch

    return torch.cat(parts).contiguous()


def gather_head_blocks(o, world: int, group=None):
    """All-gather head-sharded attention outputs: ``o`` [rows, Hl*d] on every
    rank -> [rows, world*Hl*d] with rank r's block at columns
    [r*Hl*d, (r+1)*Hl*d) - the global head order, since rank r owns the
    contiguous heads [r*Hl, (r+1)*Hl).  NCCL uses one
    all_gather_into_tensor; other backends (gloo, CPU tests) a list gather."""
    if world == 1:
        return o
    import torch
    import torch.distributed as dist

    o = o.contiguous()
    rows = o.shape[0]
    if o.is_cuda:
        buf = torch.empty(world, rows, o.shape[1], dtype=o.dtype, device=o.device)
        dist.all_gather_into_tensor(buf, o, group=group)
        return buf.permute(1, 0, 2).reshape(rows, -1)
    parts = [torch.empty_like(o) for _ in range(world)]
    dist.all_gather(parts, o, group=group)
    return torch.cat(parts, dim=1)


def all_reduce_partial(x, world: int, group=None):
    """Sum row-parallel partial products over the ranks (in place)."""
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(x, group=group)
    return x


def lpt_assignment(costs, world: int) -> list:
    """Longest-processing-time assignment of heads to ranks:
    after profiling, a head's decode cost is its live-row count (kept + D);
    heads go largest first to the least-loaded rank.  Returns, per rank, the
    sorted head indices it owns; ties between ranks go to the lower rank, so
    every rank computes the same assignment from the same costs."""
    import heapq

    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(world)]
    owned = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        owned[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(o) for o in owned]


def assignment_loads(costs, owned) -> list:
    return [sum(costs[i] for i in o) for o in owned]
