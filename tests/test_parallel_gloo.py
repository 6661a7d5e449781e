"""The N>1 path's host logic on CPU with world_size-2 gloo process groups:
shard assignment covers every head exactly once, the per-rank profiles
gather into the global profile, and per-shard results equal the unsharded
run (heads are independent, so sharding changes nothing).  The per-shard
compute here is the CPU oracle standing in for each rank's GPU."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_01801_b200.parallel import (batch_shard, gather_profile, head_shard,
                                            profile_csv, profile_rows)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_partition_the_grid():
    for B, H, world in [(8, 32, 2), (8, 32, 8), (1, 8, 3), (4, 32, 8), (3, 5, 4)]:
        for fn in (head_shard, batch_shard):
            seen = []
            for r in range(world):
                seen += fn(B, H, world, r).heads
            assert sorted(seen) == [(b, h) for b in range(B) for h in range(H)]
            assert len(seen) == len(set(seen))


def _oracle_profile(w, heads):
    from oracle import akv_oracle as O
    from paper_2310_01801_b200.workloads import class_lut

    fam = O.default_family(w.r_l, w.r_f)
    lut = class_lut()
    out = []
    for b, h in heads:
        q, k, v = (x.astype(np.float64) for x in w.head_qkv(b, h))
        cls = lut[w.tokens(b)].astype(np.int64)
        r = O.profile_head(q[:w.N], k[:w.N], v[:w.N], cls, w.slopes[h], w.sinks[h], fam,
                           [w.thresholds[0]])
        out.append((O.format_member(fam[r.choice[0]]), r.recoveries[r.choice[0]],
                    r.costs[r.choice[0]]))
    return out


def _worker(rank, world, port, mode, result_path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests"), os.path.join(root, "tests", "golden")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from cases import _c0_sink

    w = _c0_sink()
    w.B = 2
    shard = (head_shard if mode == "head" else batch_shard)(w.B, w.H, world, rank)
    local = _oracle_profile(w, shard.heads)
    rows = profile_rows(shard, *zip(*local)) if local else []
    merged = gather_profile(rows)
    if rank == 0:
        with open(result_path, "w") as f:
            f.write(profile_csv(merged))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["head", "batch"])
def test_sharded_profile_equals_unsharded(tmp_path, mode):
    from cases import _c0_sink

    out = tmp_path / "profile.csv"
    mp.spawn(_worker, args=(2, _free_port(), mode, str(out)), nprocs=2, join=True)
    w = _c0_sink()
    w.B = 2
    heads = [(b, h) for b in range(w.B) for h in range(w.H)]
    full = _oracle_profile(w, heads)
    expect = profile_csv(sorted((b, h, p, float(r), int(c))
                                for (b, h), (p, r, c) in zip(heads, full)))
    assert out.read_text() == expect


def test_lpt_assignment_balances_ragged_heads():
    from paper_2310_01801_b200.parallel import assignment_loads, lpt_assignment

    rng = np.random.default_rng(0)
    # config-1-like: most heads full (N + D), a few compressed ones
    costs = [1536] * 240 + list(rng.integers(100, 900, size=16))
    for world in (1, 2, 4, 8):
        owned = lpt_assignment(costs, world)
        assert sorted(i for o in owned for i in o) == list(range(len(costs)))
        loads = assignment_loads(costs, owned)
        assert max(loads) - min(loads) <= max(costs)
        contiguous = [sum(costs[r * len(costs) // world:(r + 1) * len(costs) // world])
                      for r in range(world)]
        assert max(loads) <= max(contiguous)
    assert lpt_assignment([5, 3, 3, 2, 2, 1], 2) == [[0, 3, 5], [1, 2, 4]]
