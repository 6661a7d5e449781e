"""Sharded workloads (bench.py's multi-GPU split) on CPU: a rank's rows /
heads regenerate exactly its slice of the whole seeded workload, and the
shards of every world size cover each (batch row, head) once."""

import numpy as np
import pytest

from paper_2310_01801_b200.parallel import batch_shard, head_shard
from paper_2310_01801_b200.workloads import config1, config4


def test_row_and_head_slices_equal_the_whole():
    w = config1(seed=1, N=12, D=3)
    s = w.rows(2, 6).heads(5, 13)
    assert (s.B, s.H) == (4, 8)
    np.testing.assert_array_equal(s.sinks, w.sinks[5:13])
    np.testing.assert_array_equal(s.slopes, w.slopes[5:13])
    for b in range(s.B):
        np.testing.assert_array_equal(s.tokens(b), w.tokens(b + 2))
        for h in (0, 7):
            for x, y in zip(s.head_qkv(b, h), w.head_qkv(b + 2, h + 5)):
                np.testing.assert_array_equal(x, y)
    q, _, _ = s.qkv()
    qa, _, _ = w.qkv()
    np.testing.assert_array_equal(q, qa[2:6, 5:13])


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_bench_shards_cover_the_workload(world):
    w1, w4 = config1(N=8, D=1), config4(N=8, D=1)
    rows = [r for k in range(world) for r in range(batch_shard(w1.B, w1.H, world, k).b0,
                                                   batch_shard(w1.B, w1.H, world, k).b1)]
    assert rows == list(range(w1.B))
    heads = [h for k in range(world) for h in range(head_shard(w4.B, w4.H, world, k).h0,
                                                    head_shard(w4.B, w4.H, world, k).h1)]
    assert heads == list(range(w4.H))


def test_bad_slices_raise():
    w = config1(N=8, D=1)
    with pytest.raises(ValueError):
        w.rows(3, 3)
    with pytest.raises(ValueError):
        w.heads(0, 33)
