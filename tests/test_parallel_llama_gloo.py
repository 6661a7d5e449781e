"""Multi-layer caller sharding (llama.py) on CPU with world_size-2 gloo
groups: the weight slicing (``shard_layer_weights``), the all-gather of
head-sharded attention outputs (``gather_head_blocks``, ``gather`` mode) and
the all-reduce of row-parallel partial sums (``all_reduce_partial``, ``tp``
mode) must reproduce the unsharded layer.  Attention itself is per head
(the GPU kernels); here each head's output is a fixed function of its own q
rows, which is all the sharding logic can observe."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

DM, H, F, ROWS = 64, 4, 96, 5
D = DM // H


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _mats(seed=0):
    g = torch.Generator().manual_seed(seed)
    shapes = dict(wq=(DM, DM), wk=(DM, DM), wv=(DM, DM), wo=(DM, DM), wg=(F, DM), wu=(F, DM),
                  wd=(DM, F))
    return {k: torch.randn(*s, generator=g) * 0.1 for k, s in shapes.items()}


def _layer(x, rank, world, mode):
    from paper_2310_01801_b200.parallel import (all_reduce_partial, gather_head_blocks,
                                                shard_layer_weights)

    Hl = H // world
    h0, h1 = rank * Hl, (rank + 1) * Hl
    f0, f1 = (rank * F // world, (rank + 1) * F // world) if mode == "tp" else (0, F)
    wqkv, wo, wgu, wdown = shard_layer_weights(_mats(), h0, h1, D, f0, f1, mode)
    qkv = x @ wqkv.T
    o = torch.tanh(qkv[:, : Hl * D])          # per-head stand-in for attention
    if mode == "tp":
        attn = all_reduce_partial(o @ wo.T, world)
    else:
        attn = gather_head_blocks(o, world) @ wo.T
    h = x + attn
    gu = h @ wgu.T
    Fl = f1 - f0
    m = torch.nn.functional.silu(gu[:, :Fl]) * gu[:, Fl:]
    down = m @ wdown.T
    if mode == "tp":
        down = all_reduce_partial(down, world)
    return h + down


def _worker(rank, world, port, mode, path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = torch.randn(ROWS, DM, generator=torch.Generator().manual_seed(1))
    y = _layer(x, rank, world, mode)
    gathered = [torch.empty_like(y) for _ in range(world)]
    dist.all_gather(gathered, y)
    if rank == 0:
        torch.save(torch.stack(gathered), path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["gather", "tp"])
def test_sharded_layer_equals_unsharded(tmp_path, mode):
    out = tmp_path / "y.pt"
    mp.spawn(_worker, args=(2, _free_port(), mode, str(out)), nprocs=2, join=True)
    ys = torch.load(out)
    x = torch.randn(ROWS, DM, generator=torch.Generator().manual_seed(1))
    ref = _layer(x, 0, 1, mode)
    for y in ys:   # every rank ends with the full, identical activation
        torch.testing.assert_close(y, ref, rtol=1e-5, atol=1e-5)


def test_gather_head_blocks_order_single_rank():
    from paper_2310_01801_b200.parallel import gather_head_blocks

    o = torch.arange(12.0).view(3, 4)
    assert gather_head_blocks(o, 1) is o


def test_shard_plan_splits():
    from paper_2310_01801_b200.llama import LLAMA_7B, LLAMA_65B, ShardPlan

    for cfg in (LLAMA_7B, LLAMA_65B):
        for world in (1, 2, 4, 8):
            seen_h, seen_f = [], []
            for r in range(world):
                p = ShardPlan(r, world, "tp")
                h0, h1 = p.heads(cfg.n_heads)
                f0, f1 = p.ffn(cfg.ffn)
                seen_h += range(h0, h1)
                seen_f += range(f0, f1)
                assert (f1 - f0) % 8 == 0  # 16-byte rows for the bf16 caller kernels
            assert seen_h == list(range(cfg.n_heads)) and seen_f == list(range(cfg.ffn))
