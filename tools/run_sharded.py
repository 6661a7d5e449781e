"""Single-layer configs (0/1/4) sharded over the GPUs of one box, one process
per GPU (BASELINE config 4 "at 1/2/4/8 GPUs by head
sharding"): every rank generates and runs only its shard - a contiguous
head block of every batch row (``--shard head``, strong scaling: the job's
work is fixed) or a block of batch rows (``--shard batch``) - with no
data-path collective.  The ranks' profile rows are gathered into the global
HeadProfile CSV (its SHA-1 is printed: identical for every world size), and
times are the max over ranks of CUDA-event intervals.

    python tools/run_sharded.py c4 --shard head                      # 1 GPU
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \\
        --master-addr 127.0.0.1 --master-port 29633 tools/run_sharded.py c4 --shard head

AKV_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 over gloo (a code-path
check on a one-GPU box; its times are not measurements).
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_01801_b200 import (ProfilerConfig, decode_step_tensors,  # noqa: E402
                                   encode_prompt_tensors)
from paper_2310_01801_b200.parallel import (batch_shard, gather_profile, head_shard,  # noqa: E402
                                            profile_csv, profile_rows)
from paper_2310_01801_b200.workloads import CONFIGS, class_lut  # noqa: E402


def shard_inputs(w, shard, dev):
    """q/k/v [Bl, Hl, N+D, d] and classes [Bl, N+D] of the shard only (every
    head is generated from its own seeded stream)."""
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    bs, hs = range(shard.b0, shard.b1), range(shard.h0, shard.h1)
    shape = (len(bs), len(hs), w.total_len, w.d)
    q, k, v = (torch.empty(shape, dtype=dt, device=dev) for _ in range(3))
    for i, b in enumerate(bs):
        for j, h in enumerate(hs):
            hq, hk, hv = w.head_qkv(b, h)
            q[i, j].copy_(torch.from_numpy(hq))
            k[i, j].copy_(torch.from_numpy(hk))
            v[i, j].copy_(torch.from_numpy(hv))
    lut = class_lut()
    cls = torch.from_numpy(np.stack([lut[w.tokens(b)] for b in bs])).to(dev)
    return q, k, v, cls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c0", "c1", "c4"])
    ap.add_argument("--shard", choices=["head", "batch"], default="head")
    ap.add_argument("--T", type=float, default=0.95)
    ap.add_argument("--sessions", type=int, default=2)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_dev = os.environ.get("AKV_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = CONFIGS[args.config]()
    shard = (head_shard if args.shard == "head" else batch_shard)(w.B, w.H, world, rank)
    q, k, v, cls = shard_inputs(w, shard, dev)
    hs = range(shard.h0, shard.h1)
    sl = torch.tensor([w.slopes[h] for h in hs], dtype=torch.float32, device=dev)
    sk = torch.tensor([w.sinks[h] for h in hs], dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    cfg = ProfilerConfig(recovery_threshold=args.T)
    dec_cls = [cls[:, N + t].contiguous() for t in range(D)]

    def session():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        res, cache = encode_prompt_tensors(q, k, v, cls, cfg, prompt_len=N, max_new_tokens=D,
                                           slopes=sl, sinks=sk)
        ev[1].record()
        for t in range(D):
            decode_step_tensors(cache, q[:, :, N + t], k[:, :, N + t], v[:, :, N + t], dec_cls[t],
                                chained=True)
        ev[2].record()
        torch.cuda.synchronize()
        cache.check()
        return res, cache, ev

    session()   # warm-up
    times = []
    for _ in range(args.sessions):
        if dist is not None:
            dist.barrier()
        res, cache, ev = session()
        times.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    enc = float(np.mean([a for a, _ in times]))
    dec = float(np.mean([b for _, b in times]))
    tot = enc + dec
    if dist is not None:
        t = torch.tensor([enc, dec, tot], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        enc, dec, tot = t.tolist()
    fam = res.family
    rows = profile_rows(shard, [fam[c] for c in res.choice[:, 0]],
                        [res.recovery[g, c] for g, c in enumerate(res.choice[:, 0])],
                        [int(x) for x in res.kept_count])
    merged = gather_profile(rows)
    if rank == 0:
        csv = profile_csv(merged)
        pol = {}
        for r in merged:
            pol[r[2]] = pol.get(r[2], 0) + 1
        print(json.dumps({
            "config": args.config, "shard": args.shard, "world": world,
            "workload": f"B={w.B} H={w.H} N={N} D={D} d={w.d} {w.dtype}, T={args.T:g}",
            "local_heads_rank0": len(shard.heads),
            "profile_ms": enc, "decode_ms": dec, "decode_us_per_step": dec * 1e3 / D,
            "session_tok_s": w.B * D / (tot / 1e3),
            "scaling": "strong" if args.shard == "head" else "weak",
            "profile_csv_sha1": hashlib.sha1(csv.encode()).hexdigest(),
            "policies": pol, "timing": "max over ranks of CUDA-event means",
            "measurement": not one_dev,
        }), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
