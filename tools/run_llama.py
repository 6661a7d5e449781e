"""Run the multi-layer caller (BASELINE configs 2/3) on the GPU(s) and
print one JSON line: prefill time, per-layer profiling time, decode tok/s,
cache occupancy, and size-independent checks (no segment overflow; every
full-policy head holds exactly prompt + steps rows; two identical runs of a
short session produce identical tokens).

    python tools/run_llama.py c2 [--layers L] [--batch B] [--prompt N] [--decode D] [--T 0.95]
    torchrun --nproc-per-node P tools/run_llama.py c2 --mode gather|tp|dp
    python tools/run_llama.py c3 --mode tp --gpus 8      # spawns the 8 ranks itself

Config 2 = Llama-7B shape (32 layers, d_model 4096, 32 heads, SwiGLU 11008,
vocab 32000), batch 16, prompt 2048, greedy decode 512; config 3 = Llama-65B
shape (80 layers, d_model 8192, 64 heads, 22016), batch 32, prompt 4096,
decode 1024, tensor parallel over 8 GPUs (``--mode tp``).  Weights are
random N(0, 0.02) bf16; prompts are seeded ids structured as config 0.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_01801_b200 import ProfilerConfig  # noqa: E402
from paper_2310_01801_b200.llama import LLAMA_7B, LLAMA_65B, FastGenLlama, ShardPlan  # noqa: E402
from paper_2310_01801_b200.workloads import PUNCT_IDS, PUNCT_PROB, SPECIAL_IDS  # noqa: E402

PRESETS = {"c2": (LLAMA_7B, 16, 2048, 512), "c3": (LLAMA_65B, 32, 4096, 1024)}


def prompt_ids(B, N, vocab, seed):
    rng = np.random.default_rng([seed, 2])
    ids = rng.integers(0, vocab, size=(B, N))
    punct = rng.random((B, N)) < PUNCT_PROB
    ids = np.where(punct, np.asarray(PUNCT_IDS)[rng.integers(0, len(PUNCT_IDS), (B, N))], ids)
    ids[:, 0] = SPECIAL_IDS[0]
    return ids


def _spawned(index, world, port, argv):
    os.environ.update({"RANK": str(index), "LOCAL_RANK": str(index), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.argv = argv
    main()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(PRESETS))
    ap.add_argument("--layers", type=int)
    ap.add_argument("--batch", type=int)
    ap.add_argument("--prompt", type=int)
    ap.add_argument("--decode", type=int)
    ap.add_argument("--T", type=float, default=0.95)
    ap.add_argument("--mode", default="gather", choices=["gather", "tp", "dp"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--simulate-world", type=int, default=0,
                    help="one process computes rank 0's shard of a P-way split without "
                         "collectives (per-GPU compute of a multi-GPU config on one GPU)")
    ap.add_argument("--diagnostics", action="store_true",
                    help="per-step recovery vs uncompressed attention (shadow keys)")
    ap.add_argument("--gpus", type=int, default=1,
                    help="without torchrun: spawn one process per GPU (NCCL), like bench.py")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket

        import torch.multiprocessing as tmp

        with socket.socket() as s_:
            s_.bind(("127.0.0.1", 0))
            port = s_.getsockname()[1]
        tmp.spawn(_spawned, args=(args.gpus, port, list(sys.argv)), nprocs=args.gpus, join=True)
        return
    cfg, B, N, D = PRESETS[args.config]
    if args.layers:
        cfg = type(cfg)(**{**cfg.__dict__, "n_layers": args.layers})
    B, N, D = args.batch or B, args.prompt or N, args.decode or D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    group = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    ids = prompt_ids(B, N, cfg.vocab, args.seed)
    if args.mode == "dp":       # independent sessions: this rank's batch rows
        per = B // world
        ids = ids[rank * per:(rank + 1) * per]
        plan = ShardPlan()
    elif args.simulate_world > 1:
        if world > 1:
            raise SystemExit("--simulate-world is a single-process measurement")
        plan = ShardPlan(0, args.simulate_world, args.mode, comm=False)
    else:
        plan = ShardPlan(rank, world, args.mode)
    t0 = time.time()
    model = FastGenLlama(cfg, seed=args.seed, plan=plan, group=group,
                         max_positions=N + D + 8)
    torch.cuda.synchronize()
    init_s = time.time() - t0
    tokens = torch.from_numpy(ids).cuda()
    pc = ProfilerConfig(recovery_threshold=args.T)

    # determinism of a short session (prefill + 4 steps)
    short = []
    for _ in range(2):
        model.prefill(tokens, pc, max_new_tokens=4)
        short.append(torch.stack([model.decode_step() for _ in range(4)], 1))
    deterministic = bool(torch.equal(short[0], short[1]))
    # warm-up at the timed size (allocator blocks, cuBLAS heuristics, clocks)
    model.prefill(tokens, pc, max_new_tokens=D)
    for _ in range(min(D, 8)):
        model.decode_step()
    model.caches = []

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev[0].record()
    pre = model.prefill(tokens, pc, max_new_tokens=D, diagnostics=args.diagnostics)
    ev[1].record()
    out = torch.empty(tokens.shape[0], D, dtype=torch.int64, device="cuda")
    for t in range(D):
        out[:, t] = model.decode_step()
        if t == 0:
            ev[3].record()   # the first step runs eagerly and captures the graphs
    mean_rec = model.mean_recovery() if args.diagnostics else None
    ev[2].record()
    torch.cuda.synchronize()
    model.check()
    prefill_ms = ev[0].elapsed_time(ev[1])
    decode_ms = ev[1].elapsed_time(ev[2])
    first_ms = ev[1].elapsed_time(ev[3])
    replay_ms = ev[3].elapsed_time(ev[2]) / max(D - 1, 1)
    prof_ms = pre.profiling_ms()
    b_local = tokens.shape[0]
    # full-policy heads hold exactly prompt + D rows; others no more
    full_ok, bound_ok, pol = True, True, {}
    for res, c in zip(pre.profiles, model.caches):
        live = c.live.cpu().numpy()
        fam = res.family
        for g, ch in enumerate(res.choice[:, 0]):
            name = str(fam[ch])
            pol[name] = pol.get(name, 0) + 1
            if fam[ch].is_full:
                full_ok &= int(live[g]) == N + D
            bound_ok &= int(live[g]) <= int(res.kept_count[g]) + D
    cache_tokens = model.cache_tokens()
    full_tokens = len(model.caches) * b_local * model.Hl * (N + D)
    dec_tok_s = b_local * D / (decode_ms / 1e3)
    if world > 1 and args.mode == "dp":
        t = torch.tensor([decode_ms, prefill_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        decode_ms, prefill_ms = t.tolist()
        dec_tok_s = B * D / (decode_ms / 1e3)
    line = dict(
        config=args.config, n_layers=cfg.n_layers, batch=B, prompt=N, decode=D, T=args.T,
        mode=args.mode, world=world, rank=rank, init_s=round(init_s, 1),
        simulated_world=args.simulate_world or None,
        local_heads=model.Hl, local_ffn=model.Fl,
        prefill_ms=prefill_ms, profiling_ms_per_layer=float(np.mean(prof_ms)),
        profiling_ms_total=float(np.sum(prof_ms)),
        decode_ms=decode_ms, decode_ms_per_step=decode_ms / D,
        first_step_ms=first_ms, replay_ms_per_step=replay_ms, decode_tok_s=dec_tok_s,
        cache_tokens=cache_tokens, full_cache_tokens=full_tokens,
        pruned_ratio=1 - cache_tokens / full_tokens, policies=pol,
        deterministic=deterministic, full_heads_exact=bool(full_ok), live_bounded=bool(bound_ok),
        first_tokens=out[0, :8].tolist(), mean_recovery_last_step=mean_rec,
        mem_gb=torch.cuda.max_memory_allocated() / 1e9)
    if rank == 0:
        print(json.dumps(line))
    assert deterministic and full_ok and bound_ok
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
