"""Per-step decode timing of the multi-layer caller (config 2 shapes by
default): the eager first step + graph capture, the first replays, and the
steady state, each bracketed by CUDA events, to separate one-time costs from
the per-step cost.

    python tools/c2_steps.py [layers] [B] [N] [steps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_01801_b200 import ProfilerConfig  # noqa: E402
from paper_2310_01801_b200.llama import LLAMA_7B, FastGenLlama  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    layers, B, N, S = (a + [32, 16, 2048, 64][len(a):])[:4]
    cfg = type(LLAMA_7B)(**{**LLAMA_7B.__dict__, "n_layers": layers})
    model = FastGenLlama(cfg, seed=0, max_positions=N + S + 8)
    ids = np.random.default_rng(0).integers(0, cfg.vocab, size=(B, N))
    ids[:, 0] = 1
    tokens = torch.from_numpy(ids).cuda()
    pc = ProfilerConfig(recovery_threshold=0.95)
    for rep in range(2):
        model.prefill(tokens, pc, max_new_tokens=S)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(S + 1)]
        ev[0].record()
        for t in range(S):
            model.decode_step()
            ev[t + 1].record()
        torch.cuda.synchronize()
        ms = [ev[t].elapsed_time(ev[t + 1]) for t in range(S)]
        blocks = [f"{np.mean(ms[i:i + 64]):.3f}" for i in range(0, S, 64)]
        print(f"rep {rep}: per-64-step means {blocks}")
        print(f"rep {rep}: first {ms[0]:.2f} ms, next {['%.3f' % x for x in ms[1:6]]}, "
              f"steady (steps 8..) {np.mean(ms[8:]):.3f} ms/step min {np.min(ms[8:]):.3f}")
    # steady state of pure graph replays, back to back
    model.prefill(tokens, pc, max_new_tokens=S)
    for _ in range(4):
        model.decode_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = S - 8
    for _ in range(n):
        model.decode_step()
    e1.record()
    torch.cuda.synchronize()
    print(f"back-to-back replays: {e0.elapsed_time(e1) / n:.3f} ms/step ({layers} layers, B={B}, N={N})")


if __name__ == "__main__":
    main()
