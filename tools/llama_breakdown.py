"""Per-op CUDA-event breakdown of one Llama layer at config-2 shapes
(prefill and decode), to find where the caller's time goes.

    python tools/llama_breakdown.py [B N]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.llama import LLAMA_7B, FastGenLlama  # noqa: E402


def timed(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / reps:9.3f} ms")
    return out


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    cfg = type(LLAMA_7B)(**{**LLAMA_7B.__dict__, "n_layers": 1})
    m = FastGenLlama(cfg, max_positions=N + 8)
    L = m.layers[0]
    d, T = cfg.head_dim, B * N
    x = torch.randn(T, cfg.d_model, device="cuda").to(torch.bfloat16)
    res = x.clone()
    print(f"prefill B={B} N={N}; sdpa backends: flash={torch.backends.cuda.flash_sdp_enabled()} "
          f"cudnn={torch.backends.cuda.cudnn_sdp_enabled()} "
          f"mem_eff={torch.backends.cuda.mem_efficient_sdp_enabled()}")
    xn = timed("rmsnorm", lambda: m._rmsnorm(res, L.attn_norm))
    qkv = timed("qkv gemm", lambda: torch.nn.functional.linear(xn, L.wqkv))
    q = torch.empty(B, cfg.n_heads, N, d, dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    timed("rope_scatter", lambda: m._rope(qkv, N, 0, q, k, v, N))
    o = timed("sdpa causal", lambda: torch.nn.functional.scaled_dot_product_attention(
        q, k, v, is_causal=True))
    for be in ("FLASH_ATTENTION", "CUDNN_ATTENTION", "EFFICIENT_ATTENTION"):
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel

            with sdpa_kernel(getattr(SDPBackend, be)):
                timed(f"  sdpa[{be.lower()}]", lambda: torch.nn.functional.scaled_dot_product_attention(
                    q, k, v, is_causal=True))
        except Exception as e:  # noqa: BLE001
            print(f"  sdpa[{be.lower()}] unavailable: {str(e).splitlines()[0][:80]}")
    cls = torch.zeros(B, N, dtype=torch.uint8, device="cuda")
    pc = ProfilerConfig(recovery_threshold=0.95)
    timed("K1+K2 encode_prompt", lambda: encode_prompt_tensors(q, k, v, cls, pc, prompt_len=N,
                                                                max_new_tokens=512))
    ot = timed("o transpose", lambda: o.transpose(1, 2).reshape(T, cfg.n_heads * d))
    attn = timed("o gemm", lambda: torch.nn.functional.linear(ot, L.wo))
    xn2 = timed("add_rmsnorm", lambda: m._rmsnorm(res, L.mlp_norm, x=attn))
    gu = timed("gate|up gemm", lambda: torch.nn.functional.linear(xn2, L.wgu))
    sw = timed("swiglu", lambda: m._swiglu(gu))
    timed("down gemm", lambda: torch.nn.functional.linear(sw, L.wdown))


if __name__ == "__main__":
    main()


def decode_breakdown(B=16, N=2048, steps=20):
    """Per-op time of one decode layer step (1-layer model, c2 shapes)."""
    from paper_2310_01801_b200 import decode_step_tensors

    cfg = type(LLAMA_7B)(**{**LLAMA_7B.__dict__, "n_layers": 1})
    m = FastGenLlama(cfg, max_positions=N + 600)
    ids = torch.randint(0, cfg.vocab, (B, N), device="cuda")
    m.prefill(ids, ProfilerConfig(recovery_threshold=0.95), max_new_tokens=512)
    for _ in range(3):
        m.decode_step()
    L = m.layers[0]
    d = cfg.head_dim
    res = m.x_next.clone()
    print(f"decode B={B} L~{N}")
    xn = timed("rmsnorm", lambda: m._rmsnorm(res, L.attn_norm), reps=steps)
    qkv = timed("qkv gemm", lambda: torch.nn.functional.linear(xn, L.wqkv), reps=steps)
    timed("rope_scatter", lambda: m._rope(qkv, 1, m.seq_len, m.q1, m.k1, m.v1, 1), reps=steps)
    c = m.caches[0]
    cls = m.next_cls.clone()

    def k3():
        o = decode_step_tensors(c, m.q1, m.k1, m.v1, cls, out=m.o_dec[0])
        return o
    o = timed("K3 decode step", k3, reps=steps)
    ob = timed("cast o", lambda: o.view(B, -1).to(torch.bfloat16), reps=steps)
    attn = timed("o gemm", lambda: torch.nn.functional.linear(ob, L.wo), reps=steps)
    xn2 = timed("add_rmsnorm", lambda: m._rmsnorm(res, L.mlp_norm, x=attn), reps=steps)
    gu = timed("gate|up gemm", lambda: torch.nn.functional.linear(xn2, L.wgu), reps=steps)
    sw = timed("swiglu", lambda: m._swiglu(gu), reps=steps)
    timed("down gemm", lambda: torch.nn.functional.linear(sw, L.wdown), reps=steps)
    logits = timed("lm_head gemm", lambda: torch.nn.functional.linear(xn2, m.lm_head), reps=steps)
    timed("greedy_next", lambda: m._greedy(logits), reps=steps)
    import time as _t
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    for _ in range(steps):
        m.decode_step()
    t1 = _t.perf_counter()
    torch.cuda.synchronize()
    t2 = _t.perf_counter()
    print(f"full 1-layer decode_step: host {1e3 * (t1 - t0) / steps:.3f} ms/step issue, "
          f"{1e3 * (t2 - t0) / steps:.3f} ms/step wall")


if __name__ == "__main__" and os.environ.get("DECODE", "1") == "1":
    decode_breakdown()
