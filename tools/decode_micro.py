"""Decode-loop microbenchmark: eager launches vs one CUDA graph of all D
steps (separates host launch overhead from kernel time)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import config1  # noqa: E402


def main():
    T = float(sys.argv[1]) if len(sys.argv) > 1 else 0.95
    dev = torch.device("cuda")
    w = config1()
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    dq = [qd[:, :, N + t] for t in range(D)]
    dk = [kd[:, :, N + t] for t in range(D)]
    dv = [vd[:, :, N + t] for t in range(D)]
    dc = [cd[:, N + t].contiguous() for t in range(D)]
    cfg = ProfilerConfig(recovery_threshold=T)

    def enc():
        return encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=N, max_new_tokens=D,
                                     slopes=sl, sinks=sk)[1]

    for _ in range(2):  # warm
        c = enc()
        for t in range(D):
            decode_step_tensors(c, dq[t], dk[t], dv[t], dc[t], chained=True)
    torch.cuda.synchronize()
    # eager
    c = enc()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for t in range(D):
        decode_step_tensors(c, dq[t], dk[t], dv[t], dc[t], chained=True)
    e1.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    eager_us = e0.elapsed_time(e1) * 1e3 / D
    host_us = (h1 - h0) * 1e6 / D
    live_eager = c.live.clone()
    # graph
    c = enc()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for t in range(D):
                decode_step_tensors(c, dq[t], dk[t], dv[t], dc[t], chained=True)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) * 1e3 / D
    same = bool(torch.equal(c.live, live_eager))
    print(f"T={T} eager {eager_us:.1f} us/step (host enqueue {host_us:.1f} us/step); "
          f"graph {graph_us:.1f} us/step; final live equal: {same}; "
          f"final cache tokens {int(c.live.sum())}")


if __name__ == "__main__":
    main()
