"""K3 decode time per step across batch sizes (heads per launch G = B*H) at
config-1 shapes: achieved GB/s over the algorithmic bytes, to expose
occupancy cliffs (two CTAs per SM need the per-head page plan to fit in
shared memory).

    python tools/decode_scaling.py [B ...]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import decode_bytes, make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_steps_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import config1  # noqa: E402


def main():
    Bs = [int(x) for x in sys.argv[1:]] or [4, 8, 16, 17, 24, 32, 64]
    dev = torch.device("cuda")
    for B in Bs:
        w = config1(seed=1, B=B, D=64)
        qd, kd, vd, cd, *_ = make_inputs(w, dev)
        sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
        sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
        N, D = w.N, w.D
        res, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=0.95),
                                       prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cls = cd[:, N:].t().contiguous()
        # 16 warm-up steps, then D-16 timed ones, each batch in one library
        # call (the step loop in C++: the host does not bound small batches)
        decode_steps_tensors(c, qd[:, :, N:N + 16], kd[:, :, N:N + 16], vd[:, :, N:N + 16],
                             cls[:16], chained=True)
        e0.record()
        decode_steps_tensors(c, qd[:, :, N + 16:N + D], kd[:, :, N + 16:N + D],
                             vd[:, :, N + 16:N + D], cls[16:], chained=True)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (D - 16)
        L = c.live.cpu().numpy().astype(np.int64)
        nbytes = float(decode_bytes(w, res, [L, L])[0])
        print(f"B={B:3d} G={B * w.H:5d}: {us:7.1f} us/step  {nbytes / us / 1e3:7.0f} GB/s", flush=True)
        del qd, kd, vd, cd, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
