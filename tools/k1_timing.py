"""CUDA-event timing of the K1 passes + policy + K2 for a config's encode
(average of several encodes after warm-up)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = CONFIGS[name]()
dev = torch.device("cuda")
qd, kd, vd, cd, *_ = make_inputs(w, dev)
sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
cfg = ProfilerConfig(recovery_threshold=0.95)
for _ in range(3):
    encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
torch.cuda.synchronize()
n = 10
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / n
flops = 2 * w.B * w.H * w.d * w.N * (w.N + 1)
print(f"{name}: encode (K1 + policy + K2, incl. one host sync) {ms:.3f} ms; "
      f"{flops / ms / 1e9:.1f} TFLOP/s on the two QK^T passes")
