"""One encode of a config (for an ncu launch list of the K1/K2 kernels)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]()
dev = torch.device("cuda")
qd, kd, vd, cd, *_ = make_inputs(w, dev)
sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
for _ in range(2):
    encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=0.95), prompt_len=w.N,
                          max_new_tokens=w.D, slopes=sl, sinks=sk)
torch.cuda.synchronize()
print("ok")
