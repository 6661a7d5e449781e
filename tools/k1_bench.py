"""K1 (akv_profile: both tcgen05 passes + the policy epilogue) timed alone
with CUDA events around the akv_profile call inside encode, as bench.py
does; c1 and c4 by default.

    python tools/k1_bench.py [c1 c4 ...]
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402


def k1_ms(name, reps=8):
    w = CONFIGS[name]()
    dev = torch.device("cuda")
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    cfg = ProfilerConfig(recovery_threshold=w.thresholds[0])
    out = []
    for i in range(reps + 2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=w.N, max_new_tokens=w.D, slopes=sl,
                              sinks=sk, k1_events=ev)
        torch.cuda.synchronize()
        if i >= 2:
            out.append(ev[0].elapsed_time(ev[1]))
    ms = statistics.median(out)
    exps = w.B * w.H * w.N * (w.N + 1)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peak = 16 * sms * 1.965e9
    return {"config": name, "k1_ms": ms, "tflops": 2 * w.d * exps / (ms * 1e-3) / 1e12,
            "exp_frac_at_1965mhz": exps / (ms * 1e-3) / peak, "env": {k: v for k, v in os.environ.items() if k.startswith("AKV_")}}


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c1", "c4"]:
        print(json.dumps(k1_ms(n)), flush=True)
