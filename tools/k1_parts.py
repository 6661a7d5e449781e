"""Per-kernel GPU time of the profiling pass (K1: row pass, column pass,
policy) inside encode, from the CUDA activity trace (torch.profiler), plus
the event-timed K1 total as bench.py measures it.

    python tools/k1_parts.py [c1 c4 ...]
"""
import collections
import json
import os
import statistics
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402


def parts(name, reps=6):
    w = CONFIGS[name]()
    dev = torch.device("cuda")
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    cfg = ProfilerConfig(recovery_threshold=w.thresholds[0])
    run = lambda ev=None: encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=w.N,  # noqa: E731
                                                max_new_tokens=w.D, slopes=sl, sinks=sk, k1_events=ev)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    tot = []
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        run(ev)
        torch.cuda.synchronize()
        tot.append(ev[0].elapsed_time(ev[1]))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            run()
        torch.cuda.synchronize()
    us = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type.name == "CUDA" and ("k1" in e.name or "k2_" in e.name):
            us[e.name.split("(")[0].replace("void ", "")].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    return {"config": name, "k1_event_ms": statistics.median(tot),
            "kernels_us": {k: round(statistics.median(v), 2) for k, v in us.items()},
            "env": {k: v for k, v in os.environ.items() if k.startswith("AKV_")}}


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c1"]:
        print(json.dumps(parts(n)), flush=True)
