"""Host-side timing of encode_prompt_tensors phases over repeated sessions
(finds host stalls that show up as profiling-time outliers)."""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
import paper_2310_01801_b200.engine as E  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import config1  # noqa: E402

marks = {}
_orig_check = E.check


def timed_check(rc, exc=None):
    marks.setdefault("calls", []).append(time.perf_counter())
    return _orig_check(rc, exc)


E.check = timed_check
w = config1()
dev = torch.device("cuda")
qd, kd, vd, cd, *_ = make_inputs(w, dev)
sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
N, D = w.N, w.D
dec = [(qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t], cd[:, N + t].contiguous()) for t in range(D)]
cfg = ProfilerConfig(recovery_threshold=0.95)
rows = []
for s in range(20):
    marks.clear()
    t0 = time.perf_counter()
    res, c = E.encode_prompt_tensors(qd, kd, vd, cd, cfg, prompt_len=N, max_new_tokens=D, slopes=sl,
                                     sinks=sk)
    t1 = time.perf_counter()
    calls = marks["calls"]
    for t in range(D):
        decode_step_tensors(c, *dec[t], chained=True)
    t2 = time.perf_counter()
    # calls: profile, plan, compact, ws_init ; phases between them
    rows.append((calls[0] - t0, calls[1] - calls[0], calls[2] - calls[1], calls[3] - calls[2],
                 t1 - calls[3], t2 - t1))
names = ["pre-profile", "profile->plan", "plan->compact(incl sync)", "compact->wsinit", "post",
         "decode enqueue"]
for i, n in enumerate(names):
    col = [r[i] * 1e3 for r in rows]
    print(f"{n:28s} median {statistics.median(col):8.3f} ms  max {max(col):8.3f} ms")
