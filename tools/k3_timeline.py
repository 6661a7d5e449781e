"""Per-CTA timeline of consecutive chained K3 steps in the middle of a c1
session (globaltimer stamps through the akv_debug_set_decode_trace hook, one
buffer per step): when each step's CTAs start, land their first page, finish
streaming and finish publishing, relative to the first CTA of the first
traced step - how much of a step overlaps its predecessor.

    python tools/k3_timeline.py [config] [T] [steps] [B] [call]

call = "step" (one decode_step_tensors call per step, the default) or
"steps" (one decode_steps_tensors call for the traced steps: the step loop
in C++, as bench sessions issue them; a trace ring keeps the steps apart).
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_01801_b200 import (ProfilerConfig, decode_step_tensors,  # noqa: E402
                                   decode_steps_tensors, encode_prompt_tensors)
from paper_2310_01801_b200._lib import lib  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    T = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    dev = torch.device("cuda")
    w = CONFIGS[name](B=int(sys.argv[4])) if len(sys.argv) > 4 else CONFIGS[name]()
    qd, kd, vd, cd, *_ = bench.make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    dec = bench._dec_inputs(qd, kd, vd, cd, w.N, w.D)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bufs = [torch.zeros(2 * sms * 16, dtype=torch.int64, device=dev) for _ in range(n)]
    lib.akv_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
    _, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                 prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
    at = w.D // 2
    call = sys.argv[5] if len(sys.argv) > 5 else "step"
    if call == "steps":
        for t in range(at):
            decode_step_tensors(c, dec[0][t], dec[1][t], dec[2][t], dec[3][t], chained=True)
        ring = torch.zeros(n * 2 * sms * 16, dtype=torch.int64, device=dev)
        lib.akv_debug_set_decode_trace_ring.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.akv_debug_set_decode_trace_ring(ring.data_ptr(), n)
        N = w.N
        cls = cd[:, N + at:N + at + n].t().contiguous()
        decode_steps_tensors(c, qd[:, :, N + at:N + at + n], kd[:, :, N + at:N + at + n],
                             vd[:, :, N + at:N + at + n], cls, chained=True)
        lib.akv_debug_set_decode_trace(None)
        torch.cuda.synchronize()
        # step s of the call wrote block (at + s) mod n
        blocks = ring.view(n, -1, 16).cpu().numpy().astype(np.float64)
        trs = [blocks[(at + s) % n] for s in range(n)]
    else:
        for t in range(at + n):
            if t >= at:
                lib.akv_debug_set_decode_trace(bufs[t - at].data_ptr())
            decode_step_tensors(c, dec[0][t], dec[1][t], dec[2][t], dec[3][t], chained=True)
        lib.akv_debug_set_decode_trace(None)
        torch.cuda.synchronize()
        trs = [b.view(-1, 16).cpu().numpy().astype(np.float64) for b in bufs]
    t0 = min(tr[tr[:, 0] > 0, 0].min() for tr in trs)
    print(f"{name} T={T}: us relative to the first traced CTA start; med / p90 / max over CTAs")
    print("step  ctas  start(min,med,max)      plan_done(med)  first_page(med,max)  last_page(med,max)  end(med,p90,max)")
    prev_end = None
    for i, tr in enumerate(trs):
        ok = tr[:, 0] > 0
        r = (tr[ok] - t0) / 1e3
        end = np.maximum(r[:, 4], r[:, 10])
        fp = r[:, 2][tr[ok, 2] > 0]
        lp = r[:, 3][tr[ok, 3] > 0]
        print(f"{i:4d}  {ok.sum():4d}  {r[:,0].min():6.1f} {np.median(r[:,0]):6.1f} {r[:,0].max():6.1f}   "
              f"{np.median(r[:,1]):6.1f}          {np.median(fp):6.1f} {fp.max():6.1f}        "
              f"{np.median(lp):6.1f} {lp.max():6.1f}      {np.median(end):6.1f} {np.percentile(end,90):6.1f} {end.max():6.1f}")
        if prev_end is not None:
            print(f"      step start (min) - previous step end (max): {r[:,0].min() - prev_end:6.1f} us;"
                  f" first page (max) - previous end (max): {fp.max() - prev_end:6.1f}")
        # the CTA that ends last: its stamps (0 start, 1 planned, 2 first page, 3 last page,
        # 8 publish start, 9 partial released, 10 segment done, 4 epilogue warps done)
        k = int(np.argmax(end))
        names = {0: "start", 1: "plan", 2: "first", 3: "last", 8: "pub", 9: "rel", 10: "seg", 4: "epi"}
        print("      last CTA:", ", ".join(f"{names[j]} {r[k, j]:.1f}" for j in (0, 1, 2, 3, 8, 9, 10, 4)
                                         if tr[ok][k, j] > 0))
        prev_end = end.max()


if __name__ == "__main__":
    main()
