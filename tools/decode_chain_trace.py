"""Per-CTA timelines of several CONSECUTIVE K3 launches in steady state
(chained, no syncs between them): shows how a step's tail overlaps the next
step's start.  Stamps: 0 start, 1 planned, 2 first page, 3 last page, 4 done."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200._lib import lib  # noqa: E402
from paper_2310_01801_b200.workloads import config1  # noqa: E402


def main():
    T = float(sys.argv[1]) if len(sys.argv) > 1 else 0.95
    at = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    K = 4
    dev = torch.device("cuda")
    w = config1()
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    cls = [cd[:, N + t].contiguous() for t in range(D)]
    _, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T), prompt_len=N,
                                 max_new_tokens=D, slopes=sl, sinks=sk)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bufs = [torch.zeros(2 * sms * 16, dtype=torch.int64, device=dev) for _ in range(K)]
    lib.akv_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
    for t in range(at + K):
        if at <= t < at + K:
            lib.akv_debug_set_decode_trace(bufs[t - at].data_ptr())
        decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t], cls[t], chained=True)
        lib.akv_debug_set_decode_trace(None)
    torch.cuda.synchronize()
    trs = [b.view(-1, 16).cpu().numpy().astype(np.float64) for b in bufs]
    t0 = min(tr[tr[:, 4] > 0, 0].min() for tr in trs)
    for k, tr in enumerate(trs):
        ok = tr[:, 4] > 0
        rel = (tr[ok, :5] - t0) / 1e3
        q = lambda col, p: np.percentile(rel[:, col], p)  # noqa: E731
        print(f"step {at + k}: CTAs {ok.sum()}  start [{q(0, 0):6.1f} {q(0, 50):6.1f} {q(0, 100):6.1f}]"
              f"  planned-start {np.median(rel[:, 1] - rel[:, 0]):5.2f}"
              f"  first page [{q(2, 0):6.1f} {q(2, 50):6.1f}] (-start {np.median(rel[:, 2] - rel[:, 0]):5.2f})"
              f"  last page [{q(3, 50):6.1f} {q(3, 100):6.1f}]"
              f"  done [{q(4, 50):6.1f} {q(4, 90):6.1f} {q(4, 100):6.1f}]")


if __name__ == "__main__":
    main()
