"""Per-CTA timeline of one K3 decode launch (globaltimer stamps):
0 start, 1 page plan done, 2 first page landed, 3 last page consumed,
4 CTA done; 5 epilogues run, 6 frequent-head epilogues."""
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
    ats = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256]
    dev = torch.device("cuda")
    w = config1()
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    _, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T), prompt_len=N,
                                 max_new_tokens=D, slopes=sl, sinks=sk)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(2 * sms * 16, dtype=torch.int64, device=dev)
    lib.akv_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
    for t in range(max(ats) + 1):
        if t in ats:
            torch.cuda.synchronize()
            buf.zero_()
            lib.akv_debug_set_decode_trace(buf.data_ptr())
        decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t],
                            cd[:, N + t].contiguous())
        if t in ats:
            torch.cuda.synchronize()
            lib.akv_debug_set_decode_trace(None)
            report(buf, T, t, verbose=len(ats) == 1)


def report(buf, T, at, verbose):
    tr = buf.view(-1, 16).cpu().numpy().astype(np.float64)
    ok = tr[:, 4] > 0
    t0 = tr[ok, 0].min()
    rel = (tr[ok, :5] - t0) / 1e3
    names = ["start", "planned", "first page", "last page", "done"]
    print(f"T={T} step {at}: {ok.sum()} working CTAs, span {rel[:, 4].max():.1f} us, "
          f"last page p50 {np.median(rel[:, 3]):.1f}, fallbacks {int(tr[ok, 7].sum())}")
    if not verbose:
        return
    for i, nm in enumerate(names):
        col = rel[:, i]
        print(f"  {nm:11s} min {col.min():6.1f} p50 {np.median(col):6.1f} p90 {np.percentile(col, 90):6.1f} max {col.max():6.1f}")
    ep = tr[ok, 5]
    fq = tr[ok, 6]
    print(f"  epilogues per CTA: {np.bincount(ep.astype(int)).tolist()}, frequent: {int(fq.sum())}, top-k fallbacks: {int(tr[ok, 7].sum())}")
    ph = (tr[ok][:, 8:11] - t0) / 1e3  # last segment: publish start, partial released, finished
    print(f"  last segment: publish start p50 {np.median(ph[:, 0]):.1f}, released p50 "
          f"{np.median(ph[:, 1]):.1f}, finished p50 {np.median(ph[:, 2]):.1f}; "
          f"last page -> publish start p50 {np.median(ph[:, 0] - rel[:, 3]):.1f} us, "
          f"publish -> released p50 {np.median(ph[:, 1] - ph[:, 0]):.1f} us, "
          f"released -> finished p50 {np.median(ph[:, 2] - ph[:, 1]):.1f} us")
    late = np.argsort(-rel[:, 4])[:5]
    for i in late:
        print(f"  late CTA: planned {rel[i,1]:.1f} first {rel[i,2]:.1f} last {rel[i,3]:.1f} "
              f"publish {ph[i,0]:.1f} released {ph[i,1]:.1f} finished {ph[i,2]:.1f} "
              f"done {rel[i,4]:.1f} ep {int(ep[i])} freq {int(fq[i])}")


if __name__ == "__main__":
    main()
