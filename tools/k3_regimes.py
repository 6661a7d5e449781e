"""K3 decode throughput across compression regimes at config-1 shapes
(B=8 x 32 heads, N=1024, D=512, bf16): the headline mix (c1, T=0.95 / 0.99:
240 of 256 heads full) and the FREQUENT-heavy mix (c1_frequent, T=0.98:
~3/4 of the heads evict through the score update + top-k every step).

Per regime: K3 us/step over a chained session (CUDA events), algorithmic
bytes per launch (bench.decode_bytes: live K/V rows + new row + 4-byte
metadata + 16 B/slot score read+write for FREQUENT heads + q/k/v/o) and the
fraction of the measured HBM peak; plus one traced mid-session step: the
epilogues run, how many were FREQUENT, radix-select fallbacks, and the
per-CTA tail after its last page.

    python tools/k3_regimes.py [c1:0.95 c1_frequent:0.98 ...]
"""
import ctypes
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200._lib import lib  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402


def regime(name, T, reps=3):
    dev = torch.device("cuda")
    w = CONFIGS[name]()
    qd, kd, vd, cd, *_ = bench.make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    dec = bench._dec_inputs(qd, kd, vd, cd, w.N, w.D)
    res, cache, lives = bench.run_session(w, T, qd, kd, vd, cd, sl, sk, dec, record=True)
    cache.check()
    nbytes = statistics.mean(bench.decode_bytes(w, res, lives))
    del cache
    ms = []
    for _ in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        bench.run_session(w, T, qd, kd, vd, cd, sl, sk, dec, ev=ev)
        torch.cuda.synchronize()
        ms.append(ev[1].elapsed_time(ev[2]))
    us = statistics.median(ms[1:]) * 1e3 / w.D
    gbs = nbytes / (us * 1e-6) / 1e9
    peaks, _ = bench._peaks()
    # one traced step in the middle of a session
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(2 * sms * 16, dtype=torch.int64, device=dev)
    lib.akv_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
    _, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                 prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
    at = w.D // 2
    for t in range(at + 1):
        if t == at:
            torch.cuda.synchronize()
            lib.akv_debug_set_decode_trace(buf.data_ptr())
        decode_step_tensors(c, dec[0][t], dec[1][t], dec[2][t], dec[3][t], chained=True)
        lib.akv_debug_set_decode_trace(None)
    torch.cuda.synchronize()
    tr = buf.view(-1, 16).cpu().numpy().astype(np.float64)
    if os.environ.get("AKV_TRACE_DUMP"):
        np.save(f"{os.environ['AKV_TRACE_DUMP']}_{name}_{T:g}.npy", buf.view(-1, 16).cpu().numpy())
    ok = tr[:, 4] > 0
    t0 = tr[ok, 0].min()
    rel = (tr[ok] - t0) / 1e3
    fam = res.family
    pol = np.bincount(res.choice[:, 0], minlength=len(fam))
    freq = sum(int(pol[i]) for i in range(len(fam)) if fam[i].bits & 4 and not fam[i].is_full)
    return {
        "workload": name, "T": T, "heads": w.B * w.H, "frequent_heads": freq,
        "policies": {str(fam[i]): int(pol[i]) for i in range(len(fam)) if pol[i]},
        "k3_us_per_step": us, "algorithmic_mb_per_launch": nbytes / 1e6, "k3_gbs": gbs,
        "frac_of_measured_peak": gbs / peaks["hbm_gbs"],
        "traced_step": {
            "ctas": int(ok.sum()), "epilogues": int(tr[ok, 5].sum()),
            "frequent_epilogues": int(tr[ok, 6].sum()), "radix_fallbacks": int(tr[ok, 7].sum()),
            "isolated_step_us": float(rel[:, 4].max()),
            "plan_us_median": float(np.median(rel[:, 1] - rel[:, 0])),
            # slots 11-15: FREQUENT policy phase cycle stamps of a -DAKV_TRACE_EPI
            # build (pass A, decision, action, evictions), relative to slot 11
            "phase_cycles_median": [float(np.median((tr[:, j] - tr[:, 11])[(tr[:, 11] > 0) & (tr[:, j] > 0)]))
                                    if ((tr[:, 11] > 0) & (tr[:, j] > 0)).any() else None
                                    for j in (12, 13, 14, 15)],
            "first_page_us_median": float(np.median(rel[:, 2] - rel[:, 0])),
            "last_page_us_median": float(np.median(rel[:, 3])),
            "tail_after_last_page_us": [float(np.percentile((rel[:, 4] - rel[:, 3])[tr[ok, 3] > 0], p))
                                        for p in (50, 90, 100)],
        },
    }


def main():
    specs = sys.argv[1:] or ["c1:0.95", "c1:0.99", "c1_frequent:0.98"]
    for s in specs:
        name, T = s.split(":")
        r = regime(name, float(T))
        r["env"] = {k: v for k, v in os.environ.items() if k.startswith("AKV_")}
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
