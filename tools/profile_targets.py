"""Small drivers for ncu captures (one process each):

    python tools/profile_targets.py k3      # c1 session: K3 launches (capture a mid-session one)
    python tools/profile_targets.py diag    # c1 session with diagnostics: akv_decode_recovery + K3
    python tools/profile_targets.py k3f     # c1_frequent session (T=0.98, FREQUENT-heavy): K3
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import config1, config1_frequent  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "k3"
    w = config1_frequent() if what == "k3f" else config1()
    T = 0.98 if what == "k3f" else 0.95
    dev = torch.device("cuda")
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    cls = [cd[:, N + t].contiguous() for t in range(D)]
    _, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                 prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk,
                                 diagnostics=(what == "diag"))
    for t in range(D):
        decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t], cls[t],
                            chained=True)
    torch.cuda.synchronize()
    c.check()
    print("ok", float(c.step_recovery.mean()) if what == "diag" else "")


if __name__ == "__main__":
    main()
