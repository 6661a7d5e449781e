"""Run one BASELINE config end to end on the GPU and report timings plus
size-independent invariants (used for c4, which the CPU oracle cannot
cover at full size):

* determinism: two identical sessions give bitwise-identical outputs,
  live counts and per-head profiles;
* budgets: every head's live count after each step equals the size of the
  policy's retained set implied by its atoms (full heads grow by one per
  step and never evict);
* capacity: no segment overflow.

    python tools/run_config.py c4 [T]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_inputs  # noqa: E402
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors  # noqa: E402
from paper_2310_01801_b200.workloads import CONFIGS  # noqa: E402


def session(w, T, qd, kd, vd, cd, sl, sk, record):
    N, D = w.N, w.D
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    cls_cols = [cd[:, N + t].contiguous() for t in range(D)]
    ev[0].record()
    res, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                   prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk)
    ev[1].record()
    outs, lives = [], []
    for t in range(D):
        o = decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t],
                                cls_cols[t], chained=True)
        if record:
            outs.append(o.clone())
            lives.append(c.live.clone())
    ev[2].record()
    torch.cuda.synchronize()
    c.check()
    return res, c, ev, outs, lives


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    T = float(sys.argv[2]) if len(sys.argv) > 2 else 0.95
    w = CONFIGS[name]()
    dev = torch.device("cuda")
    t0 = time.time()
    qd, kd, vd, cd, *_ = make_inputs(w, dev)
    print(f"{name}: B={w.B} H={w.H} N={w.N} D={w.D} d={w.d} inputs in {time.time() - t0:.1f}s")
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    r1, c1, _, o1, l1 = session(w, T, qd, kd, vd, cd, sl, sk, True)
    r2, c2, ev, o2, l2 = session(w, T, qd, kd, vd, cd, sl, sk, True)
    det = all(torch.equal(a, b) for a, b in zip(o1, o2)) and all(torch.equal(a, b) for a, b in zip(l1, l2))
    det &= np.array_equal(r1.choice, r2.choice) and np.array_equal(r1.recovery, r2.recovery)
    # budgets: full heads grow by one per step, others never exceed kept + steps
    fam = r2.family
    full = np.array([fam[c].is_full for c in r2.choice[:, 0]])
    L = torch.stack(l2).cpu().numpy()  # [D, G]
    kept = r2.kept_count
    full_ok = np.array_equal(L[:, full], kept[full][None, :] + np.arange(1, w.D + 1)[:, None])
    bound_ok = bool((L <= kept[None, :] + np.arange(1, w.D + 1)[:, None]).all())
    _, _, ev3, _, _ = session(w, T, qd, kd, vd, cd, sl, sk, False)
    enc = ev3[0].elapsed_time(ev3[1])
    dec = ev3[1].elapsed_time(ev3[2])
    pol = np.bincount(r2.choice[:, 0], minlength=len(fam))
    print(f"profile+compact {enc:.2f} ms, decode {dec:.2f} ms ({dec * 1e3 / w.D:.1f} us/step), "
          f"session {w.B * w.D / ((enc + dec) / 1e3):.0f} tok/s")
    print("policies:", {str(fam[i]): int(pol[i]) for i in range(len(fam)) if pol[i]})
    print(f"final cache tokens {int(L[-1].sum())} of {w.B * w.H * (w.N + w.D)} "
          f"(pruned {1 - L[-1].sum() / (w.B * w.H * (w.N + w.D)):.3f})")
    print(f"deterministic: {det}; full heads grow exactly: {full_ok}; live <= kept+steps: {bound_ok}")
    assert det and full_ok and bound_ok


if __name__ == "__main__":
    main()
