"""Process-pool worker for the full headline-session parity check
(tests/test_gpu_headline_session.py): the CPU oracle (float64 restatement
of the reference, pinned to its goldens) runs one config-1 head's whole
session - profiling, compaction, D teacher-forced decode steps - and returns
its policy, kept sets after encode and after every step (bit-packed) and
its outputs.  Test infrastructure only; imported by spawned workers, so it
does not import torch or the product package."""

from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _workloads():
    name = "_akv_oracle_session_workloads"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(
            name, os.path.join(ROOT, "paper_2310_01801_b200", "workloads.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
    return sys.modules[name]


def run_heads(job):
    """job = (config name, seed, B, H, N, D, T, [(b, h), ...]).  Returns a
    list of dicts."""
    from threadpoolctl import threadpool_limits

    from oracle import akv_oracle as O

    name, seed, B, H, N, D, T, heads = job
    W = _workloads()
    w = W.CONFIGS[name](seed=seed, B=B, H=H, N=N, D=D)
    lut = W.class_lut()
    fam = O.default_family(w.r_l, w.r_f)
    out = []
    with threadpool_limits(limits=1):
        for b, h in heads:
            cls = lut[w.tokens(b)].astype(np.int64)
            q, k, v = (x.astype(np.float64) for x in w.head_qkv(b, h))
            prof = O.profile_head(q[:N], k[:N], v[:N], cls, w.slopes[h], w.sinks[h], fam, [T])
            enc = np.zeros(N, bool)
            enc[prof.kept] = True
            st = O.compact_head(prof, k[:N], v[:N], fam[prof.choice[0]], N, w.slopes[h],
                                w.sinks[h])
            kept = np.zeros((D, N + D), bool)
            outs = np.zeros((D, w.d))
            for t in range(D):
                outs[t] = O.decode_head(st, q[N + t], k[N + t], v[N + t], N + t, cls, N)
                kept[t, st.positions] = True
            out.append(dict(b=b, h=h, choice=int(prof.choice[0]), R=prof.recoveries,
                            enc=np.packbits(enc), kept=np.packbits(kept, axis=-1), out=outs))
    return out
