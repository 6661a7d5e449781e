"""K3 launch-level invariants on the B200, through the C-ABI:

* chained steps (AKV_DECODE_CHAINED: a step streams settled full-cache
  pages while its predecessor drains, programmatic dependent launch) give
  bit-identical outputs and kept sets to unchained steps - with few heads
  per launch, so a head's pages split over several CTAs and the consumer
  warps publish split-K partials while the previous step may still run;
* batches beyond the 2,048 heads one launch plans for run as consecutive
  launches over batch rows, bit-identical to running the rows separately,
  and match the CPU oracle (engine.py:303-350).
"""

import numpy as np
import pytest
import torch

from helpers import NAME_BIT  # noqa: F401  (puts the oracle on the path)
from oracle import akv_oracle as O
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors
from paper_2310_01801_b200.workloads import Workload, class_lut

pytestmark = pytest.mark.gpu


def _workload(B, H, N, D, d, seed):
    """Sink strengths graded so that at T=0.98 the heads mix `special`,
    `special+punct+frequent` (evicting every step) and `full`."""
    if H <= 12:
        sinks = np.array([11.0, 0.0, 9.5, 10.5, 0.0, 12.0, 8.5, 11.0, 0, 10, 9, 0])[:H]
        slopes = np.array([0, 0.05, 0.05, 0, 0, 0, 0.05, 0, 0, 0, 0.05, 0])[:H]
    else:
        sinks = np.tile([11.0, 0.0, 9.5, 10.5], H // 4)
        slopes = np.tile([0, 0.05, 0, 0.05], H // 4)
    return Workload("chain", B, H, N, D, d, "bf16", (0.98,), seed=seed, slopes=slopes,
                    sinks=sinks)


def _inputs(w, rows=None):
    rows = list(range(w.B)) if rows is None else rows
    dev = torch.device("cuda")
    q = np.stack([np.stack([w.head_qkv(b, h)[0] for h in range(w.H)]) for b in rows])
    k = np.stack([np.stack([w.head_qkv(b, h)[1] for h in range(w.H)]) for b in rows])
    v = np.stack([np.stack([w.head_qkv(b, h)[2] for h in range(w.H)]) for b in rows])
    cls = class_lut()[np.stack([w.tokens(b) for b in rows])]
    t = lambda x: torch.from_numpy(x).to(dev).to(torch.bfloat16)
    return t(q), t(k), t(v), torch.from_numpy(cls).to(dev)


def _session(w, T, chained, rows=None, kept_every=1):
    qd, kd, vd, cd = _inputs(w, rows)
    dev = qd.device
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    res, cache = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                       prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
    G = qd.shape[0] * w.H
    outs = torch.empty(w.D, G, w.d, dtype=torch.float32, device=dev)
    kept = []
    cols = [cd[:, w.N + t].contiguous() for t in range(w.D)]
    for t in range(w.D):
        p = w.N + t
        decode_step_tensors(cache, qd[:, :, p], kd[:, :, p], vd[:, :, p], cols[t],
                            out=outs[t].view(-1, w.H, w.d), chained=chained)
        if (t + 1) % kept_every == 0 or t + 1 == w.D:
            kept.append(cache.retained_positions())
    torch.cuda.synchronize()
    cache.check()
    return res, outs.cpu().numpy(), kept


@pytest.mark.parametrize("d,H", [(128, 4), (128, 12), (64, 6)])
def test_chained_steps_bit_identical(d, H):
    w = _workload(1, H, 700, 96, d, seed=5 + d + H)
    r0, o0, k0 = _session(w, 0.98, chained=False)
    r1, o1, k1 = _session(w, 0.98, chained=True)
    np.testing.assert_array_equal(r0.choice, r1.choice)
    assert not all(r0.family[c].is_full for c in r0.choice[:, 0]), "every head full: no eviction"
    np.testing.assert_array_equal(o0, o1)
    for t, (a, b) in enumerate(zip(k0, k1)):
        for g, (x, y) in enumerate(zip(a, b)):
            np.testing.assert_array_equal(x, y, err_msg=f"step {t} head {g}")


def test_more_than_2048_heads_per_call():
    """B=72 x H=32 = 2,304 heads: two launches per step (64 + 8 rows)."""
    w = _workload(72, 32, 160, 24, 128, seed=11)
    r, o, k = _session(w, 0.98, chained=True, kept_every=8)
    ra, oa, ka = _session(w, 0.98, chained=True, rows=list(range(64)), kept_every=8)
    rb, ob, kb = _session(w, 0.98, chained=True, rows=list(range(64, 72)), kept_every=8)
    G1 = 64 * w.H
    np.testing.assert_array_equal(r.choice[:G1], ra.choice)
    np.testing.assert_array_equal(r.choice[G1:], rb.choice)
    np.testing.assert_array_equal(o[:, :G1], oa)
    np.testing.assert_array_equal(o[:, G1:], ob)
    for s in range(len(k)):
        for g in range(w.B * w.H):
            ref = ka[s][g] if g < G1 else kb[s][g - G1]
            np.testing.assert_array_equal(k[s][g], ref)
    # oracle on heads of both launches
    lut = class_lut()
    fam = O.default_family(w.r_l, w.r_f)
    for b, h in [(0, 1), (63, 30), (64, 2), (71, 31), (70, 5)]:
        g = b * w.H + h
        cls = lut[w.tokens(b)].astype(np.int64)
        q, kk, v = (x.astype(np.float64) for x in w.head_qkv(b, h))
        N = w.N
        prof = O.profile_head(q[:N], kk[:N], v[:N], cls, w.slopes[h], w.sinks[h], fam, [0.98])
        assert int(r.choice[g, 0]) == int(prof.choice[0]) or \
            np.any(np.abs(prof.recoveries[:max(int(prof.choice[0]), int(r.choice[g, 0])) + 1] - 0.98) < 1e-4)
        if int(r.choice[g, 0]) != int(prof.choice[0]):
            continue
        st = O.compact_head(prof, kk[:N], v[:N], fam[prof.choice[0]], N, w.slopes[h], w.sinks[h])
        si = 0
        for t in range(w.D):
            out = O.decode_head(st, q[N + t], kk[N + t], v[N + t], N + t, cls, N)
            sc = np.abs(out).max()
            np.testing.assert_allclose(o[t, g], out, rtol=2e-2, atol=2e-2 * sc)
            if (t + 1) % 8 == 0 or t + 1 == w.D:
                np.testing.assert_array_equal(k[si][g], np.sort(st.positions),
                                              err_msg=f"head {g} step {t}")
                si += 1


@pytest.mark.parametrize("B,H,N,D,d,dtype", [(2, 6, 300, 40, 128, torch.bfloat16),
                                             (2, 6, 300, 40, 64, torch.float32),
                                             (3, 12, 420, 40, 64, torch.bfloat16),
                                             (8, 32, 520, 48, 128, torch.bfloat16)])
def test_decode_steps_call_matches_step_by_step(B, H, N, D, d, dtype):
    """akv_decode_steps (one cooperative multi-step launch for bf16 d=64/128,
    else the step loop in C++; decode_steps_tensors) gives bit-identical
    outputs, live counts and kept sets to one call per step."""
    from paper_2310_01801_b200 import decode_steps_tensors

    w = _workload(B, H, N, D, d, seed=21 + B)
    qd, kd, vd, cd = _inputs(w)
    qd, kd, vd = qd.to(dtype), kd.to(dtype), vd.to(dtype)
    dev = qd.device
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    runs = []
    for mode in ("steps", "single"):
        res, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=0.98),
                                       prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk)
        outs = torch.empty(D, B, w.H, d, dtype=torch.float32, device=dev)
        if mode == "steps":   # two calls: 17 + 23 steps
            cls = cd[:, N:].t().contiguous()
            decode_steps_tensors(c, qd[:, :, N:N + 17], kd[:, :, N:N + 17], vd[:, :, N:N + 17],
                                 cls[:17], out=outs[:17], chained=True)
            decode_steps_tensors(c, qd[:, :, N + 17:], kd[:, :, N + 17:], vd[:, :, N + 17:],
                                 cls[17:], out=outs[17:], chained=True)
        else:
            for t in range(D):
                decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t],
                                    cd[:, N + t].contiguous(), out=outs[t], chained=True)
        torch.cuda.synchronize()
        c.check()
        runs.append((res.choice.copy(), outs.cpu().numpy(), c.live.cpu().numpy(),
                     c.retained_positions(), c.seq_len))
    a, b = runs
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    assert a[4] == b[4] == N + D
    for x, y in zip(a[3], b[3]):
        np.testing.assert_array_equal(x, y)


def test_decode_steps_chunk_edges():
    """decode_steps_tensors with 1-step and 0-step calls between longer ones
    equals one decode_step_tensors call per step (outputs, live counts)."""
    from paper_2310_01801_b200 import decode_steps_tensors

    w = _workload(2, 6, 200, 12, 128, seed=77)
    qd, kd, vd, cd = _inputs(w)
    dev = qd.device
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    N, D = w.N, w.D
    runs = []
    for mode in ("steps", "single"):
        res, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=0.98),
                                       prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk)
        outs = torch.zeros(D, 2, w.H, 128, dtype=torch.float32, device=dev)
        if mode == "steps":
            cls = cd[:, N:].t().contiguous()
            t0 = 0
            for n in (1, 0, 5, 1, 0, 5):
                sl_ = slice(N + t0, N + t0 + n)
                ret = decode_steps_tensors(c, qd[:, :, sl_], kd[:, :, sl_], vd[:, :, sl_],
                                           cls[t0:t0 + n], out=outs[t0:t0 + n], chained=True)
                assert ret.shape[0] == n
                t0 += n
            assert t0 == D
        else:
            for t in range(D):
                decode_step_tensors(c, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t],
                                    cd[:, N + t].contiguous(), out=outs[t], chained=True)
        torch.cuda.synchronize()
        c.check()
        runs.append((outs.cpu().numpy(), c.live.cpu().numpy(), c.seq_len))
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2] == N + D
