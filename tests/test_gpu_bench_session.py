"""The headline session itself against the oracle: bench.py's config-1
workload (B=8, H=32, N=1024, D=512, bf16, T=0.95, seed 1) through exactly
the path bench.py times - device arena pool, K1 + K2 enqueued without a host
round trip, 512 chained K3 steps over all 256 heads - with the kept-index
sets of sampled heads (every planted head of two batch rows plus a plain
one) compared bit-exactly with the CPU oracle after encode and at
checkpoints through the session, and their outputs within the bf16
tolerance (rtol 2e-2, floor 2e-2 * max|o|)."""

import numpy as np
import pytest
import torch

from oracle import akv_oracle as O

pytestmark = pytest.mark.gpu

CHECKPOINTS = (1, 2, 64, 200, 383, 512)   # steps completed


def test_bench_session_matches_oracle_on_sampled_heads():
    import bench
    from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors
    from paper_2310_01801_b200.workloads import class_lut, config1

    dev = torch.device("cuda")
    w = config1(seed=1)
    T = w.thresholds[0]
    N, D, H = w.N, w.D, w.H
    qd, kd, vd, cd, q, k, v, cls = bench.make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev)
    sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    pool = bench.arena_pool(w, dev)
    pool.reset()
    res, cache = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=T),
                                       prompt_len=N, max_new_tokens=D, slopes=sl, sinks=sk,
                                       pool=pool)
    planted = [h for h in range(H) if w.slopes[h] or w.sinks[h]]
    plain = [h for h in range(H) if h not in planted][:1]
    heads = [(b, h) for b in (0, 5) for h in planted + plain]
    gidx = [b * H + h for b, h in heads]
    kept = {0: [cache.retained_positions()[g] for g in gidx]}
    outs = {}
    dc = [cd[:, N + t].contiguous() for t in range(D)]
    for t in range(D):
        o = decode_step_tensors(cache, qd[:, :, N + t], kd[:, :, N + t], vd[:, :, N + t], dc[t],
                                chained=True)
        if t + 1 in CHECKPOINTS:
            pos = cache.retained_positions()
            kept[t + 1] = [pos[g] for g in gidx]
            outs[t + 1] = o.reshape(-1, w.d)[gidx].cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    cache.check()

    lut = class_lut()
    fam = O.default_family(w.r_l, w.r_f)
    compressed = 0
    for i, (b, h) in enumerate(heads):
        cls_b = lut[w.tokens(b)].astype(np.int64)
        qh, kh, vh = (x[b, h].astype(np.float64) for x in (q, k, v))
        prof = O.profile_head(qh[:N], kh[:N], vh[:N], cls_b, w.slopes[h], w.sinks[h], fam, [T])
        g = gidx[i]
        assert int(res.choice[g, 0]) == prof.choice[0], (b, h, res.recovery[g], prof.recoveries)
        st = O.compact_head(prof, kh[:N], vh[:N], fam[prof.choice[0]], N, w.slopes[h], w.sinks[h])
        compressed += fam[prof.choice[0]].atoms != O.ATOM_FULL
        np.testing.assert_array_equal(np.sort(kept[0][i]), np.sort(st.positions))
        for t in range(D):
            o = O.decode_head(st, qh[N + t], kh[N + t], vh[N + t], N + t, cls_b, N)
            if t + 1 in CHECKPOINTS:
                np.testing.assert_array_equal(np.sort(kept[t + 1][i]), np.sort(st.positions),
                                              err_msg=f"head {(b, h)} after step {t + 1}")
                ref = np.asarray(o, np.float64)
                got = outs[t + 1][i]
                np.testing.assert_allclose(got, ref, rtol=2e-2, atol=2e-2 * np.abs(ref).max(),
                                           err_msg=f"head {(b, h)} output of step {t + 1}")
    assert compressed >= 4   # the sample exercises evicting heads, not only full ones
