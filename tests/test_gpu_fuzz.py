"""Randomised parity sweep: the CUDA path (through the C-ABI) against the CPU
oracle on seeded random small configurations - batch rows, heads, prompt
length (down to 1), head dim 16..128, fp32 / bf16, random feasible-family
order and drops, random ratios, thresholds anywhere in [0, 1], planted
local / sink biases, punctuation density, decode length - the shapes the
golden cases do not pin one by one.  The oracle itself is pinned to the
reference (tests/test_oracle_golden.py).

Bar: per-head policies and kept-index sets after encode and after every
decode step bit-exact; outputs within rtol 1e-4 (fp32) / 2e-2 (bf16) with an
rtol*max|o| floor.  Heads whose recovery of a member up to the chosen one
lies within 1e-4 of T are listed separately (the north star's near-T rule;
with the cosine criterion, heads whose chosen members' similarities lie
within 1e-4).  Nothing else is exempt: a kept-set difference at a near tie
of frequent scores fails like any other, its relative score gap in the
message (the round-2 sweep of 6,668 seeds met no such tie,
profiles/r2_fuzz.md)."""

import os

import numpy as np
import pytest
import torch

from oracle import akv_oracle as O

pytestmark = pytest.mark.gpu

ATOMS = [O.ATOM_SPECIAL, O.ATOM_PUNCT, O.ATOM_FREQUENT, O.ATOM_LOCAL]


def _api_family(order, r_l, r_f):
    from paper_2310_01801_b200 import feasible_set
    from paper_2310_01801_b200.policies import PolicyAtom

    m = {O.ATOM_SPECIAL: PolicyAtom.SPECIAL, O.ATOM_PUNCT: PolicyAtom.PUNCTUATION,
         O.ATOM_FREQUENT: PolicyAtom.FREQUENT, O.ATOM_LOCAL: PolicyAtom.LOCAL}
    return feasible_set(r_l=r_l, r_f=r_f, atom_order=[m[a] for a in order])


def _case(seed):
    rng = np.random.default_rng([seed, 4242])
    B = int(rng.integers(1, 3))
    H = int(rng.integers(1, 5))
    d = int(rng.choice([16, 32, 64, 128]))
    if seed >= WIDE_BASE:   # many heads per launch (several heads per CTA, large page plans)
        B, H, d = int(rng.choice([8, 16, 24])), int(rng.choice([16, 32])), int(rng.choice([64, 128]))
    sizes = [1, 2, 7, 33, 64, 129, 200, 300]
    if seed >= WIDE_BASE:
        sizes = [16, 33, 64, 130]
    elif seed >= LARGE_BASE:   # the large sweep: multi-page segments, long budgets
        sizes = [255, 511, 640, 1024, 1500]
    N = int(rng.choice(sizes))
    D = int(rng.integers(0, 25)) if seed < WIDE_BASE else int(rng.integers(1, 9))
    dtype = "bf16" if rng.random() < 0.5 else "f32"
    order = list(rng.permutation(ATOMS))
    if rng.random() < 0.3:
        order = order[: int(rng.integers(1, 4))]
    r_l = float(rng.choice([0.05, 0.2, 0.3, 0.5, 1.0]))
    r_f = float(rng.choice([0.05, 0.2, 0.3, 0.5, 1.0]))
    T = float(rng.choice([0.0, 0.5, 0.8, 0.9, 0.95, 0.99, 1.0]))
    x = rng.standard_normal((3, B, H, N + D, d)).astype(np.float32)
    if dtype == "bf16":
        from paper_2310_01801_b200.workloads import round_bf16

        x = round_bf16(x)
    slopes = np.where(rng.random(H) < 0.4, rng.choice([0.02, 0.05, 0.1], H), 0.0)
    sinks = np.where(rng.random(H) < 0.4, rng.choice([4.0, 8.0, 11.0], H), 0.0)
    cls = np.where(rng.random((B, N + D)) < rng.choice([0.0, 0.05, 0.3]), 2, 0).astype(np.uint8)
    cls[:, 0] = 1
    cls[rng.random((B, N + D)) < 0.02] = 1
    # selection criterion and row averaging from a separate stream (the draws
    # above stay those of the round-1 sweep): the cosine criterion
    # (profiler.py:148-178) and last-row recovery (profiler.py:84-85) on every
    # kernel path, the tcgen05 one included (bf16, d=128)
    r2 = np.random.default_rng([seed, 5151])
    crit = O.CRIT_COSINE if r2.random() < 0.2 else O.CRIT_RECOVERY
    rows = O.ROWS_LAST if r2.random() < 0.25 else O.ROWS_ALL
    return dict(B=B, H=H, d=d, N=N, D=D, dtype=dtype, order=order, r_l=r_l, r_f=r_f, T=T,
                q=x[0], k=x[1], v=x[2], slopes=slopes, sinks=sinks, cls=cls, crit=crit, rows=rows)


def _freq_gap(st, attended, cur):
    """Relative gap between the last kept and the first dropped frequent
    candidate of the oracle's decode step (policies.py:229-241 ranking)."""
    import math

    m = st.member
    if st.scores is None or not (m.atoms & O.ATOM_FREQUENT) or (m.atoms & O.ATOM_FULL):
        return np.inf
    b = max(1, math.ceil(m.r_f * cur - 1e-9))
    if b >= len(attended):
        return np.inf
    sc = st.scores[attended]
    order = np.lexsort((attended, -sc))
    hi, lo = sc[order[b - 1]], sc[order[b]]
    return (hi - lo) / max(abs(hi), 1e-300)


LARGE_BASE = 100000
WIDE_BASE = 200000
# AKV_FUZZ_SEEDS="a:b" widens the sweep (tools runs: profiles/r1_fuzz.md);
# seeds >= LARGE_BASE draw prompts of 255-1500 positions, seeds >= WIDE_BASE
# 128-768 heads per launch
_rng = os.environ.get("AKV_FUZZ_SEEDS", "0:96").split(":")
SEEDS = range(int(_rng[0]), int(_rng[1]))


@pytest.mark.parametrize("seed", SEEDS)
def test_random_configuration_matches_oracle(seed):
    from gpu_runner import run_arrays
    from paper_2310_01801_b200 import ProfilerConfig

    c = _case(seed)
    B, H, N, D = c["B"], c["H"], c["N"], c["D"]
    fam_o = O.default_family(c["r_l"], c["r_f"], c["order"])
    from paper_2310_01801_b200 import RowAveraging, SelectionCriterion

    cfg = ProfilerConfig(recovery_threshold=c["T"], feasible=_api_family(c["order"], c["r_l"],
                                                                         c["r_f"]),
                         criterion=SelectionCriterion("cosine" if c["crit"] == O.CRIT_COSINE
                                                      else "recovery"),
                         rows=RowAveraging("last" if c["rows"] == O.ROWS_LAST else "all"))
    r = run_arrays(c["q"], c["k"], c["v"], c["cls"], N, D, c["slopes"], c["sinks"], cfg,
                   dtype=torch.bfloat16 if c["dtype"] == "bf16" else torch.float32)
    res = r["res"]
    rtol = 2e-2 if c["dtype"] == "bf16" else 1e-4
    try:
        sess = O.encode_session(c["q"][:, :, :N].astype(np.float64),
                                c["k"][:, :, :N].astype(np.float64),
                                c["v"][:, :, :N].astype(np.float64),
                                c["cls"][:, :N].astype(np.int64),
                                c["slopes"], c["sinks"], fam_o, [c["T"]], rows=c["rows"],
                                criterion=c["crit"], cls_capacity=N + D)
    except ValueError as e:
        # T = 1: the reference's float64 mean row sum of the full member can
        # round below 1.0, so it finds no feasible member (profiler.py:144-145);
        # the GPU reports the full member's exact recovery 1.0 and selects
        # it.  A near-T head by definition (the north star lists those apart).
        assert c["T"] == 1.0 and "no feasible policy" in str(e), e
        ch = res.choice[:, 0]   # the GPU's choices are keep-all members at R ~ 1
        assert np.all(np.abs(res.recovery[np.arange(len(ch)), ch] - 1.0) < 1e-4)
        pytest.skip("T = 1: the reference raises ProfilerError (full member's R rounds below 1)")
    G = B * H
    skip = set()
    near_t = []
    rec_atol = 2e-4 if c["dtype"] == "bf16" else 5e-5
    cosine = c["crit"] == O.CRIT_COSINE
    for g, prof in enumerate(sess.profiles):
        cg, co = int(res.choice[g, 0]), prof.choice[0]
        np.testing.assert_allclose(res.recovery[g], prof.recoveries, rtol=0, atol=rec_atol,
                                   err_msg=f"seed {seed} head {g} recoveries")
        if cosine:
            np.testing.assert_allclose(res.cosine[g], prof.cosine, rtol=0, atol=rec_atol,
                                       err_msg=f"seed {seed} head {g} cosine")
        if cg != co:
            upto = max(cg, co) + 1
            if cosine:   # argmax with ties to the earlier member: a near tie of similarities
                assert abs(prof.cosine[cg] - prof.cosine[co]) < 1e-4, \
                    (seed, g, res.cosine[g], prof.cosine)
            else:        # only a near-T head may choose differently
                assert np.any(np.abs(prof.recoveries[:upto] - c["T"]) < 1e-4) or \
                    np.any(np.abs(res.recovery[g, :upto] - c["T"]) < 1e-4), \
                    (seed, g, res.recovery[g], prof.recoveries)
            near_t.append(g)
            skip.add(g)
            continue
        got = np.flatnonzero(r["enc_kept"][g])
        np.testing.assert_array_equal(got, np.sort(prof.kept),
                                      err_msg=f"seed {seed} head {g} encode kept set "
                                              f"(frequent boundary gap {res.topk_gap[g]:.2e})")
    keep = [g for g in range(G) if g not in skip]
    stats = {"max_rel_out_err": 0.0}
    # T = 1 puts every member that keeps all positions at R == T (rounding)
    assert c["T"] == 1.0 or len(keep) >= (G + 1) // 2, (seed, skip)
    for t in range(D):
        pos = N + t
        attended = {g: np.append(sess.heads[g].positions, pos) for g in keep}
        ref = O.decode_session_step(sess, c["q"][:, :, pos].astype(np.float64),
                                    c["k"][:, :, pos].astype(np.float64),
                                    c["v"][:, :, pos].astype(np.float64),
                                    c["cls"][:, pos].astype(np.int64))
        for g in list(keep):
            got_kept = np.flatnonzero(r["dec_kept"][t, g])
            want_kept = np.sort(sess.heads[g].positions)
            if not np.array_equal(got_kept, want_kept):
                gap = _freq_gap(sess.heads[g], attended[g], pos + 1)
                np.testing.assert_array_equal(
                    got_kept, want_kept,
                    err_msg=f"seed {seed} step {t} head {g} (frequent boundary gap {gap:.2e})")
        if not keep:   # T = 1: every head may sit at R == T
            break
        got = r["dec_out"][t]
        ref = ref.reshape(G, -1)
        sc = np.abs(ref[keep]).max()
        np.testing.assert_allclose(got[keep], ref[keep], rtol=rtol, atol=rtol * sc,
                                   err_msg=f"seed {seed} step {t}")
        err = float(np.abs(got[keep] - ref[keep]).max() / max(sc, 1e-30))
        stats["max_rel_out_err"] = max(stats["max_rel_out_err"], err)
    stats_path = os.environ.get("AKV_FUZZ_STATS")
    if stats_path:   # one JSON line per seed for tools/fuzz_report.py
        import json

        stats.update(seed=seed, dtype=c["dtype"], N=N, D=D, d=c["d"], G=G, T=c["T"],
                     criterion="cosine" if cosine else "recovery",
                     rows="last" if c["rows"] == O.ROWS_LAST else "all",
                     compared=len(keep), skipped=len(skip), near_t_heads=near_t,
                     near_tie_encode_heads=[], decode_ties=0, near_tie_decode=[],
                     head_steps=D * len(keep),
                     evict_steps=int(sum(1 for t in range(1, D) for g in keep
                                         if r["dec_kept"][t, g].sum() <= r["dec_kept"][t - 1, g].sum())))
        with open(f"{stats_path}.{os.getpid()}", "a") as f:
            f.write(json.dumps(stats) + "\n")
