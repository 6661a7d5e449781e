"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py [case ...]

For every case in ``cases.py`` this drives the reference's public API
(``prompt_head_data``/``recovery_ratio``/``profile_model``/``encode_prompt``/
``generate_step``) through a duck-typed array model over the
seeded workload tensors.  The planted head bias is folded exactly into
two extra Q/K dimensions (q'=[q*sqrt(d')/sqrt(d), 1, 1],
k'=[k, slope*j*sqrt(d'), sink*sqrt(d')*[special]]), because the reference
has no logit-bias hook; under the causal softmax -slope*|i-j| equals
+slope*j up to a row constant.  Decode is teacher-forced with the
workload's own token ids.  Outputs are written to ``tests/golden/*.npz``.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)

import cases as C  # noqa: E402
from adaptive_kv import (  # noqa: E402
    ProfilerConfig, RowAveraging, SelectionCriterion, encode_prompt,
    feasible_set, generate_step, parse_policy, profile_model, recovery_ratio,
    retained_indices,
)
from adaptive_kv.engine import prompt_head_data  # noqa: E402
from adaptive_kv.model import ModelConfig, SyntheticModel  # noqa: E402
from adaptive_kv.policies import PolicyAtom, cache_memory_cost  # noqa: E402
from adaptive_kv.profiler import masked_cosine_similarity  # noqa: E402
from adaptive_kv.tokens import TokenClass, VocabMetadata  # noqa: E402

from paper_2310_01801_b200.workloads import PUNCT_IDS, SPECIAL_IDS, VOCAB_SIZE  # noqa: E402

ATOM_BITS = {PolicyAtom.SPECIAL: 1, PolicyAtom.PUNCTUATION: 2, PolicyAtom.FREQUENT: 4,
             PolicyAtom.LOCAL: 8, PolicyAtom.FULL: 16}
NAME_ATOM = {"special": PolicyAtom.SPECIAL, "punct": PolicyAtom.PUNCTUATION,
             "frequent": PolicyAtom.FREQUENT, "local": PolicyAtom.LOCAL}


def atom_bits(policy) -> int:
    return sum(ATOM_BITS[a] for a in policy.atoms)


class ArrayModel:
    """Duck-typed reference model (model.py:150-286 protocol) over arrays
    q,k,v [G, T, d] (float64) of one token sequence, with the planted bias
    folded into two extra dimensions."""

    def __init__(self, q, k, v, slopes, sinks, vocab):
        self.q, self.k, self.v = q, k, v
        self.slopes, self.sinks = slopes, sinks
        g, _, d = q.shape
        self.d = d
        self.d2 = d + 2
        self.config = ModelConfig(num_layers=1, num_heads=g, head_dim=d + 2,
                                  vocab_size=1, seed=0)
        self.vocab = vocab
        self._qscale = math.sqrt(self.d2) / math.sqrt(d)

    def k_row(self, layer, head, pos, klass, prompt_len):
        row = np.zeros(self.d2)
        row[: self.d] = self.k[head, pos]
        row[self.d] = self.slopes[head] * pos * math.sqrt(self.d2)
        row[self.d + 1] = self.sinks[head] * math.sqrt(self.d2) * (klass is TokenClass.SPECIAL)
        return row

    def q_row(self, layer, head, pos, prompt_len):
        row = np.ones(self.d2)
        row[: self.d] = self.q[head, pos] * self._qscale
        return row

    def v_row(self, layer, head, pos):
        return self.v[head, pos].copy()

    def head_logits(self, concat):
        return np.zeros(1)


def profiler_cfg(w, opts, T):
    order = [NAME_ATOM[a] for a in opts.get("order", C.ORDER_DEFAULT)]
    drop = [NAME_ATOM[a] for a in opts.get("drop", ())]
    fam = feasible_set(r_l=w.r_l, r_f=w.r_f, atom_order=order, drop=drop)
    return ProfilerConfig(
        recovery_threshold=T, feasible=fam,
        criterion=SelectionCriterion(opts.get("criterion", "recovery")),
        rows=RowAveraging(opts.get("rows", "all")))


def run_sequence(model, tokens, N, D, cfg_list, decode_cfg, fixed):
    """Reference run for one token sequence: per-head profiling tables for
    every threshold in cfg_list, then a teacher-forced decode session."""
    grid = model.config.head_grid()
    _, _, head_data = prompt_head_data(model, list(tokens[:N]))
    fam = cfg_list[0].feasible if fixed is None else (fixed,)
    rows = cfg_list[0].rows
    R = np.zeros((len(grid), len(fam)))
    cost = np.zeros((len(grid), len(fam)), dtype=np.int64)
    cos = np.zeros((len(grid), len(fam)))
    colsum = np.zeros((len(grid), N))
    lastrow = np.zeros((len(grid), N))
    for gi, key in enumerate(grid):
        A, ctx = head_data[key]
        colsum[gi] = ctx.cumulative_scores
        lastrow[gi] = A.matrix[N - 1]
        for fi, pol in enumerate(fam):
            ret = retained_indices(pol, ctx)
            R[gi, fi] = recovery_ratio(A, ret, rows)
            cost[gi, fi] = cache_memory_cost(pol, ctx)
            cos[gi, fi] = masked_cosine_similarity(A, ret)
    csvs, choice = [], np.zeros((len(grid), len(cfg_list)), dtype=np.int64)
    if fixed is None:
        for ti, cfg in enumerate(cfg_list):
            prof = profile_model(head_data, cfg, grid=grid)
            csvs.append(prof.to_csv())
            for gi, key in enumerate(grid):
                choice[gi, ti] = list(cfg.feasible).index(prof[key].policy)

    # decode session (engine.py:203-371), teacher-forced
    if fixed is None:
        prof, cache = encode_prompt(model, list(tokens[:N]), decode_cfg, diagnostics=True)
    else:
        prof, cache = encode_prompt(model, list(tokens[:N]), None, fixed_policy=fixed,
                                    diagnostics=True)
        csvs.append(prof.to_csv())
    total = N + D
    enc_kept = np.zeros((len(grid), N), dtype=bool)
    enc_out = np.zeros((len(grid), model.v.shape[-1]))
    enc_rec = np.zeros(len(grid))
    dec_choice = np.zeros(len(grid), dtype=np.int64)
    for gi, key in enumerate(grid):
        st = cache.heads[key]
        enc_kept[gi, st.positions] = True
        enc_out[gi] = st.pending_output
        enc_rec[gi] = prof[key].recovery
        dec_choice[gi] = list(fam).index(st.policy)
    generate_step(model, cache, None)
    # diagnostics: per-head recovery vs the uncompressed shadow softmax
    # (engine.py:341-349); row 0 is the first (sampling-only) step, whose
    # recoveries are the prompt's last-row recoveries (engine.py:362-363)
    dec_rec = np.zeros((D + 1, len(grid)))
    dec_mean = np.zeros(D + 1)
    dec_rec[0] = [cache.heads[key].last_row_recovery for key in grid]
    dec_mean[0] = cache.last_record.mean_recovery
    dec_kept = np.zeros((D, len(grid), total), dtype=bool)
    dec_out = np.zeros((D, len(grid), model.v.shape[-1]))
    for t in range(D):
        generate_step(model, cache, int(tokens[N + t]))
        rec = cache.last_record.retained_positions
        dec_mean[t + 1] = cache.last_record.mean_recovery
        for gi, key in enumerate(grid):
            dec_kept[t, gi, list(rec[key])] = True
            dec_out[t, gi] = cache.heads[key].pending_output
            dec_rec[t + 1, gi] = cache.heads[key].last_row_recovery
    return dict(R=R, cost=cost, cos=cos, colsum=colsum, lastrow=lastrow, choice=choice,
                csvs=csvs, enc_kept=enc_kept, enc_out=enc_out, enc_rec=enc_rec,
                dec_choice=dec_choice, dec_kept=dec_kept, dec_out=dec_out, dec_rec=dec_rec,
                dec_mean=dec_mean,
                family=np.array([atom_bits(p) for p in fam]))


def make_workload_case(name):
    w, opts = C.case_workload(name)
    heads = C.case_heads(w, opts)
    vocab = VocabMetadata(special_ids=frozenset(SPECIAL_IDS), punctuation_ids=frozenset(PUNCT_IDS))
    fixed = parse_policy(opts["fixed"]) if "fixed" in opts else None
    cfg_list = [profiler_cfg(w, opts, T) for T in w.thresholds]
    decode_cfg = profiler_cfg(w, opts, opts.get("decode_T", w.thresholds[0]))
    per_b = {}
    for b, h in heads:
        per_b.setdefault(b, []).append(h)
    parts, tokens = [], {}
    for b, hs in sorted(per_b.items()):
        tok = w.tokens(b)
        tokens[b] = tok
        qs, ks, vs = zip(*(w.head_qkv(b, h) for h in hs))
        model = ArrayModel(np.stack(qs).astype(np.float64), np.stack(ks).astype(np.float64),
                           np.stack(vs).astype(np.float64), w.slopes[hs], w.sinks[hs], vocab)
        parts.append(run_sequence(model, tok, w.N, w.D, cfg_list, decode_cfg, fixed))
    out = {}
    for key in ("R", "cost", "cos", "colsum", "lastrow", "choice", "enc_kept", "enc_out",
                "enc_rec", "dec_choice"):
        out[key] = np.concatenate([p[key] for p in parts], axis=0)
    out["dec_kept"] = np.packbits(np.concatenate([p["dec_kept"] for p in parts], axis=1), axis=-1)
    out["enc_kept"] = np.packbits(out["enc_kept"], axis=-1)
    out["dec_out"] = np.concatenate([p["dec_out"] for p in parts], axis=1)
    out["dec_rec"] = np.concatenate([p["dec_rec"] for p in parts], axis=1)
    out["dec_mean"] = np.stack([p["dec_mean"] for p in parts])  # [batch rows, D+1]
    out["family"] = parts[0]["family"]
    # CSV per threshold, one block per batch row (the reference grid is per sequence)
    out["csvs"] = np.array(["\n---\n".join(p["csvs"][i] for p in parts)
                            for i in range(len(parts[0]["csvs"]))])
    out["heads"] = np.array(heads, dtype=np.int64)
    out["tokens"] = np.stack([tokens[b] for b in sorted(tokens)])
    np.savez_compressed(C.golden_path(name), **out)


def make_mixed():
    sys.path.insert(0, REF_TESTS)
    from conftest import MIXED_PLAN_4X4  # the reference's own fixture

    m = C.MIXED
    cfgm = ModelConfig(num_layers=4, num_heads=4, head_dim=16, vocab_size=48, seed=m["seed"])
    model = SyntheticModel(cfgm, MIXED_PLAN_4X4, dominance=m["dominance"])
    P, S = m["prompt_len"], m["steps"]
    prompt = model.prompt_token_ids(P)
    cfg = ProfilerConfig(recovery_threshold=m["T"])
    prof, cache = encode_prompt(model, prompt, cfg, diagnostics=True)
    grid = sorted(cfgm.head_grid())
    enc_kept = np.zeros((len(grid), P), dtype=bool)
    enc_out = np.zeros((len(grid), 16))
    for gi, key in enumerate(grid):
        enc_kept[gi, cache.heads[key].positions] = True
        enc_out[gi] = cache.heads[key].pending_output
    tok, _ = generate_step(model, cache, None)
    tokens = list(prompt)
    dec_kept = np.zeros((S, len(grid), P + S), dtype=bool)
    dec_out = np.zeros((S, len(grid), 16))
    dec_rec = np.zeros((S + 1, len(grid)))
    dec_rec[0] = [cache.heads[key].last_row_recovery for key in grid]
    for t in range(S):
        tokens.append(tok)
        tok, _ = generate_step(model, cache, tokens[-1])
        rec = cache.last_record.retained_positions
        for gi, key in enumerate(grid):
            dec_kept[t, gi, list(rec[key])] = True
            dec_out[t, gi] = cache.heads[key].pending_output
            dec_rec[t + 1, gi] = cache.heads[key].last_row_recovery
    T = len(tokens)
    klass = [model.vocab.classify_id(t) for t in tokens]
    q = np.zeros((len(grid), T, 16))
    k = np.zeros((len(grid), T, 16))
    v = np.zeros((len(grid), T, 16))
    for gi, (l, h) in enumerate(grid):
        for p in range(T):
            q[gi, p] = model.q_row(l, h, p, P)
            k[gi, p] = model.k_row(l, h, p, klass[p], P)
            v[gi, p] = model.v_row(l, h, p)
    choice = np.array([list(cfg.feasible).index(prof[key].policy) for key in grid])
    np.savez_compressed(
        C.golden_path(m["name"]), q=q, k=k, v=v, tokens=np.array(tokens),
        special=np.array(sorted(model.vocab.special_ids)),
        punct=np.array(sorted(model.vocab.punctuation_ids)),
        choice=choice, csv=np.array(prof.to_csv()),
        enc_kept=np.packbits(enc_kept, axis=-1), enc_out=enc_out,
        dec_kept=np.packbits(dec_kept, axis=-1), dec_out=dec_out, dec_rec=dec_rec)


def make_metrics():
    """Reference metrics.py reports (tradeoff_curve, consistency_report,
    compare_adaptive_vs_fixed, layer_distribution_report and their CSV /
    JSON renderings) on the FoldedArrayModel of metrics_model.py."""
    import json

    import metrics_model as MM
    from adaptive_kv import metrics as RM
    from adaptive_kv.engine import GenerationConfig, generate

    vocab = VocabMetadata(special_ids=frozenset(MM.SPECIAL), punctuation_ids=frozenset(MM.PUNCT))
    model = MM.FoldedArrayModel(vocab, TokenClass.SPECIAL)
    prompt = model.prompt_token_ids()
    T_values = [0.5, 0.8, 0.9, 0.95, 0.98, 0.99, 0.995, 0.999, 1.0]
    points = RM.tradeoff_curve(model, prompt, T_values)
    cfg = ProfilerConfig(recovery_threshold=0.95)
    entries = RM.consistency_report(model, prompt, [1, 4, 9, 17], cfg, max_new_tokens=24)
    gen_cfg = GenerationConfig(max_new_tokens=12)
    fixed = [parse_policy("special+punct+frequent(r_f=0.3)+local(r_l=0.3)"),
             parse_policy("frequent(r_f=0.25)"), parse_policy("local(r_l=0.2)")]
    extra = {"drop_punct": ProfilerConfig(recovery_threshold=0.95,
                                          feasible=feasible_set(drop=[PolicyAtom.PUNCTUATION]))}
    rows = RM.compare_adaptive_vs_fixed(model, prompt, cfg, fixed, gen_cfg, extra_adaptive=extra)
    adaptive = generate(model, prompt, cfg, gen_cfg)
    prof = adaptive.profile
    dist = RM.layer_distribution_report(prof)
    reports = {
        "tradeoff": RM.tradeoff_rows(points), "consistency": RM.consistency_rows(entries),
        "comparison": RM.comparison_rows(rows), "layers": RM.layer_distribution_rows(dist),
    }
    np.savez_compressed(
        C.golden_path("metrics"),
        T=np.array([p.T for p in points]), pruned=np.array([p.pruned_ratio for p in points]),
        mean_rec=np.array([p.mean_recovery for p in points]),
        cons_step=np.array([e.step for e in entries]),
        cons_key=np.array([(e.layer, e.head) for e in entries]),
        cons_policy=np.array([e.policy for e in entries]),
        cons_match=np.array([e.matches_first for e in entries]),
        cmp_method=np.array([r.method for r in rows]),
        cmp_pruned=np.array([r.pruned_ratio for r in rows]),
        cmp_rec=np.array([r.mean_step_recovery for r in rows]),
        gen_tokens=np.array(adaptive.tokens), profile_csv=np.array(prof.to_csv()),
        layers_json=np.array(json.dumps({str(k): v for k, v in dist.items()}, sort_keys=True)),
        csv=np.array([RM.rows_to_csv(*reports[k]) for k in sorted(reports)]),
        json=np.array([RM.rows_to_json(k, *reports[k]) for k in sorted(reports)]),
        report_names=np.array(sorted(reports)),
        stability=np.array(RM.stability_fraction(entries)))


def make_trace():
    """AKVT files written by the reference (binary + NDJSON) of a recorded
    run of the reference's small_model fixture (pkg/tests/conftest.py:64-73,
    the recording of test_trace.py:124-162), plus the reference's generate()
    replayed from that trace: tokens, profile CSV, per-step retained counts
    and mean recoveries."""
    from adaptive_kv.engine import GenerationConfig, generate, reference_generate
    from adaptive_kv.model import Archetype, HeadPlan
    from adaptive_kv.tokens import TokenAnnotation
    from adaptive_kv.trace import (AttentionTrace, TraceBlock, TraceModel, read_trace,
                                   write_trace, write_trace_ndjson)

    config = ModelConfig(num_layers=2, num_heads=2, head_dim=16, vocab_size=32, seed=7)
    plan = {(0, 0): HeadPlan(Archetype.SPECIAL_DOMINANT), (0, 1): HeadPlan(Archetype.LOCAL_DOMINANT),
            (1, 0): HeadPlan(Archetype.COLUMN_SPARSE), (1, 1): HeadPlan(Archetype.DIFFUSE)}
    model = SyntheticModel(config, plan, dominance=0.97)
    prompt_len, steps = 24, 8
    prompt = model.prompt_token_ids(prompt_len)
    ref = reference_generate(model, prompt, GenerationConfig(max_new_tokens=steps))
    all_tokens = prompt + ref.tokens[: steps - 1]
    ann = [TokenAnnotation(p, t, model.vocab.classify_id(t)) for p, t in enumerate(all_tokens)]
    blocks = {key: [TraceBlock(step=p, k=model.k_row(*key, p, ann[p].klass, prompt_len),
                               v=model.v_row(*key, p), q=model.q_row(*key, p, prompt_len))
                    for p in range(len(all_tokens))] for key in config.head_grid()}
    trace = AttentionTrace(config, ann, blocks)
    write_trace(trace, os.path.join(C.HERE, "replay.akvt"))
    write_trace_ndjson(trace, os.path.join(C.HERE, "replay.ndjson"))
    replay = TraceModel(read_trace(os.path.join(C.HERE, "replay.akvt")))
    res = generate(replay, prompt, ProfilerConfig(recovery_threshold=0.95),
                   GenerationConfig(max_new_tokens=steps))
    grid = config.head_grid()
    np.savez_compressed(
        C.golden_path("replay"), prompt_len=prompt_len, steps=steps,
        tokens=np.array(res.tokens), profile_csv=np.array(res.profile.to_csv()),
        retained=np.array([[r.head_retained[k] for k in grid] for r in res.records]),
        mean_rec=np.array([r.mean_recovery for r in res.records]),
        retained_pos=np.array([json.dumps({f"{k[0]},{k[1]}": list(r.retained_positions[k])
                                           for k in grid}) for r in res.records]))


NUCLEUS = ((0.8, 0.9, 3), (1.5, 0.5, 11), (0.3, 1.0, 0))


def make_nucleus():
    """The reference's nucleus sampler (engine.py:71-90): (1) tokens drawn by
    its _Sampler from seeded logit vectors; (2) generate() with Nucleus on
    the recorded replay trace (replay.akvt, written by make_trace)."""
    from adaptive_kv.engine import GenerationConfig, Nucleus, _Sampler, generate
    from adaptive_kv.trace import TraceModel, read_trace

    rng = np.random.default_rng(2024)
    logits = rng.standard_normal((64, 40)) * 3.0
    draws = []
    for temp, top_p, seed in NUCLEUS:
        smp = _Sampler(Nucleus(temperature=temp, top_p=top_p, seed=seed))
        draws.append([smp(row) for row in logits])
    z = dict(np.load(C.golden_path("replay")))
    P, S = int(z["prompt_len"]), int(z["steps"])
    model = TraceModel(read_trace(os.path.join(C.HERE, "replay.akvt")))
    prompt = model.prompt_token_ids(P)
    gen = []
    for temp, top_p, seed in NUCLEUS:
        res = generate(model, prompt, ProfilerConfig(recovery_threshold=0.95),
                       GenerationConfig(max_new_tokens=S,
                                        sampling=Nucleus(temperature=temp, top_p=top_p, seed=seed)))
        gen.append(res.tokens)
    np.savez_compressed(C.golden_path("nucleus"), params=np.array(NUCLEUS), logits=logits,
                        draws=np.array(draws), gen_tokens=np.array(gen))


def main(argv):
    names = argv or list(C.CASES) + [C.MIXED["name"], "metrics", "replay", "nucleus"]
    for name in names:
        t0 = time.time()
        if name == C.MIXED["name"]:
            make_mixed()
        elif name == "metrics":
            make_metrics()
        elif name == "replay":
            make_trace()
        elif name == "nucleus":
            make_nucleus()
        else:
            make_workload_case(name)
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
