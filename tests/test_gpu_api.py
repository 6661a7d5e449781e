"""The reference's single-context API on the GPU: the cases of the
reference's own unit tests (pkg/tests/test_attention.py, test_policies.py),
restated against paper_2310_01801_b200's kernel-backed functions, the SPEC
examples verified against the reference, and profile_model on
the reference's MIXED_PLAN_4X4 fixture against its golden profile."""

import math

import numpy as np
import pytest

import cases as C
from paper_2310_01801_b200 import (AttentionError, AttentionMap, CompressionPolicy, HeadProfile,
                                   PolicyAtom, PolicyContext, PolicyError, ProfilerConfig,
                                   RetainedSet, RowAveraging, apply_policy, cache_memory_cost,
                                   causal_attention, feasible_set, full_policy,
                                   masked_cosine_similarity, profile_model, recovery_ratio,
                                   retained_indices, select_policy, select_policy_by_similarity,
                                   softmax_rows, softmax_vector, tv_distance_row,
                                   update_cumulative_scores)
from paper_2310_01801_b200.tokens import TokenAnnotation, TokenClass

pytestmark = pytest.mark.gpu

S, P, O = TokenClass.SPECIAL, TokenClass.PUNCTUATION, TokenClass.OTHER


def anns(classes):
    return tuple(TokenAnnotation(pos, 100 + pos, k) for pos, k in enumerate(classes))


def ctx_of(classes, prompt_len=None, scores=None):
    n = len(classes)
    return PolicyContext(anns(classes), prompt_len if prompt_len is not None else n, n,
                         np.zeros(n) if scores is None else np.asarray(scores, float))


def random_context(rng, max_len=24):
    cur = int(rng.integers(1, max_len + 1))
    plen = int(rng.integers(1, cur + 1))
    classes = [[S, P, O][i] for i in rng.integers(0, 3, size=cur)]
    return PolicyContext(anns(classes), plen, cur, rng.uniform(0.0, 5.0, size=cur))


def atom(a, **kw):
    return CompressionPolicy(frozenset({a}), **kw)


# ---- attention (test_attention.py) ----
def test_softmax_kats():
    assert softmax_rows([[0.0, 0.0]])[0] == pytest.approx([0.5, 0.5], abs=1e-12)
    assert softmax_rows([[math.log(2.0), 0.0]])[0] == pytest.approx([2 / 3, 1 / 3], abs=1e-12)
    out = softmax_rows([[1000.0, 0.0]])
    assert np.all(np.isfinite(out)) and out[0, 0] == pytest.approx(1.0, abs=1e-12) and out[0, 1] < 1e-300
    with pytest.raises(AttentionError, match="empty input"):
        softmax_rows(np.zeros((0, 0)))
    with pytest.raises(AttentionError, match="empty input"):
        softmax_vector([])
    m = softmax_rows(np.ones((3, 3)), causal_lengths=[1, 2, 3])
    assert m[0, 1] == 0.0 and m[0, 2] == 0.0 and m[1, 2] == 0.0
    assert np.allclose(m.sum(axis=1), 1.0, atol=1e-12)


def test_causal_attention_kats():
    V = np.array([[4.0, -1.0]])
    A, out = causal_attention(np.array([[1.0, 0.0]]), np.array([[2.0, 3.0]]), V, 2)
    assert A.matrix.shape == (1, 1) and A.matrix[0, 0] == 1.0
    assert out[0] == pytest.approx(V[0])
    A, out = causal_attention(np.array([[1.0], [2.0]]), np.array([[1.0], [-1.0]]),
                              np.array([[3.0], [5.0]]), 1)
    w0 = math.exp(2.0) / (math.exp(2.0) + math.exp(-2.0))
    assert A.matrix[0] == pytest.approx([1.0, 0.0], abs=1e-15)
    assert A.matrix[1] == pytest.approx([w0, 1 - w0], abs=1e-15)
    assert out[1, 0] == pytest.approx(3.0 * w0 + 5.0 * (1 - w0), abs=1e-12)
    rng = np.random.default_rng(5)
    for _ in range(20):
        n, d = int(rng.integers(1, 12)), int(rng.integers(1, 6))
        A, _ = causal_attention(rng.normal(size=(n, d)), rng.normal(size=(n, d)),
                                rng.normal(size=(n, d)), d)
        assert np.abs(A.matrix.sum(axis=1) - 1.0).max() <= 1e-9
        assert np.all(np.triu(A.matrix, k=1) == 0.0)
    with pytest.raises(AttentionError, match="V has 3 rows"):
        causal_attention(np.zeros((2, 3)), np.zeros((2, 3)), np.zeros((3, 3)), 3)
    with pytest.raises(AttentionError, match="K has 3 columns"):
        causal_attention(np.zeros((2, 2)), np.zeros((2, 3)), np.zeros((2, 2)), 2)


def test_attention_map_invariants():
    with pytest.raises(AttentionError, match="square"):
        AttentionMap(np.ones((2, 3)) / 3.0)
    with pytest.raises(AttentionError, match="sum to 1"):
        AttentionMap(np.array([[0.4, 0.0], [0.5, 0.5]]))
    with pytest.raises(AttentionError, match="causal"):
        AttentionMap(np.array([[0.5, 0.5], [0.5, 0.5]]))
    A = AttentionMap(np.array([[1.0, 0.0], [0.5, 0.5]]))
    with pytest.raises(ValueError):
        A.matrix[0, 0] = 2.0


# ---- policies (test_policies.py) ----
def test_atom_kats():
    assert retained_indices(atom(PolicyAtom.LOCAL, r_l=0.3), ctx_of([O] * 10)).indices == (7, 8, 9)
    ctx = ctx_of([O] * 4, scores=[0.9, 0.05, 0.03, 0.02])
    assert retained_indices(atom(PolicyAtom.FREQUENT, r_f=0.5), ctx).indices == (0, 1)
    ctx = ctx_of([O] * 6, scores=[1.0, 2.0, 2.0, 2.0, 1.0, 1.0])
    assert retained_indices(atom(PolicyAtom.FREQUENT, r_f=0.5), ctx).indices == (1, 2, 3)
    hybrid = CompressionPolicy(frozenset({PolicyAtom.SPECIAL, PolicyAtom.PUNCTUATION,
                                          PolicyAtom.LOCAL}), r_l=0.2)
    assert retained_indices(hybrid, ctx_of([S, O, O, O, O, P, O, O, O, O])).indices == (0, 5, 8, 9)
    assert retained_indices(full_policy(), ctx_of([O] * 7)).indices == tuple(range(7))
    assert len(retained_indices(atom(PolicyAtom.SPECIAL), ctx_of([O] * 5))) == 0
    ctx = ctx_of([O] * 10, scores=[9, 8, 7, 6, 5, 4, 3, 2, 1, 0])
    pol = atom(PolicyAtom.FREQUENT, r_f=0.3)
    assert retained_indices(pol, ctx).indices == (0, 1, 2)
    assert retained_indices(pol, ctx, candidates=[2, 5, 7, 9]).indices == (2, 5, 7)
    with pytest.raises(PolicyError, match=">= current_len"):
        retained_indices(pol, ctx, candidates=[10])


def test_policy_properties_random():
    rng = np.random.default_rng(30)
    fam = feasible_set(r_l=0.25, r_f=0.25)
    a = CompressionPolicy(frozenset({PolicyAtom.SPECIAL, PolicyAtom.LOCAL}))
    b = atom(PolicyAtom.FREQUENT)
    for _ in range(40):
        ctx = random_context(rng)
        sets = [set(retained_indices(p, ctx)) for p in fam]
        assert all(x <= y for x, y in zip(sets, sets[1:]))
        assert sets[-1] == set(range(ctx.current_len))
        assert set(retained_indices(a.union(b), ctx)) == set(retained_indices(a, ctx)) | set(
            retained_indices(b, ctx))
        r_l = int(rng.integers(1, 17)) / 16.0
        r_f = int(rng.integers(1, 17)) / 16.0
        assert len(retained_indices(atom(PolicyAtom.LOCAL, r_l=r_l), ctx)) == min(
            math.ceil(r_l * ctx.prompt_len), ctx.current_len)
        assert cache_memory_cost(atom(PolicyAtom.FREQUENT, r_f=r_f), ctx) == math.ceil(
            r_f * ctx.current_len)


def test_apply_policy():
    K = np.arange(8.0).reshape(4, 2)
    V = -K
    K_C, V_C = apply_policy(K, V, RetainedSet.of(range(4)))
    assert np.array_equal(K_C, K) and np.array_equal(V_C, V)
    K_E, V_E = apply_policy(K, V, RetainedSet.of([]))
    assert K_E.shape == (0, 2) and V_E.shape == (0, 2)
    K_S, _ = apply_policy(K, V, RetainedSet.of([0, 3]))
    assert np.array_equal(K_S, K[[0, 3]])
    with pytest.raises(PolicyError, match="out of range"):
        apply_policy(np.zeros((4, 2)), np.zeros((4, 2)), RetainedSet.of([4]))


def test_update_scores():
    ctx = ctx_of([O] * 4, scores=[0.3, 0.3, 0.2, 0.2])
    out = update_cumulative_scores(ctx, np.array([0.4, 0.3, 0.2, 0.1]), RetainedSet.of(range(4)))
    assert out.current_len == 5 and out.cumulative_scores.sum() == pytest.approx(2.0)
    assert out.cumulative_scores[-1] == 0.0
    ctx = ctx_of([O] * 3, scores=[1.0, 2.0, 3.0])
    assert update_cumulative_scores(ctx, np.zeros(0), RetainedSet.of([])).cumulative_scores.tolist() == [1, 2, 3, 0]
    ctx = ctx_of([O] * 4, scores=[5.0, 1.0, 1.0, 1.0])
    out = update_cumulative_scores(ctx, np.array([0.7, 0.3]), RetainedSet.of([1, 3]))
    assert out.cumulative_scores.tolist() == [5.0, 1.7, 1.0, 1.3, 0.0]
    with pytest.raises(PolicyError, match="one score per retained"):
        update_cumulative_scores(ctx_of([O] * 3), np.zeros(3), RetainedSet.of([0, 1]))


# ---- profiler (SPEC examples) ----
def test_spec_examples():
    A4, _ = causal_attention(np.zeros((4, 1)), np.zeros((4, 1)), np.zeros((4, 1)), 1)
    assert recovery_ratio(A4, RetainedSet.of([0])) == pytest.approx((1 + 1 / 2 + 1 / 3 + 1 / 4) / 4, abs=1e-12)
    assert recovery_ratio(A4, RetainedSet.of(range(4))) == pytest.approx(1.0)
    assert recovery_ratio(A4, RetainedSet.of([])) == 0.0
    assert tv_distance_row([0.6, 0.3, 0.1], RetainedSet.of([0, 1])) == pytest.approx(0.1, abs=1e-12)
    assert tv_distance_row([0.6, 0.3, 0.1], RetainedSet.of([])) == 1.0
    A2 = AttentionMap(np.array([[1.0, 0.0], [0.5, 0.5]]))
    assert masked_cosine_similarity(A2, RetainedSet.of([0])) == pytest.approx(0.912870929175277, abs=1e-12)
    A10, _ = causal_attention(np.zeros((10, 1)), np.zeros((10, 1)), np.zeros((10, 1)), 1)
    ctx = ctx_of([S] + [O] * 9, scores=A10.matrix.sum(axis=0))
    pol, _ = select_policy(A10, ctx, ProfilerConfig(recovery_threshold=0.95))
    assert pol.is_full
    pol, _ = select_policy(A10, ctx, ProfilerConfig(recovery_threshold=0.0))
    assert pol.atoms == {PolicyAtom.SPECIAL}
    mass0 = np.zeros((10, 10))
    mass0[:, 0] = 1.0
    A0 = AttentionMap(mass0)
    pol, r = select_policy(A0, ctx_of([S] + [O] * 9, scores=mass0.sum(0)), ProfilerConfig(recovery_threshold=0.99))
    assert pol.atoms == {PolicyAtom.SPECIAL} and r == pytest.approx(1.0)
    fam = feasible_set()
    assert select_policy_by_similarity(A10, fam, ctx).is_full


def test_profile_model_matches_reference_on_mixed_fixture():
    m = C.MIXED
    z = dict(np.load(C.golden_path(m["name"])))
    P = m["prompt_len"]
    special, punct = set(z["special"].tolist()), set(z["punct"].tolist())
    toks = z["tokens"][:P]
    classes = [S if t in special else (TokenClass.PUNCTUATION if t in punct else O) for t in toks]
    head_data = {}
    keys = [(l, h) for l in range(4) for h in range(4)]
    for gi, key in enumerate(keys):
        A, _ = causal_attention(z["q"][gi, :P], z["k"][gi, :P], z["v"][gi, :P], 16)
        ctx = PolicyContext(anns(classes), P, P, A.matrix.sum(axis=0))
        head_data[key] = (A, ctx)
    cfg = ProfilerConfig(recovery_threshold=m["T"])
    prof = profile_model(head_data, cfg, grid=keys)
    golden = HeadProfile.from_csv(str(z["csv"]))
    for key in keys:
        assert prof[key].policy == golden[key].policy, key
        assert prof[key].cost_tokens == golden[key].cost_tokens, key
        assert prof[key].recovery == pytest.approx(golden[key].recovery, abs=1e-12)
