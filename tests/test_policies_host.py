"""Host-side policy algebra, grammar, family and profile CSV — mirrors the
reference's pkg/tests/test_policies.py:159-336 cases for the API objects
the drop-in keeps (CPU only)."""

import numpy as np
import pytest

from paper_2310_01801_b200 import (CompressionPolicy, HeadDecision, HeadProfile, PolicyAtom,
                                   PolicyError, ProfilerConfig, ProfilerError, RetainedSet,
                                   feasible_set, format_policy, full_policy, parse_policy)
from paper_2310_01801_b200.tokens import TokenClass, VocabMetadata, classify_tokens


def test_feasible_set_default_is_nested_five_policy_family():
    fam = feasible_set()
    assert [p.atoms for p in fam[:-1]] == [
        {PolicyAtom.SPECIAL},
        {PolicyAtom.SPECIAL, PolicyAtom.PUNCTUATION},
        {PolicyAtom.SPECIAL, PolicyAtom.PUNCTUATION, PolicyAtom.FREQUENT},
        {PolicyAtom.SPECIAL, PolicyAtom.PUNCTUATION, PolicyAtom.FREQUENT, PolicyAtom.LOCAL},
    ]
    assert fam[-1].is_full
    assert [p.bits for p in fam] == [1, 3, 7, 15, 16]


def test_feasible_set_order_and_drop_ablations():
    fam = feasible_set(atom_order=(PolicyAtom.SPECIAL, PolicyAtom.FREQUENT, PolicyAtom.LOCAL,
                                   PolicyAtom.PUNCTUATION))
    assert [p.bits for p in fam] == [1, 5, 13, 15, 16]
    fam = feasible_set(drop={PolicyAtom.FREQUENT})
    assert len(fam) == 4 and all(PolicyAtom.FREQUENT not in p.atoms for p in fam)
    assert feasible_set(drop={PolicyAtom.SPECIAL})[0].atoms == {PolicyAtom.PUNCTUATION}
    with pytest.raises(PolicyError, match="backstop"):
        feasible_set(atom_order=(PolicyAtom.FULL,))
    with pytest.raises(PolicyError, match="duplicates"):
        feasible_set(atom_order=(PolicyAtom.SPECIAL, PolicyAtom.SPECIAL))
    with pytest.raises(PolicyError, match="at least one atom"):
        feasible_set(drop=set(PolicyAtom) - {PolicyAtom.FULL})


def test_policy_invariants():
    with pytest.raises(PolicyError, match="at least one atom"):
        CompressionPolicy(frozenset())
    with pytest.raises(PolicyError, match="full cannot be combined"):
        CompressionPolicy(frozenset({PolicyAtom.FULL, PolicyAtom.LOCAL}))
    with pytest.raises(PolicyError, match="r_l"):
        CompressionPolicy(frozenset({PolicyAtom.LOCAL}), r_l=0.0)
    with pytest.raises(PolicyError, match="r_f"):
        CompressionPolicy(frozenset({PolicyAtom.FREQUENT}), r_f=1.5)


def test_policy_string_round_trips():
    for text in ["full", "special", "special+punct",
                 "special+punct+frequent(r_f=0.3)+local(r_l=0.3)", "frequent(r_f=0.15)",
                 "local(r_l=0.5)"]:
        assert format_policy(parse_policy(text)) == text
    assert format_policy(parse_policy("local(r_l=0.3)+special")) == "special+local(r_l=0.3)"
    rng = np.random.default_rng(44)
    atoms = [PolicyAtom.SPECIAL, PolicyAtom.PUNCTUATION, PolicyAtom.FREQUENT, PolicyAtom.LOCAL]
    for _ in range(100):
        chosen = [a for a in atoms if rng.random() < 0.5] or [PolicyAtom.SPECIAL]
        pol = CompressionPolicy(frozenset(chosen), r_l=round(float(rng.uniform(0.05, 1)), 3),
                                r_f=round(float(rng.uniform(0.05, 1)), 3))
        back = parse_policy(format_policy(pol))
        assert back.atoms == pol.atoms
        if PolicyAtom.LOCAL in pol.atoms:
            assert back.r_l == pol.r_l
        if PolicyAtom.FREQUENT in pol.atoms:
            assert back.r_f == pol.r_f


def test_parse_policy_errors():
    with pytest.raises(PolicyError, match="unknown policy atom"):
        parse_policy("special+average")
    with pytest.raises(PolicyError, match="bad ratio"):
        parse_policy("local(r_l=abc)")
    with pytest.raises(PolicyError, match="not valid"):
        parse_policy("special(r_f=0.3)")


def test_union_and_full():
    a = CompressionPolicy(frozenset({PolicyAtom.SPECIAL, PolicyAtom.LOCAL}))
    b = CompressionPolicy(frozenset({PolicyAtom.FREQUENT}))
    assert a.union(b).atoms == a.atoms | b.atoms
    assert a.union(full_policy()).is_full


def test_retained_set_sorted_dedup():
    r = RetainedSet.of([5, 1, 5, 3])
    assert r.indices == (1, 3, 5) and len(r) == 3 and 3 in r
    with pytest.raises(PolicyError, match="negative"):
        RetainedSet.of([-1])


def test_profiler_config_validation():
    with pytest.raises(ProfilerError, match="recovery_threshold"):
        ProfilerConfig(recovery_threshold=1.5)
    with pytest.raises(ProfilerError, match="empty"):
        ProfilerConfig(feasible=())
    with pytest.raises(ProfilerError, match="full cache"):
        ProfilerConfig(feasible=tuple(feasible_set()[:-1]))


def test_head_profile_csv_round_trip():
    prof = HeadProfile({(1, 0): HeadDecision(parse_policy("special"), 0.96, 3),
                        (0, 1): HeadDecision(full_policy(), 1.0, 256)})
    text = prof.to_csv()
    assert text.splitlines()[0] == "layer,head,policy,recovery,cost_tokens"
    assert text.splitlines()[1] == "0,1,full,1.0,256"
    back = HeadProfile.from_csv(text)
    assert back.to_csv() == text
    with pytest.raises(ProfilerError, match="header"):
        HeadProfile.from_csv("a,b\n")


def test_classification_special_wins_and_warns():
    vocab = VocabMetadata(special_ids={1, 2}, punctuation_ids={2, 3})
    with pytest.warns(UserWarning, match="overlap"):
        anns = classify_tokens([1, 2, 3, 4], vocab)
    assert [a.klass for a in anns] == [TokenClass.SPECIAL, TokenClass.SPECIAL,
                                       TokenClass.PUNCTUATION, TokenClass.OTHER]
    assert vocab.class_codes([1, 2, 3, 4]).tolist() == [1, 1, 2, 0]


def test_nucleus_sampler_matches_reference_draws():
    """engine.py:71-90: the restated nucleus sampler draws the same tokens
    as the reference's _Sampler on seeded logits (golden from the reference,
    tests/golden/make_golden.py nucleus)."""
    import numpy as np

    import cases as C
    from paper_2310_01801_b200.engine import EngineError, Nucleus, _Sampler

    z = dict(np.load(C.golden_path("nucleus")))
    for (temp, top_p, seed), want in zip(z["params"], z["draws"]):
        smp = _Sampler(Nucleus(temperature=float(temp), top_p=float(top_p), seed=int(seed)))
        assert [smp(row) for row in z["logits"]] == want.tolist()
    import pytest

    with pytest.raises(EngineError, match="temperature"):
        Nucleus(temperature=0.0)
    with pytest.raises(EngineError, match="top_p"):
        Nucleus(top_p=1.5)
