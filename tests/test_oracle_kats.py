"""Known-answer tests pinning the CPU oracle: the reference's own unit-test
cases (pkg/tests/test_attention.py, test_policies.py) and the SPEC.md
examples verified against the reference, restated on the
oracle's functions.  CPU only."""

import math

import numpy as np
import pytest

from oracle import akv_oracle as O

S, P, X = O.CLS_SPECIAL, O.CLS_PUNCT, O.CLS_OTHER


def keep(atoms, classes, scores=None, prompt_len=None, r_l=0.3, r_f=0.3, cand=None):
    n = len(classes)
    cls = np.asarray(classes)
    sc = np.zeros(n) if scores is None else np.asarray(scores, float)
    c = np.arange(n) if cand is None else np.asarray(sorted(cand))
    return tuple(O.keep_positions(atoms, c, cls, sc, prompt_len or n, n, r_l, r_f).tolist())


def test_softmax_kats():  # test_attention.py:17-31
    assert np.allclose(O.softmax_vector(np.array([0.0, 0.0])), [0.5, 0.5], atol=1e-12)
    assert np.allclose(O.softmax_vector(np.array([math.log(2.0), 0.0])), [2 / 3, 1 / 3], atol=1e-12)
    out = O.softmax_vector(np.array([1000.0, 0.0]))
    assert np.isfinite(out).all() and abs(out[0] - 1) < 1e-12 and out[1] < 1e-300


def test_causal_mask_exact_zero():  # test_attention.py:41-45
    A = O.causal_softmax(np.ones((3, 3)))
    assert A[0, 1] == 0.0 and A[0, 2] == 0.0 and A[1, 2] == 0.0
    assert np.allclose(A.sum(axis=1), 1.0, atol=1e-12)


def test_two_by_two_hand_evaluated():  # test_attention.py:55-66
    q = np.array([[1.0], [2.0]])
    k = np.array([[1.0], [-1.0]])
    A = O.causal_softmax(O.prompt_logits(q, k, np.zeros(2, int), 0.0, 0.0))
    w0 = math.exp(2.0) / (math.exp(2.0) + math.exp(-2.0))
    assert A[0] == pytest.approx([1.0, 0.0], abs=1e-15)
    assert A[1] == pytest.approx([w0, 1 - w0], abs=1e-15)


def test_atom_kats():  # test_policies.py:45-79, 115-121
    assert keep(O.ATOM_LOCAL, [X] * 10) == (7, 8, 9)
    assert keep(O.ATOM_FREQUENT, [X] * 4, [0.9, 0.05, 0.03, 0.02], r_f=0.5) == (0, 1)
    assert keep(O.ATOM_FREQUENT, [X] * 6, [1, 2, 2, 2, 1, 1], r_f=0.5) == (1, 2, 3)
    assert keep(O.ATOM_SPECIAL | O.ATOM_PUNCT | O.ATOM_LOCAL,
                [S, X, X, X, X, P, X, X, X, X], r_l=0.2) == (0, 5, 8, 9)
    assert keep(O.ATOM_FULL, [X] * 7) == tuple(range(7))
    assert keep(O.ATOM_SPECIAL, [X] * 5) == ()
    sc = [9, 8, 7, 6, 5, 4, 3, 2, 1, 0]
    assert keep(O.ATOM_FREQUENT, [X] * 10, sc) == (0, 1, 2)
    assert keep(O.ATOM_FREQUENT, [X] * 10, sc, cand=[2, 5, 7, 9]) == (2, 5, 7)


def test_exact_budget_counts():  # test_policies.py:181-191
    rng = np.random.default_rng(32)
    for _ in range(200):
        n = int(rng.integers(1, 25))
        p = int(rng.integers(1, n + 1))
        r_l = int(rng.integers(1, 17)) / 16.0
        r_f = int(rng.integers(1, 17)) / 16.0
        cls = rng.integers(0, 3, size=n)
        sc = rng.uniform(0, 5, size=n)
        loc = O.keep_positions(O.ATOM_LOCAL, np.arange(n), cls, sc, p, n, r_l, r_f)
        assert len(loc) == min(math.ceil(r_l * p), n)
        fr = O.keep_positions(O.ATOM_FREQUENT, np.arange(n), cls, sc, p, n, r_l, r_f)
        assert len(fr) == math.ceil(r_f * n)


def test_budget_epsilon_guard():  # policies.py:20-22
    assert O.budget(0.57, 100) == 57
    assert O.budget(0.3, 256) == 77 and O.budget(0.3, 1024) == 308 and O.budget(0.3, 16384) == 4916
    assert O.budget(1e-6, 10) == 1


def _profile(q, k, cls, family, T, sink=0.0, rows=O.ROWS_ALL, crit=O.CRIT_RECOVERY):
    v = np.zeros_like(q)
    return O.profile_head(q, k, v, np.asarray(cls), 0.0, sink, family, [T], rows, crit)


def test_spec_examples():  # SPEC.md:242-268 (verified against the reference)
    fam = O.default_family()
    z4 = np.zeros((4, 1))
    r = _profile(z4, z4, [S, X, X, X], fam, 0.95)
    assert r.recoveries[0] == pytest.approx((1 + 1 / 2 + 1 / 3 + 1 / 4) / 4, abs=1e-12)
    z10 = np.zeros((10, 1))
    assert _profile(z10, z10, [S] + [X] * 9, fam, 0.95).choice == [4]      # diffuse -> full
    assert _profile(z10, z10, [S] + [X] * 9, fam, 0.0).choice == [0]       # T=0 -> special
    mass0 = _profile(z10, z10, [S] + [X] * 9, fam, 0.99, sink=1000.0)
    assert mass0.choice == [0] and mass0.recoveries[0] == pytest.approx(1.0)
    z2 = np.zeros((2, 1))
    cos = _profile(z2, z2, [S, X], fam, 0.95, crit=O.CRIT_COSINE)
    assert cos.cosine[0] == pytest.approx(1.25 / (math.sqrt(1.5) * math.sqrt(1.25)), abs=1e-12)


def test_score_update_semantics():  # test_policies.py:240-275 via one decode step
    fam = [O.Member(O.ATOM_FREQUENT, 0.3, 0.5)]
    n = 4
    q = np.zeros((n + 1, 1))
    k = np.zeros((n + 1, 1))
    v = np.zeros((n + 1, 1))
    cls = np.zeros(n + 1, int)
    prof = O.profile_head(q[:n], k[:n], v[:n], cls, 0.0, 0.0, fam, [-1.0])
    st = O.compact_head(prof, k[:n], v[:n], fam[0], n, 0.0, 0.0)
    before = st.scores.copy()
    O.decode_head(st, q[n], k[n], v[n], n, cls, n)
    assert st.scores.shape == (n + 1,) and st.scores[-1] == 0.0
    kept_before = prof.kept
    # kept rows gained the uniform 1/(kept+1) weight; evicted rows frozen
    gained = st.scores[:n] - before
    assert np.allclose(gained[kept_before], 1.0 / (len(kept_before) + 1))
    mask = np.ones(n, bool)
    mask[kept_before] = False
    assert np.all(gained[mask] == 0.0)
