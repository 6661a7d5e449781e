"""Pin the CPU oracle against golden vectors produced by running the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import cases as C
from helpers import load_golden, oracle_case

CPU_CASES = [n for n in C.CASES if n not in C.LONG_CASES]


@pytest.mark.parametrize("name", CPU_CASES)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    o = oracle_case(name)
    # profiling: every family member's recovery and cost, the choice per T
    np.testing.assert_allclose(o["R"], g["R"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(o["cost"], g["cost"])
    # masked cosine similarity of every member (profiler.py:148-161)
    np.testing.assert_allclose(o["cos"], g["cos"], rtol=0, atol=1e-12)
    if g["choice"].size and "fixed" not in C.CASES[name][1]:
        np.testing.assert_array_equal(o["choice"], g["choice"])
    np.testing.assert_array_equal(o["dec_choice"], g["dec_choice"])
    np.testing.assert_allclose(o["colsum"], g["colsum"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(o["lastrow"], g["lastrow"], rtol=1e-12, atol=1e-15)
    # compaction: kept sets bit-exact, pending output of the prompt's last row
    np.testing.assert_array_equal(o["enc_kept"], g["enc_kept"])
    np.testing.assert_allclose(o["enc_out"], g["enc_out"], rtol=1e-10, atol=1e-12)
    # decode: per-step kept sets bit-exact and outputs
    np.testing.assert_array_equal(o["dec_kept"], g["dec_kept"])
    np.testing.assert_allclose(o["dec_out"], g["dec_out"], rtol=1e-9, atol=1e-11)
    # diagnostics: recovery of the attended set vs the uncompressed shadow
    # softmax at every step, and the per-step mean over heads (StepRecord)
    np.testing.assert_allclose(o["dec_rec"], g["dec_rec"], rtol=0, atol=1e-12)
    rows = g["dec_mean"].shape[0]
    np.testing.assert_allclose(o["dec_rec"].reshape(o["dec_rec"].shape[0], rows, -1).mean(-1).T,
                               g["dec_mean"], rtol=0, atol=1e-12)


def test_golden_cases_exercise_every_policy_kind():
    """The golden set must exercise compaction and eviction, not only full
    heads (SURVEY §7 'Degenerate configs')."""
    seen = set()
    for name in C.CASES:
        g = load_golden(name)
        fam = g["family"]
        for c in g["dec_choice"]:
            seen.add(int(fam[c]))
    assert {1, 7, 15, 16} <= seen
