"""The exact block-wide top-k (csrc/akv_common.cuh block_topk_threshold: radix
passes, then - once the bucket holding the k-th key has at most 64 members -
an exact in-warp rank) against the reference's order: larger score first,
ties by lower position (policies.py:232-240, a stable argsort of -scores),
with -0.0 tied to +0.0.  Driven through akv_keep_mask (FREQUENT only), the
same device routine the profiling policy epilogue and K3's radix fallback
use; sizes and tie patterns put the boundary in large and small buckets."""

import math

import numpy as np
import pytest

from paper_2310_01801_b200 import _ops

pytestmark = pytest.mark.gpu

ATOM_FREQUENT = 4


def _budget(r, n):
    return max(1, math.ceil(r * n - 1e-9))  # policies.py:205-206


def _expected(scores, cand, r_f):
    L = len(scores)
    idx = np.arange(L) if cand is None else np.flatnonzero(cand)
    kb = _budget(r_f, L)
    s = scores[idx] + 0.0  # -0.0 ties +0.0
    order = np.lexsort((idx, -s))
    keep = np.zeros(L, bool)
    keep[idx[order[:kb]]] = True
    return keep


def _patterns(rng, L):
    yield "continuous", rng.random(L)
    yield "four values", rng.integers(0, 4, L) / 8.0
    yield "all equal", np.full(L, 0.25)
    z = np.where(rng.random(L) < 0.5, 0.0, -0.0)
    z[rng.random(L) < 0.3] = 1e-3
    yield "signed zeros", z
    base = rng.random(L)
    k = _budget(0.3, L)
    if L > 4:
        # a run of equal keys straddling the 30 % boundary, wider than 64
        # when L is large enough (the radix tie path) and narrower otherwise
        srt = np.sort(base)[::-1]
        v = srt[min(k - 1, L - 1)]
        near = np.argsort(np.abs(base - v))[:min(L, 200)]
        base = base.copy()
        base[near] = v
    yield "boundary run", base
    yield "close doubles", 1.0 + rng.integers(0, 50, L) * np.finfo(np.float64).eps


@pytest.mark.parametrize("L", [1, 2, 37, 64, 65, 130, 1000, 3000])
def test_topk_matches_stable_argsort(L):
    rng = np.random.default_rng(L)
    items, want = [], []
    for name, scores in _patterns(rng, L):
        for r_f in (0.05, 0.3, 0.77, 1.0):
            for use_cand in (False, True):
                cand = (rng.random(L) < 0.7) if use_cand else None
                if cand is not None and not cand.any():
                    cand[0] = True
                items.append(dict(cls=np.zeros(L, np.uint8), scores=scores.astype(np.float64),
                                  cand=cand, prompt_len=L, current_len=L, atoms=ATOM_FREQUENT,
                                  r_l=0.0, r_f=r_f))
                want.append((name, r_f, use_cand, _expected(scores, cand, r_f)))
    keep, cnt = _ops.keep_masks(items)
    for g, (name, r_f, use_cand, exp) in enumerate(want):
        got = keep[g, :L]
        assert np.array_equal(got, exp), (L, name, r_f, use_cand, np.flatnonzero(got ^ exp)[:10])
        assert cnt[g] == exp.sum()
