"""CPU oracle for the FastGen adaptive-KV hot path — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
``adaptive_kv`` (``/root/reference/pkg/src/adaptive_kv``) for the three
hot-path stages: prompt profiling, per-head compaction and compressed
decode with insert/evict.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The product package ``paper_2310_01801_b200`` never imports
it and has no CPU fallback.

Pinning: the oracle is checked against golden vectors produced by running
the unmodified reference in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``; test
``tests/test_oracle_golden.py``) and against the reference's own unit-test
KATs restated in ``tests/test_oracle_kats.py``.

Conventions shared with the CUDA path:

* atoms are bit flags (ATOM_*), classes are small ints (CLS_*);
* a head's logit for query position i and key position j is
  ``q_i·k_j/sqrt(d) - slope*(i-j) + sink*[class_j == special]``; the two
  planted terms are the synthetic workloads' head structure (BASELINE.json
  configs) and are folded exactly into extra Q/K dimensions when the
  reference itself is run;
* scores / colsums are float64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ATOM_SPECIAL = 1
ATOM_PUNCT = 2
ATOM_FREQUENT = 4
ATOM_LOCAL = 8
ATOM_FULL = 16

CLS_OTHER = 0
CLS_SPECIAL = 1
CLS_PUNCT = 2

ROWS_ALL = 0
ROWS_LAST = 1
CRIT_RECOVERY = 0
CRIT_COSINE = 1

_BUDGET_EPS = 1e-9  # policies.py:22


def budget(ratio: float, length: int) -> int:
    """policies.py:205-206 — ``max(1, ceil(r*L - 1e-9))`` in float64."""
    return max(1, math.ceil(ratio * length - _BUDGET_EPS))


def keep_positions(atoms, cand, cls_of_pos, scores, prompt_len, current_len, r_l, r_f):
    """Union of the policy's atom position sets over ``cand``.

    policies.py:214-241 (``_atom_indices``) and :244-267
    (``retained_indices``).  ``cand`` is a sorted int array of candidate
    positions (all of ``range(current_len)`` at profiling time, the live
    positions plus the new one during decode, engine.py:317/333);
    ``cls_of_pos[p]`` the class of position p; ``scores[p]`` the cumulative
    score of position p (only read for FREQUENT).
    Returns the sorted kept positions.
    """
    cand = np.asarray(cand, dtype=np.int64)
    if atoms & ATOM_FULL:
        return cand.copy()
    keep = np.zeros(cand.shape[0], dtype=bool)
    if atoms & ATOM_SPECIAL:
        keep |= cls_of_pos[cand] == CLS_SPECIAL
    if atoms & ATOM_PUNCT:
        keep |= cls_of_pos[cand] == CLS_PUNCT
    if atoms & ATOM_LOCAL:
        window_start = current_len - budget(r_l, prompt_len)  # policies.py:209-211,230
        keep |= cand >= window_start
    if atoms & ATOM_FREQUENT and cand.size:
        b = budget(r_f, current_len)  # policies.py:233
        s = np.asarray(scores, dtype=np.float64)[cand]
        order = np.argsort(-s, kind="stable")  # ties -> lower position, :238-240
        keep[order[:b]] = True
    return cand[keep]


def causal_softmax(logits: np.ndarray) -> np.ndarray:
    """attention.py:64-89 with causal_lengths = 1..n: row i normalised over
    columns <= i, the rest exactly zero."""
    n = logits.shape[0]
    masked = np.where(np.tri(n, dtype=bool), logits, -np.inf)
    m = masked.max(axis=1, keepdims=True)
    e = np.exp(masked - m)
    return e / e.sum(axis=1, keepdims=True)


def softmax_vector(v: np.ndarray) -> np.ndarray:
    """attention.py:92-99."""
    shifted = v - v.max()
    e = np.exp(shifted)
    return e / e.sum()


def prompt_logits(q, k, cls_pos, slope, sink):
    """attention.py:125 plus the planted head bias."""
    n, d = q.shape
    logits = (q @ k.T) / np.sqrt(float(d))
    if slope != 0.0:
        idx = np.arange(n, dtype=np.float64)
        logits = logits - slope * (idx[:, None] - idx[None, :])
    if sink != 0.0:
        logits = logits + sink * (cls_pos[:n] == CLS_SPECIAL)[None, :]
    return logits


@dataclass
class Member:
    """One policy of the feasible family (policies.py:48-74)."""

    atoms: int
    r_l: float = 0.3
    r_f: float = 0.3


def default_family(r_l=0.3, r_f=0.3, order=(ATOM_SPECIAL, ATOM_PUNCT, ATOM_FREQUENT, ATOM_LOCAL)):
    """policies.py:296-329 (``feasible_set``): nested unions then FULL."""
    fam, acc = [], 0
    for a in order:
        acc |= a
        fam.append(Member(acc, r_l, r_f))
    fam.append(Member(ATOM_FULL, r_l, r_f))
    return fam


@dataclass
class HeadProfileResult:
    choice: list          # chosen family index per threshold
    recoveries: np.ndarray  # R_k per family member
    costs: np.ndarray       # |S_k| per member
    cosine: np.ndarray      # cosine similarity per member
    colsum: np.ndarray
    lastp: np.ndarray
    out_last: np.ndarray
    kept: np.ndarray        # kept positions of the chosen policy (primary T)
    last_row_recovery: float


def profile_head(q, k, v, cls_pos, slope, sink, family, thresholds,
                 rows=ROWS_ALL, criterion=CRIT_RECOVERY):
    """engine.py:161-200 (prompt_head_data) + profiler.py:70-87
    (recovery_ratio), :135-145 (select_policy), :148-178 (cosine) and
    engine.py:236-259 (compaction bookkeeping) for one head."""
    n = q.shape[0]
    A = causal_softmax(prompt_logits(q, k, cls_pos, slope, sink))
    colsum = A.sum(axis=0)                     # engine.py:196
    all_pos = np.arange(n)
    sets, rec, cost, cos = [], [], [], []
    total_norm = float(np.linalg.norm(A))      # profiler.py:157
    for mem in family:
        idx = keep_positions(mem.atoms, all_pos, cls_pos, colsum, n, n, mem.r_l, mem.r_f)
        sets.append(idx)
        cost.append(idx.size)
        if idx.size == 0:
            rec.append(0.0)
            cos.append(0.0)
            continue
        per_row = A[:, idx].sum(axis=1)        # profiler.py:84
        rec.append(float(per_row[-1]) if rows == ROWS_LAST else float(per_row.mean()))
        masked = float(np.linalg.norm(A[:, idx]))
        cos.append(0.0 if masked == 0.0 else masked / total_norm)
    choice = []
    if criterion == CRIT_COSINE:
        best, best_sim = 0, -1.0
        for i, s in enumerate(cos):            # strict > : ties to earlier, :174-177
            if s > best_sim:
                best, best_sim = i, s
        choice = [best for _ in thresholds]
    else:
        for t in thresholds:
            c = next((i for i, r in enumerate(rec) if r >= t), None)
            if c is None:
                raise ValueError("no feasible policy met the threshold")  # :144-145
            choice.append(c)
    kept = sets[choice[0]]
    lastp = A[n - 1].copy()
    return HeadProfileResult(
        choice=choice, recoveries=np.asarray(rec), costs=np.asarray(cost),
        cosine=np.asarray(cos), colsum=colsum, lastp=lastp,
        out_last=lastp @ v,                    # engine.py:248,255
        kept=kept,
        last_row_recovery=float(lastp[kept].sum()) if kept.size else 0.0,
    )


@dataclass
class HeadState:
    """engine.py:100-117 (HeadCacheState) restated with position arrays."""

    member: Member
    positions: np.ndarray   # ascending live positions
    K: np.ndarray
    V: np.ndarray
    scores: np.ndarray | None  # full-length (current_len) scores, FREQUENT heads only
    out: np.ndarray
    slope: float = 0.0
    sink: float = 0.0
    evictions: int = 0
    shadow: np.ndarray | None = None  # every key by position (diagnostics, engine.py:260-261)
    recovery: float = 0.0             # last_row_recovery (engine.py:256-258, 348)


def compact_head(res: HeadProfileResult, k, v, member: Member, n, slope, sink):
    """engine.py:236-259: keep rows in ascending position order; scores
    copied only for FREQUENT policies."""
    kept = res.kept
    scores = res.colsum.copy() if member.atoms & ATOM_FREQUENT else None
    return HeadState(member, kept.copy(), k[kept].copy(), v[kept].copy(), scores,
                     res.out_last.copy(), slope, sink, shadow=k[:n].copy(),
                     recovery=float(res.lastp[kept].sum()) if kept.size else 0.0)


def decode_head(st: HeadState, q, k_new, v_new, pos, cls_pos, prompt_len):
    """engine.py:303-339 + policies.py:332-360 for one head and one step.

    ``cls_pos`` must already hold the class of ``pos``.  Returns the
    attention output; mutates ``st``.
    """
    d = q.shape[0]
    attended = np.append(st.positions, pos)
    K_att = np.vstack([st.K, k_new[None, :]])
    V_att = np.vstack([st.V, v_new[None, :]])
    logits = (K_att @ q) / np.sqrt(float(d))   # engine.py:95
    if st.slope != 0.0:
        logits = logits - st.slope * (pos - attended)
    if st.sink != 0.0:
        logits = logits + st.sink * (cls_pos[attended] == CLS_SPECIAL)
    w = softmax_vector(logits)
    out = w @ V_att
    cur = pos + 1
    if st.scores is not None:                  # engine.py:320-330
        sc = st.scores.copy()
        sc[st.positions] += w[:-1]             # policies.py:356
        st.scores = np.append(sc, 0.0)         # :357
        scores = st.scores
    else:
        scores = None
    m = st.member
    kept = keep_positions(m.atoms, attended, cls_pos, scores, prompt_len, cur, m.r_l, m.r_f)
    sel = np.isin(attended, kept)
    st.evictions += int((~sel).sum())
    st.positions = attended[sel]
    st.K = K_att[sel]
    st.V = V_att[sel]
    st.out = out
    if st.shadow is not None:              # engine.py:341-349
        st.shadow = np.vstack([st.shadow, k_new[None, :]])
        full = (st.shadow @ q) / np.sqrt(float(d))
        allpos = np.arange(pos + 1)
        if st.slope != 0.0:
            full = full - st.slope * (pos - allpos)
        if st.sink != 0.0:
            full = full + st.sink * (cls_pos[allpos] == CLS_SPECIAL)
        st.recovery = float(softmax_vector(full)[attended].sum())
    return out


@dataclass
class Session:
    """A batch of independent sequences x heads (the reference's
    (layer, head) grid, engine.py:130-141)."""

    heads: list            # [B*H] HeadState
    profiles: list         # [B*H] HeadProfileResult
    cls: np.ndarray        # [B, N+D] classes (grown as decode proceeds)
    prompt_len: int
    seq_len: int
    H: int
    history: list = field(default_factory=list)


def encode_session(q, k, v, cls, slopes, sinks, family, thresholds,
                   rows=ROWS_ALL, criterion=CRIT_RECOVERY, fixed: Member | None = None,
                   cls_capacity=None):
    """engine.py:203-272 over tensors q,k,v [B,H,N,d] (float64 views of
    the device inputs), cls [B,>=N] int classes, per-head slopes/sinks [H]."""
    B, H, N, _ = q.shape
    fam = [fixed] if fixed is not None else family
    thr = [-1.0] if fixed is not None else list(thresholds)
    cap = cls.shape[1] if cls_capacity is None else cls_capacity
    cls_full = np.zeros((B, cap), dtype=np.int64)
    cls_full[:, :cls.shape[1]] = cls
    heads, profiles = [], []
    for b in range(B):
        for h in range(H):
            res = profile_head(q[b, h], k[b, h], v[b, h], cls_full[b], slopes[h], sinks[h],
                               fam, thr, rows, criterion)
            profiles.append(res)
            heads.append(compact_head(res, k[b, h], v[b, h], fam[res.choice[0]], N,
                                      slopes[h], sinks[h]))
    return Session(heads, profiles, cls_full, N, N, H)


def decode_session_step(sess: Session, q, k, v, cls_new):
    """engine.py:283-350 for one inserted token per sequence.
    q,k,v [B,H,d]; cls_new [B].  Returns outputs [B,H,d]."""
    B = q.shape[0]
    H = sess.H
    pos = sess.seq_len
    if sess.cls.shape[1] <= pos:
        grow = np.zeros((B, pos + 1), dtype=np.int64)
        grow[:, :sess.cls.shape[1]] = sess.cls
        sess.cls = grow
    sess.cls[:, pos] = cls_new
    out = np.zeros(q.shape, dtype=np.float64)
    for b in range(B):
        for h in range(H):
            out[b, h] = decode_head(sess.heads[b * H + h], q[b, h], k[b, h], v[b, h],
                                    pos, sess.cls[b], sess.prompt_len)
    sess.seq_len = pos + 1
    return out


def format_member(m: Member) -> str:
    """policies.py:84-98 (``format_policy``)."""
    if m.atoms & ATOM_FULL:
        return "full"
    parts = []
    if m.atoms & ATOM_SPECIAL:
        parts.append("special")
    if m.atoms & ATOM_PUNCT:
        parts.append("punct")
    if m.atoms & ATOM_FREQUENT:
        parts.append(f"frequent(r_f={m.r_f:g})")
    if m.atoms & ATOM_LOCAL:
        parts.append(f"local(r_l={m.r_l:g})")
    return "+".join(parts)
