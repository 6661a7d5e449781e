"""Profiler configuration and per-head profile records (reference:
profiler.py:37-48, 90-132, 181-228).  The selection itself — recovery of
every family member, first member with recovery >= T, cosine argmax — runs
in the K1 policy epilogue on the GPU (akv_profile)."""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field
from enum import Enum
from typing import Mapping

import numpy as np

from .policies import CompressionPolicy, feasible_set, format_policy, parse_policy


class ProfilerError(ValueError):
    """Invalid profiler configuration or inputs (profiler.py:37-38)."""


class SelectionCriterion(Enum):
    RECOVERY_MASS = "recovery"
    COSINE_SIMILARITY = "cosine"


class RowAveraging(Enum):
    ALL_ROWS = "all"
    LAST_ROW = "last"


@dataclass(frozen=True)
class RecoveryReport:
    policy: CompressionPolicy
    recovery: float
    cost_tokens: int
    pruned_ratio: float


@dataclass(frozen=True)
class ProfilerConfig:
    recovery_threshold: float = 0.95
    feasible: tuple = field(default_factory=lambda: tuple(feasible_set()))
    criterion: SelectionCriterion = SelectionCriterion.RECOVERY_MASS
    rows: RowAveraging = RowAveraging.ALL_ROWS

    def __post_init__(self):
        object.__setattr__(self, "feasible", tuple(self.feasible))
        if not 0.0 <= self.recovery_threshold <= 1.0:
            raise ProfilerError(
                f"recovery_threshold must be in [0, 1], got {self.recovery_threshold}")
        if not self.feasible:
            raise ProfilerError("feasible set is empty")
        if not self.feasible[-1].is_full:
            raise ProfilerError(
                "last feasible policy must be the full cache (feasibility backstop)")
        if len(self.feasible) > 8:
            raise ProfilerError("feasible family longer than 8 policies is not supported")


@dataclass(frozen=True)
class HeadDecision:
    policy: CompressionPolicy
    recovery: float
    cost_tokens: int


@dataclass(frozen=True)
class HeadProfile:
    """Per-head policy choices, fixed once at prompt encoding."""

    decisions: Mapping

    def __post_init__(self):
        object.__setattr__(self, "decisions", dict(self.decisions))

    def __getitem__(self, key) -> HeadDecision:
        return self.decisions[key]

    def __len__(self) -> int:
        return len(self.decisions)

    def items(self):
        return sorted(self.decisions.items())

    def to_csv(self) -> str:
        """``layer,head,policy,recovery,cost_tokens`` (profiler.py:206-214)."""
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["layer", "head", "policy", "recovery", "cost_tokens"])
        for (layer, head), d in self.items():
            w.writerow([layer, head, format_policy(d.policy), repr(d.recovery), d.cost_tokens])
        return buf.getvalue()

    @classmethod
    def from_csv(cls, text: str) -> "HeadProfile":
        rows = csv.reader(io.StringIO(text))
        header = next(rows, None)
        if header != ["layer", "head", "policy", "recovery", "cost_tokens"]:
            raise ProfilerError(f"bad profile CSV header: {header}")
        out = {}
        for r in rows:
            out[(int(r[0]), int(r[1]))] = HeadDecision(parse_policy(r[2]), float(r[3]), int(r[4]))
        return cls(out)


# ---------------------------------------------------------------------------
# Map-level profiling functions (profiler.py:51-178, 231-269) on the GPU:
# retained sets from akv_keep_mask, recoveries / cosines from
# akv_map_recovery_f64 — batched over heads and family members.

def _rows_code(rows: RowAveraging) -> int:
    return 1 if rows is RowAveraging.LAST_ROW else 0


def _mask(retained, n: int) -> np.ndarray:
    m = np.zeros(n, bool)
    idx = [i for i in retained.indices if i < n]
    m[idx] = True
    return m


def tv_distance_row(p, retained) -> float:
    """Total variation between a row and its renormalised compressed form."""
    from . import _ops

    row = np.asarray(p, dtype=np.float64)
    if row.ndim != 1:
        raise ProfilerError("probability row must be 1-D")
    return _ops.tv_distance(row, _mask(retained, row.size), ProfilerError)


def recovery_ratio(A, retained, rows: RowAveraging = RowAveraging.ALL_ROWS) -> float:
    """Mean (or last-row) retained attention mass (profiler.py:70-87)."""
    from . import _ops

    m = A.matrix
    rec, _ = _ops.map_recovery(m[None], _mask(retained, A.size)[None, None], _rows_code(rows),
                               ProfilerError)
    return float(rec[0, 0])


def masked_cosine_similarity(A, retained) -> float:
    from . import _ops

    _, cos = _ops.map_recovery(A.matrix[None], _mask(retained, A.size)[None, None], 0,
                               ProfilerError)
    return float(cos[0, 0])


def _family_tables(head_data, family, rows):
    """One keep-mask launch for every (head, member) and one map-recovery
    launch per map size: (masks [H,F,n], costs [H,F], recoveries, cosines)."""
    from . import _ops
    from .policies import _keep_item

    keys = list(head_data)
    items = []
    for key in keys:
        _, ctx = head_data[key]
        items += [_keep_item(pol, ctx) for pol in family]
    keep, cnt = _ops.keep_masks(items, ProfilerError)
    F = len(family)
    out = {}
    by_n = {}
    for hi, key in enumerate(keys):
        by_n.setdefault(head_data[key][0].size, []).append(hi)
    for n, his in by_n.items():
        maps = np.stack([head_data[keys[hi]][0].matrix for hi in his])
        masks = np.stack([keep[hi * F:(hi + 1) * F, :n] for hi in his])
        rec, cos = _ops.map_recovery(maps, masks, _rows_code(rows), ProfilerError)
        for r, hi in enumerate(his):
            out[keys[hi]] = (rec[r], cos[r], cnt[hi * F:(hi + 1) * F])
    return out


def evaluate_policy(A, ctx, policy, rows: RowAveraging = RowAveraging.ALL_ROWS) -> RecoveryReport:
    """Fixed-policy recovery, cost and pruned ratio (profiler.py:100-109)."""
    rec, _, cost = _family_tables({0: (A, ctx)}, [policy], rows)[0]
    return RecoveryReport(policy, float(rec[0]), int(cost[0]), 1.0 - cost[0] / ctx.current_len)


def select_policy(A, ctx, cfg: ProfilerConfig):
    """First family member with recovery >= T (profiler.py:135-145)."""
    rec, _, _ = _family_tables({0: (A, ctx)}, list(cfg.feasible), cfg.rows)[0]
    for pol, r in zip(cfg.feasible, rec):
        if r >= cfg.recovery_threshold:
            return pol, float(r)
    raise ProfilerError("no feasible policy met the threshold")


def select_policy_by_similarity(A, schemes, ctx):
    """Argmax masked cosine similarity, ties to the earlier scheme (profiler.py:164-178)."""
    if not schemes:
        raise ProfilerError("schemes list is empty")
    _, cos, _ = _family_tables({0: (A, ctx)}, list(schemes), RowAveraging.ALL_ROWS)[0]
    best, best_sim = schemes[0], -1.0
    for pol, s in zip(schemes, cos):
        if s > best_sim:
            best, best_sim = pol, s
    return best


def profile_model(head_data, cfg: ProfilerConfig, grid=None, threads=None) -> HeadProfile:
    """Select a policy for every head (profiler.py:243-269): one batched
    keep-mask launch and one recovery launch per map size for all heads;
    ``threads`` is accepted for API compatibility."""
    keys = sorted(head_data)
    if grid is not None:
        for key in grid:
            if key not in head_data:
                raise ProfilerError(
                    f"missing profiling data for head (layer={key[0]}, head={key[1]})")
    fam = list(cfg.feasible)
    tables = _family_tables({k: head_data[k] for k in keys}, fam, cfg.rows)
    decisions = {}
    for key in keys:
        rec, cos, cost = tables[key]
        if cfg.criterion is SelectionCriterion.COSINE_SIMILARITY:
            c, best = 0, -1.0
            for i, s in enumerate(cos):
                if s > best:
                    c, best = i, s
        else:
            c = next((i for i, r in enumerate(rec) if r >= cfg.recovery_threshold), None)
            if c is None:
                raise ProfilerError("no feasible policy met the threshold")
        decisions[key] = HeadDecision(fam[c], float(rec[c]), int(cost[c]))
    return HeadProfile(decisions)
