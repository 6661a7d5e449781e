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
