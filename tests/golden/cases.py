"""Golden-case definitions shared by ``make_golden.py`` (run once, in the
build container, against the unmodified reference) and the parity tests.

Each workload case is fully determined by a seeded ``Workload`` plus the
profiler options below, so the tests regenerate the inputs bit-for-bit
instead of storing them.  The reference's own MIXED_PLAN_4X4 fixture
(``pkg/tests/conftest.py:38-61``) is stored with its rows (it comes from
the reference's SyntheticModel, which is not available on the GPU box).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2310_01801_b200.workloads import (  # noqa: E402
    LOCAL_SLOPE, SINK_LOGIT, Workload, config0, config1, config4,
)

ORDER_DEFAULT = ("special", "punct", "frequent", "local")


def _c0_sink(seed=0) -> Workload:
    w = config0(seed)
    w.name = "c0_sink"
    w.sinks = w.sinks.copy()
    w.slopes = w.slopes.copy()
    # graded sinks so the T sweep walks the whole family at N=256
    w.sinks[[2, 3, 5, 6]] = (8.5, 9.0, 9.5, 10.0)
    w.sinks[4] = SINK_LOGIT
    w.slopes[4] = LOCAL_SLOPE
    w.thresholds = (0.95, 0.98, 0.99)
    return w


def _c1_small(seed=1) -> Workload:
    w = config1(seed, B=2, H=32, N=256, D=48)
    w.name = "c1_small"
    return w


def _c1_heads(seed=1) -> Workload:
    """Config-1 shapes (N=1024, d=128, bf16) on the planted heads plus two
    plain ones, B=1, 96 decode steps."""
    w = config1(seed, B=1, H=32, N=1024, D=96)
    w.name = "c1_heads"
    return w


def _c4_heads(seed=4) -> Workload:
    """Config-4 shapes (N=16384, d=128, bf16, 256 decode steps) on three
    heads of batch row 1: two sink heads that compress (special+punct+
    frequent at T=0.95, evicting at every step) and a local+sink head."""
    w = config4(seed, B=1)
    w.name = "c4_heads"
    return w


def c1_heads_subset(w: Workload) -> list:
    planted = [h for h in range(w.H) if w.slopes[h] != 0 or w.sinks[h] != 0]
    plain = [h for h in range(w.H) if h not in planted][:2]
    return sorted(planted + plain)


# name -> (workload factory, options)
# options: decode_T (threshold used for the decode session), rows, criterion,
# order, drop, fixed (policy string for generate_fixed_baseline-style runs)
CASES = {
    "c0": (config0, dict(decode_T=0.95)),
    "c0_sink": (_c0_sink, dict(decode_T=0.98)),
    "c0_sink_t95": (_c0_sink, dict(decode_T=0.95)),
    "c0_sink_last": (_c0_sink, dict(decode_T=0.95, rows="last")),
    "c0_sink_cosine": (_c0_sink, dict(decode_T=0.95, criterion="cosine")),
    "c0_sink_order": (_c0_sink, dict(decode_T=0.98, order=("special", "frequent", "local", "punct"))),
    "c0_sink_drop": (_c0_sink, dict(decode_T=0.98, drop=("punct",))),
    "c0_fixed_spfl": (_c0_sink, dict(fixed="special+punct+frequent(r_f=0.3)+local(r_l=0.3)")),
    "c0_fixed_freq": (_c0_sink, dict(fixed="frequent(r_f=0.25)")),
    "c1_small": (_c1_small, dict(decode_T=0.98)),
    # the tcgen05 profiling path's secondary outputs (bf16, d=128): the
    # cosine criterion (colsq, profiler.py:148-178) and last-row recovery
    # (profiler.py:84-85)
    "c1_small_cosine": (_c1_small, dict(decode_T=0.98, criterion="cosine")),
    "c1_small_last": (_c1_small, dict(decode_T=0.98, rows="last")),
    "c1_heads": (_c1_heads, dict(decode_T=0.98, heads="planted+2")),
    "c4_heads": (_c4_heads, dict(decode_T=0.95, heads=[(1, 0), (1, 3), (1, 18)])),
}

# cases whose oracle run is too slow for the CPU suite (checked on the GPU
# against the reference's goldens directly)
LONG_CASES = ("c4_heads",)

MIXED = dict(name="mixed4x4", prompt_len=64, steps=24, T=0.95, seed=101, dominance=0.97)


def golden_path(name: str) -> str:
    return os.path.join(HERE, f"{name}.npz")


def case_workload(name: str) -> tuple:
    factory, opts = CASES[name]
    return factory(), dict(opts)


def case_heads(w: Workload, opts: dict) -> list:
    """(b, h) pairs of the case, in the reference's sorted grid order."""
    if opts.get("heads") == "planted+2":
        return [(0, h) for h in c1_heads_subset(w)]
    if isinstance(opts.get("heads"), list):
        return [tuple(x) for x in opts["heads"]]
    return [(b, h) for b in range(w.B) for h in range(w.H)]


def unpack_kept(bits: np.ndarray, length: int) -> np.ndarray:
    return np.unpackbits(bits, axis=-1, count=length).astype(bool)
