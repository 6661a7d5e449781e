"""Seeded synthetic workloads for the BASELINE.json configurations.

No dataset or checkpoint is available offline, so every configuration is
synthesised from seeded numpy streams with the shapes and value
distributions BASELINE.json names:

* Q/K/V ~ N(0,1) per (batch row, head), rounded to the config dtype
  (fp32 or bf16, round-to-nearest-even); attention logits use the
  standard 1/sqrt(d) scale (``attention.py:125``).
* Token ids uniform over [0, 32000); position 0 is the special id 1;
  every other position independently (p=0.05) takes one of 16 fixed
  punctuation ids.  Classes follow the vocab (special wins, tokens.py:39-44).
* Planted head structure (the only non-random part): a relative-position
  bias ``-slope*|i-j|`` ("local" heads) and/or a sink ``+sink`` on
  special-class keys.  Config 0 plants slope 0.05 on heads 0-1; configs
  1 and 4 plant {local, sink, local+sink} on a seeded 25% of heads with
  slope 0.05 and sink ``SINK_LOGIT``.

Every (b, h) slice comes from its own stream ``default_rng([seed, b, h])``
so any head can be regenerated independently (the CPU oracle samples a
subset of heads at full size).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

VOCAB_SIZE = 32000
SPECIAL_IDS = (1,)
# 16 fixed punctuation ids (arbitrary but fixed; Llama-style byte ids).
PUNCT_IDS = (29871, 29889, 29892, 29901, 29936, 29973, 29991, 29908,
             29915, 29899, 29898, 29897, 29962, 29961, 29930, 29905)
PUNCT_PROB = 0.05
LOCAL_SLOPE = 0.05
SINK_LOGIT = 11.0

CLS_OTHER, CLS_SPECIAL, CLS_PUNCT = 0, 1, 2


def class_lut(vocab_size: int = VOCAB_SIZE, special=SPECIAL_IDS, punct=PUNCT_IDS) -> np.ndarray:
    """uint8 class of every token id; special takes precedence (tokens.py:39-44)."""
    lut = np.zeros(vocab_size, dtype=np.uint8)
    lut[list(punct)] = CLS_PUNCT
    lut[list(special)] = CLS_SPECIAL
    return lut


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (nearest-even); returns float32
    arrays holding exactly representable bf16 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) & np.uint32(0xFFFF0000)).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 storage of already-bf16-rounded float32 values."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


@dataclass
class Workload:
    name: str
    B: int
    H: int
    N: int            # prompt length
    D: int            # decode steps (K/V insertions)
    d: int            # head dim
    dtype: str        # "f32" | "bf16"
    thresholds: tuple
    r_l: float = 0.3
    r_f: float = 0.3
    seed: int = 0
    slopes: np.ndarray = field(default=None)
    sinks: np.ndarray = field(default=None)
    row0: int = 0     # global index of local batch row 0 (a rank's shard)
    head0: int = 0    # global index of local head 0

    def rows(self, b0: int, b1: int) -> "Workload":
        """Batch rows [b0, b1) of this workload as a workload of their own
        (same seeded streams: a shard's inputs equal its slice of the whole)."""
        if not 0 <= b0 < b1 <= self.B:
            raise ValueError(f"rows [{b0}, {b1}) outside B={self.B}")
        return replace(self, B=b1 - b0, row0=self.row0 + b0)

    def heads(self, h0: int, h1: int) -> "Workload":
        """Heads [h0, h1) of every batch row (head sharding)."""
        if not 0 <= h0 < h1 <= self.H:
            raise ValueError(f"heads [{h0}, {h1}) outside H={self.H}")
        return replace(self, H=h1 - h0, head0=self.head0 + h0,
                       slopes=np.asarray(self.slopes)[h0:h1].copy(),
                       sinks=np.asarray(self.sinks)[h0:h1].copy())

    @property
    def total_len(self) -> int:
        return self.N + self.D

    def head_kinds(self) -> list:
        out = []
        for h in range(self.H):
            s, c = self.slopes[h] != 0.0, self.sinks[h] != 0.0
            out.append("local+sink" if s and c else "local" if s else "sink" if c else "plain")
        return out

    def tokens(self, b: int) -> np.ndarray:
        """Token ids [N+D] of batch row b."""
        rng = np.random.default_rng([self.seed, b + self.row0, 1_000_003])
        n = self.total_len
        ids = rng.integers(0, VOCAB_SIZE, size=n)
        punct = rng.random(n) < PUNCT_PROB
        pick = rng.integers(0, len(PUNCT_IDS), size=n)
        ids = np.where(punct, np.asarray(PUNCT_IDS)[pick], ids)
        ids[0] = SPECIAL_IDS[0]
        return ids.astype(np.int64)

    def all_tokens(self) -> np.ndarray:
        return np.stack([self.tokens(b) for b in range(self.B)])

    def head_qkv(self, b: int, h: int) -> tuple:
        """(q, k, v) float32 [N+D, d] of one head, dtype-rounded."""
        rng = np.random.default_rng([self.seed, b + self.row0, h + self.head0])
        x = rng.standard_normal((3, self.total_len, self.d), dtype=np.float32)
        if self.dtype == "bf16":
            x = round_bf16(x)
        return x[0], x[1], x[2]

    def qkv(self) -> tuple:
        """Full float32 tensors q,k,v [B,H,N+D,d] (dtype-rounded values)."""
        shape = (self.B, self.H, self.total_len, self.d)
        q = np.empty(shape, np.float32)
        k = np.empty(shape, np.float32)
        v = np.empty(shape, np.float32)
        for b in range(self.B):
            for h in range(self.H):
                q[b, h], k[b, h], v[b, h] = self.head_qkv(b, h)
        return q, k, v


def _planted(H: int, seed: int, frac: float = 0.25):
    rng = np.random.default_rng([seed, 7777])
    n = max(1, int(round(frac * H)))
    heads = rng.choice(H, size=n, replace=False)
    kinds = rng.integers(0, 3, size=n)       # 0 local, 1 sink, 2 local+sink
    slopes = np.zeros(H)
    sinks = np.zeros(H)
    for h, kd in zip(heads, kinds):
        if kd in (0, 2):
            slopes[h] = LOCAL_SLOPE
        if kd in (1, 2):
            sinks[h] = SINK_LOGIT
    return slopes, sinks


def config0(seed: int = 0) -> Workload:
    """BASELINE config 0: B=1, H=8, d=64, N=256, D=32, fp32, heads 0-1 local."""
    slopes = np.zeros(8)
    slopes[:2] = LOCAL_SLOPE
    return Workload("c0", 1, 8, 256, 32, 64, "f32", (0.95,), seed=seed,
                    slopes=slopes, sinks=np.zeros(8))


def config1(seed: int = 1, B: int = 8, H: int = 32, N: int = 1024, D: int = 512) -> Workload:
    """BASELINE config 1 (Llama-7B-shape layer): B=8, H=32, d=128, N=1024,
    D=512, bf16, planted structure on a seeded 25% of heads, T sweep."""
    slopes, sinks = _planted(H, seed)
    return Workload("c1", B, H, N, D, 128, "bf16", (0.95, 0.98, 0.99), seed=seed,
                    slopes=slopes, sinks=sinks)


def config1_frequent(seed: int = 1, B: int = 8, H: int = 32, N: int = 1024,
                     D: int = 512) -> Workload:
    """Config-1 shapes in the paper's compression regime (PAPER.md:473-475,
    ~40 % pruned): a sink on EVERY head, strengths seeded uniform in
    [9.6, 11.0] logits, no local bias.  At T=0.98 about three quarters of the
    heads profile special+punct+frequent(+local) and evict at every decode
    step (the FREQUENT score update and top-k run on most heads), the rest
    special+punct or full.  Not a BASELINE config: the workload of the K3
    FREQUENT-heavy measurement."""
    rng = np.random.default_rng([seed, 31337])
    sinks = rng.uniform(9.6, 11.0, H)
    w = Workload("c1_frequent", B, H, N, D, 128, "bf16", (0.98,), seed=seed,
                 slopes=np.zeros(H), sinks=sinks)
    return w


def config4(seed: int = 4, B: int = 4, H: int = 32, N: int = 16384, D: int = 256) -> Workload:
    """BASELINE config 4 (long-context stress): B=4, H=32, N=16384, D=256."""
    slopes, sinks = _planted(H, seed)
    return Workload("c4", B, H, N, D, 128, "bf16", (0.95, 0.98, 0.99), seed=seed,
                    slopes=slopes, sinks=sinks)


CONFIGS = {"c0": config0, "c1": config1, "c4": config4, "c1_frequent": config1_frequent}
