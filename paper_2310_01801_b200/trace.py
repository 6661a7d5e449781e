"""AKVT attention traces: the reference's wire/disk format for recorded
per-(layer, head, position) K/V/Q rows (reference: trace.py:1-349), read
in bulk and staged onto the GPU for replay through K1/K2/K3.

Format (little endian, written by ``write_trace`` byte-identically to the
reference):

    "AKVT" | u16 version=1 | u32 layers, heads, head_dim, vocab | i64 seed
    | u32 n_tokens | n_tokens x (u32 id, u8 class: 0 special 1 punct 2 other)
    | blocks, sorted by (layer, head) then step:
      u16 layer, u16 head, u32 step, then K, V, Q each as u32 n + n x f64

Reading is vectorised: when every block carries head_dim-long rows (the
normal case) the block region is viewed as one structured numpy array - no
per-block Python work - and ``trace_tensors`` turns a complete trace into
head-major device tensors [1, G, T, d] in one host->device copy per
operand; heads then run through the tensor entry points
(``replay_tensors``).  Irregular or damaged files take a sequential scan
that reports the same errors as the reference (TraceHeaderError,
TraceTruncatedError, TraceDimensionError with its messages).  The NDJSON
variant is supported for hand-written fixtures.
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .tokens import TokenAnnotation, TokenClass, VocabMetadata

MAGIC = b"AKVT"
VERSION = 1
_HEAD = struct.Struct("<4sH")
_CONFIG = struct.Struct("<IIIIq")
_TAG = struct.Struct("<HHI")
_TOKEN = np.dtype([("id", "<u4"), ("code", "u1")])          # packed 5-byte records
_WIRE_CLASS = (TokenClass.SPECIAL, TokenClass.PUNCTUATION, TokenClass.OTHER)
_WIRE_CODE = {k: i for i, k in enumerate(_WIRE_CLASS)}
_ROLE_HEAD_WEIGHTS = 4   # spawn key of the seeded next-token head (model.py:119-124)


class ModelError(ValueError):
    """Invalid model configuration (model.py:48-49)."""


@dataclass(frozen=True)
class ModelConfig:
    """Grid and sizes of a (recorded) model (model.py:60-77)."""

    num_layers: int
    num_heads: int
    head_dim: int
    vocab_size: int
    seed: int

    def __post_init__(self):
        for name in ("num_layers", "num_heads", "head_dim", "vocab_size"):
            value = getattr(self, name)
            if value < 1:
                raise ModelError(f"{name} must be >= 1, got {value}")

    def head_grid(self) -> list:
        return [(layer, head) for layer in range(self.num_layers) for head in range(self.num_heads)]


def linear_head_weights(config: ModelConfig) -> np.ndarray:
    """The seeded next-token projection shared by synthetic and trace models
    (model.py:119-124): uniform(-1, 1) / sqrt(L*H*d) from the config seed."""
    dim = config.num_layers * config.num_heads * config.head_dim
    seq = np.random.SeedSequence(entropy=config.seed, spawn_key=(_ROLE_HEAD_WEIGHTS,))
    gen = np.random.Generator(np.random.PCG64(seq))
    return gen.uniform(-1.0, 1.0, (config.vocab_size, dim)) / math.sqrt(dim)


class TraceError(Exception):
    """Base class of trace file problems (trace.py:30-44)."""


class TraceHeaderError(TraceError):
    """Bad magic, version or config counts."""


class TraceDimensionError(TraceError):
    """Rows or indices inconsistent with the declared config."""


class TraceTruncatedError(TraceError):
    """The data ends inside a structure."""


@dataclass(frozen=True)
class TraceBlock:
    step: int
    k: np.ndarray
    v: np.ndarray
    q: np.ndarray


@dataclass
class AttentionTrace:
    """Recorded rows per (layer, head), steps strictly increasing; every row
    finite and head_dim long (validated on construction, trace.py:55-86)."""

    config: ModelConfig
    tokens: list
    blocks: dict = field(default_factory=dict)

    def __post_init__(self):
        cfg = self.config
        for (layer, head), entries in self.blocks.items():
            if not 0 <= layer < cfg.num_layers:
                raise TraceDimensionError(f"layer {layer} out of range")
            if not 0 <= head < cfg.num_heads:
                raise TraceDimensionError(f"head {head} out of range")
            steps = np.fromiter((b.step for b in entries), dtype=np.int64, count=len(entries))
            bad = np.flatnonzero(np.diff(steps) <= 0)
            if bad.size:
                raise TraceDimensionError(
                    f"steps not strictly increasing at (layer={layer}, head={head}, "
                    f"step={int(steps[bad[0] + 1])})")
            for b in entries:
                for name, row in (("K", b.k), ("V", b.v), ("Q", b.q)):
                    where = f"(layer={layer}, head={head}, step={b.step})"
                    if row.shape != (cfg.head_dim,):
                        raise TraceDimensionError(
                            f"{name} row at {where} has length {row.shape}, "
                            f"expected {cfg.head_dim}")
                    if not np.isfinite(row).all():
                        raise TraceDimensionError(f"{name} row at {where} has non-finite entries")

    def vocab_metadata(self) -> VocabMetadata:
        """Special / punctuation id sets recovered from the token table
        (trace.py:88-94); an id recorded as both counts as special."""
        special = {t.token_id for t in self.tokens if t.klass is TokenClass.SPECIAL}
        punct = {t.token_id for t in self.tokens if t.klass is TokenClass.PUNCTUATION}
        return VocabMetadata(frozenset(special), frozenset(punct - special))

    def dense_rows(self):
        """(k, v, q) float64 [G, T, d] in head-grid order when every head
        records exactly positions 0..T-1 (T = token count), else None."""
        grid = self.config.head_grid()
        T, d = len(self.tokens), self.config.head_dim
        out = np.empty((3, len(grid), T, d))
        for gi, key in enumerate(grid):
            entries = self.blocks.get(key)
            if entries is None or len(entries) != T or any(b.step != i for i, b in
                                                             enumerate(entries)):
                return None
            for i, b in enumerate(entries):
                out[0, gi, i], out[1, gi, i], out[2, gi, i] = b.k, b.v, b.q
        return out[0], out[1], out[2]


# ---------------------------------------------------------------------------
# writing

def _encode(trace: AttentionTrace) -> bytes:
    cfg = trace.config
    parts = [_HEAD.pack(MAGIC, VERSION),
             _CONFIG.pack(cfg.num_layers, cfg.num_heads, cfg.head_dim, cfg.vocab_size, cfg.seed),
             struct.pack("<I", len(trace.tokens))]
    table = np.empty(len(trace.tokens), dtype=_TOKEN)
    table["id"] = [t.token_id for t in trace.tokens]
    table["code"] = [_WIRE_CODE[t.klass] for t in trace.tokens]
    parts.append(table.tobytes())
    for key in sorted(trace.blocks):
        for b in trace.blocks[key]:
            parts.append(_TAG.pack(key[0], key[1], b.step))
            for row in (b.k, b.v, b.q):
                arr = np.ascontiguousarray(row, dtype="<f8")
                parts.append(struct.pack("<I", arr.size))
                parts.append(arr.tobytes())
    return b"".join(parts)


def write_trace(trace: AttentionTrace, sink):
    """Binary AKVT to a path or a binary file object (trace.py:123-129)."""
    data = _encode(trace)
    if hasattr(sink, "write"):
        sink.write(data)
    else:
        with open(sink, "wb") as fh:
            fh.write(data)


def write_trace_ndjson(trace: AttentionTrace, sink):
    """The NDJSON variant: header line, token-table line, one line per block
    (trace.py:132-178)."""
    cfg = trace.config
    header = {"magic": "AKVT", "version": VERSION,
              "config": {"num_layers": cfg.num_layers, "num_heads": cfg.num_heads,
                         "head_dim": cfg.head_dim, "vocab_size": cfg.vocab_size,
                         "seed": cfg.seed}}
    lines = [json.dumps(header, sort_keys=True),
             json.dumps({"tokens": [{"id": t.token_id, "klass": t.klass.value}
                                    for t in trace.tokens]}, sort_keys=True)]
    for key in sorted(trace.blocks):
        for b in trace.blocks[key]:
            lines.append(json.dumps({"layer": key[0], "head": key[1], "step": b.step,
                                     "k": b.k.tolist(), "v": b.v.tolist(), "q": b.q.tolist()},
                                    sort_keys=True))
    text = "\n".join(lines) + "\n"
    if hasattr(sink, "write"):
        sink.write(text)
    else:
        with open(sink, "w", encoding="utf-8") as fh:
            fh.write(text)


# ---------------------------------------------------------------------------
# reading

def _need(data: bytes, off: int, n: int, what: str):
    if off + n > len(data):
        raise TraceTruncatedError(f"truncated payload while reading {what}")


def _block_dtype(d: int) -> np.dtype:
    row = [("n", "<u4"), ("x", "<f8", (d,))]
    return np.dtype([("layer", "<u2"), ("head", "<u2"), ("step", "<u4"),
                     ("k", np.dtype(row)), ("v", np.dtype(row)), ("q", np.dtype(row))])


def _blocks_bulk(data: bytes, off: int, d: int):
    """Uniform block region as one structured array, or None."""
    dt = _block_dtype(d)
    rest = len(data) - off
    if rest % dt.itemsize:
        return None
    arr = np.frombuffer(data, dtype=dt, offset=off)
    for r in ("k", "v", "q"):
        if not (arr[r]["n"] == d).all():
            return None
    return arr


def _blocks_scan(data: bytes, off: int) -> dict:
    blocks: dict = {}
    while off < len(data):
        _need(data, off, _TAG.size, "block tag")
        layer, head, step = _TAG.unpack_from(data, off)
        off += _TAG.size
        rows = []
        for name in ("K", "V", "Q"):
            _need(data, off, 4, f"{name} length at step {step}")
            (n,) = struct.unpack_from("<I", data, off)
            off += 4
            _need(data, off, 8 * n, f"{name} row at step {step}")
            rows.append(np.frombuffer(data, dtype="<f8", count=n, offset=off).astype(np.float64))
            off += 8 * n
        blocks.setdefault((layer, head), []).append(TraceBlock(step, *rows))
    return blocks


def _parse_binary(data: bytes) -> AttentionTrace:
    if len(data) < 4 or data[:4] != MAGIC:
        raise TraceHeaderError(f"malformed header: bad magic {data[:4]!r}")
    _need(data, 4, 2, "version")
    (version,) = struct.unpack_from("<H", data, 4)
    if version != VERSION:
        raise TraceHeaderError(f"unsupported version {version}")
    _need(data, 6, _CONFIG.size, "model config")
    try:
        config = ModelConfig(*_CONFIG.unpack_from(data, 6))
    except ModelError as exc:
        raise TraceHeaderError(f"malformed header: {exc}") from exc
    off = 6 + _CONFIG.size
    _need(data, off, 4, "token count")
    (ntok,) = struct.unpack_from("<I", data, off)
    off += 4
    # errors in the order a sequential reader meets them: an unknown class
    # code among the complete records, else the first record that does not fit
    avail = min(ntok, (len(data) - off) // _TOKEN.itemsize)
    table = np.frombuffer(data, dtype=_TOKEN, count=avail, offset=off)
    bad = np.flatnonzero(table["code"] > 2)
    if bad.size:
        raise TraceHeaderError(f"token {int(bad[0])}: unknown class code {int(table['code'][bad[0]])}")
    if avail < ntok:
        raise TraceTruncatedError(f"truncated payload while reading token {avail}")
    tokens = [TokenAnnotation(i, int(t), _WIRE_CLASS[c])
              for i, (t, c) in enumerate(zip(table["id"].tolist(), table["code"].tolist()))]
    off += ntok * _TOKEN.itemsize
    arr = _blocks_bulk(data, off, config.head_dim)
    if arr is None:
        return AttentionTrace(config, tokens, _blocks_scan(data, off))
    blocks: dict = {}
    keys = arr["layer"].astype(np.int64) * 65536 + arr["head"]
    cut = np.flatnonzero(np.diff(keys)) + 1
    for lo, hi in zip(np.r_[0, cut], np.r_[cut, len(arr)]):
        if hi <= lo:
            continue
        seg = arr[lo:hi]
        k, v, q = (np.array(seg[r]["x"], dtype=np.float64) for r in ("k", "v", "q"))
        key = (int(seg["layer"][0]), int(seg["head"][0]))
        lst = blocks.setdefault(key, [])
        lst.extend(TraceBlock(int(s), k[i], v[i], q[i]) for i, s in enumerate(seg["step"].tolist()))
    return AttentionTrace(config, tokens, blocks)


def _parse_ndjson(text: str) -> AttentionTrace:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise TraceHeaderError("malformed header: empty file")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as exc:
        raise TraceHeaderError(
            f"malformed header: no AKVT magic and first line is not JSON ({exc})") from exc
    if not isinstance(header, dict) or header.get("magic") != "AKVT":
        raise TraceHeaderError("malformed header: missing AKVT magic")
    if header.get("version") != VERSION:
        raise TraceHeaderError(f"unsupported version {header.get('version')}")
    try:
        config = ModelConfig(**header["config"])
    except (TypeError, KeyError, ModelError) as exc:
        raise TraceHeaderError(f"malformed header: {exc}") from exc
    if len(lines) < 2:
        raise TraceTruncatedError("truncated payload: missing token table")
    tokens = []
    for pos, entry in enumerate(json.loads(lines[1]).get("tokens", [])):
        try:
            klass = TokenClass(entry["klass"])
        except ValueError as exc:
            raise TraceHeaderError(f"token {pos}: unknown class {entry['klass']!r}") from exc
        tokens.append(TokenAnnotation(pos, int(entry["id"]), klass))
    blocks: dict = {}
    for line in lines[2:]:
        try:
            rec = json.loads(line)
            key = (int(rec["layer"]), int(rec["head"]))
            blk = TraceBlock(int(rec["step"]), *(np.asarray(rec[r], dtype=np.float64)
                                                  for r in ("k", "v", "q")))
        except (json.JSONDecodeError, KeyError, ValueError) as exc:
            raise TraceTruncatedError(f"truncated payload: bad block line: {exc}") from exc
        blocks.setdefault(key, []).append(blk)
    return AttentionTrace(config, tokens, blocks)


def read_trace(source) -> AttentionTrace:
    """Binary AKVT or NDJSON from a path or a binary file object (trace.py:277-290)."""
    if hasattr(source, "read"):
        data = source.read()
    else:
        with open(source, "rb") as fh:
            data = fh.read()
    if data[:4] == MAGIC:
        return _parse_binary(data)
    try:
        text = data.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise TraceHeaderError("malformed header: neither AKVT binary nor NDJSON") from exc
    return _parse_ndjson(text)


# ---------------------------------------------------------------------------
# replay

class TraceModel:
    """The reference's model protocol over recorded rows (trace.py:293-349):
    teacher-forced K/V/Q rows, the seeded linear next-token head."""

    def __init__(self, trace: AttentionTrace):
        self.trace = trace
        self.config = trace.config
        self.vocab = trace.vocab_metadata()
        self.max_context = len(trace.tokens)
        self._rows = {}
        for key in self.config.head_grid():
            entries = trace.blocks.get(key)
            if entries is None:
                raise TraceDimensionError(f"trace has no blocks for (layer={key[0]}, head={key[1]})")
            by_step = {b.step: b for b in entries}
            missing = [s for s in range(self.max_context) if s not in by_step]
            if missing:
                raise TraceDimensionError(
                    f"trace is missing steps {missing[:4]} for (layer={key[0]}, head={key[1]})")
            self._rows[key] = by_step
        self._head = linear_head_weights(self.config)

    def _row(self, layer, head, pos) -> TraceBlock:
        if pos >= self.max_context:
            raise ModelError(f"position {pos} beyond trace length {self.max_context}")
        return self._rows[(layer, head)][pos]

    def prompt_token_ids(self, prompt_len: int) -> list:
        if prompt_len > len(self.trace.tokens):
            raise ModelError(
                f"prompt_len {prompt_len} exceeds trace length {len(self.trace.tokens)}")
        return [t.token_id for t in self.trace.tokens[:prompt_len]]

    def k_row(self, layer, head, pos, klass, prompt_len):
        return self._row(layer, head, pos).k

    def v_row(self, layer, head, pos):
        return self._row(layer, head, pos).v

    def q_row(self, layer, head, pos, prompt_len):
        return self._row(layer, head, pos).q

    def head_logits(self, concat):
        return self._head @ concat


def trace_tensors(trace: AttentionTrace, dtype=None, device=None):
    """Stage a complete trace on the GPU: (q, k, v) [1, G, T, d] in head-grid
    order and token classes [1, T] (uint8 0 other / 1 special / 2 punct), one
    host->device copy per operand, cast on the device."""
    import torch

    from .tokens import CLASS_CODE

    dense = trace.dense_rows()
    if dense is None:
        raise TraceDimensionError("trace is not dense: every head must record positions 0..T-1")
    dev = torch.device("cuda") if device is None else torch.device(device)
    dt = torch.float32 if dtype is None else dtype
    k, v, q = (torch.from_numpy(x).to(dev).to(dt).unsqueeze(0) for x in dense)
    cls = torch.tensor([[CLASS_CODE[t.klass] for t in trace.tokens]], dtype=torch.uint8,
                       device=dev)
    return q.contiguous(), k.contiguous(), v.contiguous(), cls


def replay_tensors(trace: AttentionTrace, prompt_len: int, profiler_cfg=None, fixed_policy=None,
                   dtype=None, diagnostics: bool = False):
    """Teacher-forced replay of a recorded run on the GPU: profile + compact
    the first ``prompt_len`` positions of every head, then one decode step
    per remaining recorded position.  Returns (ProfileResult, cache, outputs
    [steps, 1, G, d] fp32)."""
    import torch

    from .engine import decode_steps_tensors, encode_prompt_tensors

    q, k, v, cls = trace_tensors(trace, dtype)
    T = q.shape[2]
    if not 1 <= prompt_len <= T:
        raise TraceDimensionError(f"prompt_len {prompt_len} out of range for {T} positions")
    steps = T - prompt_len
    res, cache = encode_prompt_tensors(q, k, v, cls, profiler_cfg, fixed_policy,
                                       prompt_len=prompt_len, max_new_tokens=max(steps, 1),
                                       diagnostics=diagnostics)
    outs = torch.empty(max(steps, 0), 1, q.shape[1], q.shape[3], dtype=torch.float32,
                       device=q.device)
    if steps > 0:   # the recorded positions, teacher-forced, in one library call
        decode_steps_tensors(cache, q[:, :, prompt_len:], k[:, :, prompt_len:],
                             v[:, :, prompt_len:], cls[:, prompt_len:].t().contiguous(),
                             out=outs, chained=True)
    return res, cache, outs
