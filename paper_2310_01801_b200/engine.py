"""Two-phase generation over the compressed KV cache (reference:
engine.py:39-525), B200-native.

Phase one (``encode_prompt``) runs K1 (profiling) and K2 (compaction) on
the GPU; phase two (``generate_step``) runs one K3 launch per token for all
heads.  The reference's duck-typed model protocol
(``config``/``vocab``/``k_row``/``v_row``/``q_row``/``head_logits``,
model.py:150-286) is kept for drop-in use; ``encode_prompt_tensors`` /
``decode_step_tensors`` are the tensor-level entry points the model-protocol
functions are built on: q, k, v are device tensors ``[B, H, ld, d]``
(fp32 or bf16), every (b, h) an independent head.

The host only orchestrates: it allocates device memory (PyTorch is used
for allocation and streams), reads back the per-head profile once after
K1 (one small device->host copy that also sizes the ragged arena - or, with
an ``ArenaPool``, no synchronous read at all), and launches kernels.  There
is no CPU compute path.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (CRIT_COSINE, CRIT_RECOVERY, DTYPE_BF16, DTYPE_F32, ROWS_ALL, ROWS_LAST,
                   CompactArgs, DecodeArgs, ProfileArgs, check, lib)
from .policies import CompressionPolicy, full_policy
from .profiler import (HeadDecision, HeadProfile, ProfilerConfig, ProfilerError, RowAveraging,
                       SelectionCriterion)
from .tokens import CLASS_CODE, TokenAnnotation, classify_tokens


class EngineError(ValueError):
    """Invalid generation state or configuration (engine.py:39-40)."""


@dataclass(frozen=True)
class GreedyArgmax:
    pass


@dataclass(frozen=True)
class Nucleus:
    temperature: float = 0.6
    top_p: float = 0.9
    seed: int = 0

    def __post_init__(self):
        if self.temperature <= 0.0:
            raise EngineError(f"temperature must be > 0, got {self.temperature}")
        if not 0.0 < self.top_p <= 1.0:
            raise EngineError(f"top_p must be in (0, 1], got {self.top_p}")


@dataclass(frozen=True)
class GenerationConfig:
    max_new_tokens: int
    sampling: object = field(default_factory=GreedyArgmax)

    def __post_init__(self):
        if self.max_new_tokens < 0:
            raise EngineError("max_new_tokens must be >= 0")


class _Sampler:
    """Next-token choice from the model's logits (engine.py:71-90)."""

    def __init__(self, sampling):
        self.sampling = sampling
        self._rng = (np.random.Generator(np.random.PCG64(sampling.seed))
                     if isinstance(sampling, Nucleus) else None)

    def __call__(self, logits) -> int:
        logits = np.asarray(logits, dtype=np.float64)
        if isinstance(self.sampling, GreedyArgmax):
            return int(np.argmax(logits))
        z = logits / self.sampling.temperature
        z = np.exp(z - z.max())
        probs = z / z.sum()
        order = np.argsort(-probs, kind="stable")
        cum = np.cumsum(probs[order])
        cut = min(int(np.searchsorted(cum, self.sampling.top_p, side="left")), probs.size - 1)
        kept = order[:cut + 1]
        return int(self._rng.choice(kept, p=probs[kept] / probs[kept].sum()))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    raise EngineError(f"unsupported dtype {t.dtype}; use float32 or bfloat16")


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class ProfileResult:
    """Everything K1 reports per head (flattened g = b*H + h)."""

    family: tuple                 # CompressionPolicy per family member
    thresholds: tuple
    recovery: np.ndarray          # [G, F]
    cost: np.ndarray              # [G, F]
    cosine: np.ndarray            # [G, F]
    choice: np.ndarray            # [G, nT]
    kept_count: np.ndarray        # [G]
    last_row_recovery: np.ndarray  # [G]
    topk_gap: np.ndarray          # [G]

    def near_threshold(self, tol: float = 1e-4) -> np.ndarray:
        """Heads whose recovery of any member up to the chosen one lies within
        ``tol`` of T (listed separately by the parity contract)."""
        G, F = self.recovery.shape
        out = np.zeros((G, len(self.thresholds)), dtype=bool)
        for t, T in enumerate(self.thresholds):
            for g in range(G):
                c = self.choice[g, t]
                upto = F if c < 0 else c + 1
                out[g, t] = bool(np.any(np.abs(self.recovery[g, :upto] - T) < tol))
        return out

    def policies(self, t: int = 0) -> list:
        return [self.family[c] for c in self.choice[:, t]]


class CompressedCache:
    """Per-head compressed KV state of one batch of sessions, resident in HBM
    (engine.py:100-144).  Head g = b*H + h owns arena slots
    [seg_off[g], seg_off[g] + seg_cap[g])."""

    def __init__(self, B, H, d, dtype, prompt_len, capacity_steps, device):
        self.B, self.H, self.d = B, H, d
        self.G = B * H
        self.dtype = dtype
        self.prompt_len = prompt_len
        self.seq_len = prompt_len
        self.capacity_steps = capacity_steps
        self.device = device
        self.profile: HeadProfile | None = None
        self.profile_result: ProfileResult | None = None
        self.keys: list = []
        self.annotations: list = []
        self.diagnostics = False
        self.last_record = None
        self._parity = 0

    # live slot counts (double-buffered across steps)
    @property
    def live(self) -> torch.Tensor:
        return self.live_buf[self._parity]

    def total_retained(self) -> int:
        return int(self.live.sum().item())

    def head_retained(self) -> np.ndarray:
        return self.live.cpu().numpy().astype(np.int64)

    def retained_positions(self, g: int | None = None):
        """Sorted live positions of head g (or a list for all heads); one
        device->host copy per call (diagnostics only)."""
        self.check()
        live = self.live.cpu().numpy()
        off = self.seg_off.cpu().numpy()
        meta = self.meta.cpu().numpy()
        def one(i):
            m = meta[off[i]: off[i] + live[i]]
            return np.sort(m & ((1 << 24) - 1))
        if g is not None:
            return one(g)
        return [one(i) for i in range(self.G)]

    @property
    def pending_output(self) -> torch.Tensor:
        """Latest attention output per head, fp32 [B, H, d]: the buffer the
        last decode step wrote (its ``out=`` argument when one was given)."""
        latest = getattr(self, "_latest_out", None)
        return self.out if latest is None else latest

    @property
    def heads(self) -> dict:
        """Host snapshot of every head's state in the reference's layout
        (engine.py:100-117 HeadCacheState), keyed by the model grid's
        (layer, head) keys (or (b, h) for tensor-level caches): live
        positions ascending (the reference keeps attended order, which is
        ascending), their K/V rows, the score sidecar, the pending output and
        the latest recovery.  ``scores`` is full length with NaN at evicted
        positions (the reference keeps their frozen values; only live slots
        take part in later decisions).  One device->host copy per call."""
        self.check()
        keys = self.keys or [(b, h) for b in range(self.B) for h in range(self.H)]
        live = self.live.cpu().numpy()
        off = self.seg_off.cpu().numpy()
        meta = self.meta.cpu().numpy()
        kc = self.kc.float().cpu().numpy()
        vc = self.vc.float().cpu().numpy()
        score = self.score.cpu().numpy()
        out = self.pending_output.reshape(self.G, -1).double().cpu().numpy()
        rec = self.step_recovery.cpu().numpy()
        atoms = self.head_atoms.cpu().numpy()
        fam = self.profile_result.family if self.profile_result is not None else ()
        by_bits = {pol.bits: pol for pol in fam}
        states = {}
        for g, key in enumerate(keys):
            sl = slice(int(off[g]), int(off[g]) + int(live[g]))
            pos = meta[sl] & ((1 << 24) - 1)
            order = np.argsort(pos, kind="stable")
            freq = bool(atoms[g] & 4) and not bool(atoms[g] & 16)
            scores = None
            if freq:
                scores = np.full(self.seq_len, np.nan)
                scores[pos] = score[sl]
            states[key] = HeadCacheState(
                policy=self.profile.decisions[key].policy if (self.profile is not None and
                                                              key in self.profile.decisions)
                else by_bits.get(int(atoms[g])),
                positions=[int(p) for p in pos[order]], K=kc[sl][order], V=vc[sl][order],
                scores=scores, pending_output=out[g], last_row_recovery=float(rec[g]))
        return states

    def check(self):
        st = int(self.status.item())
        if st != 0:
            raise _lib.AkvError(st, "capacity exceeded: a cache segment or the arena pool "
                                    "cannot hold the retained rows")


@dataclass
class HeadCacheState:
    """One head's compressed state (engine.py:100-117), as a host snapshot."""

    policy: CompressionPolicy | None
    positions: list
    K: np.ndarray
    V: np.ndarray
    scores: np.ndarray | None
    pending_output: np.ndarray
    last_row_recovery: float

    @property
    def sidecar(self):
        """Cumulative scores of the retained positions (engine.py:112-117)."""
        if self.scores is None:
            return None
        return self.scores[np.asarray(self.positions, dtype=np.intp)]


class ArenaPool:
    """Device memory for compressed caches with a device-side bump allocator
    (``akv_plan_segments_pool``): ``encode_prompt_tensors(..., pool=pool)``
    carves its ragged segments from the pool without the host read that sizes
    a private arena, so profiling, compaction and decoding are enqueued
    back to back.  ``reset()`` (stream-ordered) releases every segment carved
    so far; a session that does not fit flags a capacity error
    (``CompressedCache.check``)."""

    def __init__(self, slots: int, d: int, dtype=torch.bfloat16, device=None):
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.slots, self.d, self.dtype, self.device = int(slots), int(d), dtype, dev
        self.kc = torch.empty(self.slots, d, dtype=dtype, device=dev)
        self.vc = torch.empty(self.slots, d, dtype=dtype, device=dev)
        self.meta = torch.empty(self.slots, dtype=torch.int32, device=dev)
        self.score = torch.empty(self.slots, dtype=torch.float64, device=dev)
        self.used = torch.zeros(1, dtype=torch.int64, device=dev)

    def reset(self):
        self.used.zero_()

    def used_slots(self) -> int:
        return int(self.used.item())


class _PendingProfile:
    """A ProfileResult whose device->host copy is still in flight (pool
    sessions): materialised, and any profiling error raised, on first use."""

    def __init__(self, build, event):
        self._build, self._event, self._res = build, event, None

    def _get(self):
        if self._res is None:
            self._event.synchronize()
            self._res = self._build()
        return self._res

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self._get(), name)


def _family_arrays(family, args):
    if len(family) > _lib.MAX_FAMILY:
        raise ProfilerError(f"feasible family longer than {_lib.MAX_FAMILY} policies")
    args.n_family = len(family)
    for i, pol in enumerate(family):
        args.family_atoms[i] = pol.bits
        args.family_r_l[i] = pol.r_l
        args.family_r_f[i] = pol.r_f


def encode_prompt_tensors(q, k, v, classes, profiler_cfg: ProfilerConfig | None = None,
                          fixed_policy: CompressionPolicy | None = None, *, prompt_len=None,
                          max_new_tokens: int = 0, extra_thresholds=(), slopes=None,
                          sinks=None, diagnostics: bool = False, local_len: int = 0,
                          k1_events=None, pool: ArenaPool | None = None):
    """Profile, select and compact every head of a batch (Alg. 1,
    engine.py:203-272) on the GPU.

    q, k, v: CUDA tensors [B, H, ld, d] (float32 or bfloat16); the first
    ``prompt_len`` rows of every head are the prompt.  classes: CUDA uint8
    [B, >= prompt_len] token classes (0 other, 1 special, 2 punct).
    slopes/sinks: optional CUDA float32 [H] planted head bias (synthetic
    workloads).  Returns (ProfileResult, CompressedCache) with capacity for
    ``max_new_tokens`` inserted tokens per head.

    ``diagnostics=True`` also keeps every key by position (the reference's
    shadow keys, engine.py:260-261) so that each decode step reports the
    recovery of its attended set against uncompressed attention
    (``cache.step_recovery``, engine.py:341-349).

    ``pool``: carve the compressed cache from an ArenaPool instead of a
    private arena sized by a host read; the returned ProfileResult then
    materialises lazily (its host copy overlaps the compaction and decoding).
    """
    if profiler_cfg is None and fixed_policy is None:
        raise EngineError("need a profiler config or a fixed policy")
    _lib.require_device()
    if q.dim() != 4 or q.shape != k.shape or q.shape != v.shape:
        raise EngineError("q, k, v must be [B, H, ld, d] tensors of one shape")
    if not (q.is_cuda and k.is_cuda and v.is_cuda and classes.is_cuda):
        raise EngineError("inputs must be CUDA tensors")
    for t in (q, k, v):
        if not t.is_contiguous():
            raise EngineError("q, k, v must be contiguous")
    B, H, ld, d = q.shape
    N = ld if prompt_len is None else int(prompt_len)
    if N < 1:
        raise EngineError("empty prompt")
    if N > ld:
        raise EngineError(f"prompt_len {N} out of range for {ld} rows")
    dt = _dtype_code(q)
    dev = q.device
    G = B * H
    if fixed_policy is not None:
        family = (fixed_policy,)
        thresholds = (-1.0,)
        rows, crit = ROWS_ALL, CRIT_RECOVERY
    else:
        family = tuple(profiler_cfg.feasible)
        thresholds = (profiler_cfg.recovery_threshold,) + tuple(extra_thresholds)
        rows = ROWS_LAST if profiler_cfg.rows is RowAveraging.LAST_ROW else ROWS_ALL
        crit = (CRIT_COSINE if profiler_cfg.criterion is SelectionCriterion.COSINE_SIMILARITY
                else CRIT_RECOVERY)
    if len(thresholds) > _lib.MAX_THRESHOLDS:
        raise ProfilerError(f"at most {_lib.MAX_THRESHOLDS} thresholds per profiling pass")
    F = len(family)
    nT = len(thresholds)
    f32, f64, i32 = torch.float32, torch.float64, torch.int32
    classes = classes.to(torch.uint8).contiguous()
    # per-head summary outputs share one device buffer -> one device->host copy
    sections = [("recovery", G * F, f64), ("cosine", G * F, f64), ("lrr", G, f64),
                ("gap", G, f64), ("total", 1, torch.int64), ("cost", G * F, i32),
                ("kept_count", G, i32), ("choice", G * nT, torch.int8)]
    offs, nbytes = {}, 0
    for name, n, dtp in sections:
        offs[name] = (nbytes, n, dtp)
        nbytes += ((n * torch.empty(0, dtype=dtp).element_size() + 7) // 8) * 8
    summary = torch.empty(nbytes, dtype=torch.uint8, device=dev)

    def view(buf, name):
        o, n, dtp = offs[name]
        return buf[o:o + n * torch.empty(0, dtype=dtp).element_size()].view(dtp)

    out = {name: view(summary, name) for name, _, _ in sections}
    out.update(
        thr_key=torch.empty(G, dtype=torch.int64, device=dev),
        thr_pos=torch.empty(G, dtype=i32, device=dev),
        lse=torch.empty(G, N, dtype=f32, device=dev),
        colsum=torch.empty(G, N, dtype=f64, device=dev),
        colsq=torch.empty(G, N, dtype=f64, device=dev),
        lastp=torch.empty(G, N, dtype=f32, device=dev),
        out_last=torch.empty(B, H, d, dtype=f32, device=dev),
        kept_pos=torch.empty(G, N, dtype=i32, device=dev),
    )
    ws_bytes = lib.akv_profile_workspace_size(B, H, N, d)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    a = ProfileArgs()
    a.B, a.H, a.N, a.d, a.dtype = B, H, N, d, dt
    a.q_dev, a.k_dev, a.v_dev, a.ld = _ptr(q), _ptr(k), _ptr(v), ld
    a.cls_dev, a.cls_ld = _ptr(classes), classes.shape[1]
    a.slope_dev, a.sink_dev = _ptr(slopes), _ptr(sinks)
    _family_arrays(family, a)
    a.n_thresholds = nT
    for i, t in enumerate(thresholds):
        a.thresholds[i] = t
    a.rows, a.criterion = rows, crit
    (a.lse_dev, a.colsum_dev, a.colsq_dev, a.lastp_dev, a.out_last_dev, a.recovery_dev,
     a.cost_dev, a.cosine_dev, a.choice_dev, a.kept_pos_dev, a.kept_count_dev,
     a.last_row_recovery_dev, a.topk_gap_dev) = (
        _ptr(out[n]) for n in ("lse", "colsum", "colsq", "lastp", "out_last", "recovery", "cost",
                               "cosine", "choice", "kept_pos", "kept_count", "lrr", "gap"))
    a.topk_thr_key_dev, a.topk_thr_pos_dev = _ptr(out["thr_key"]), _ptr(out["thr_pos"])
    a.workspace_dev, a.workspace_bytes = _ptr(ws), ws_bytes
    a.local_len = int(local_len)
    stream = _stream()
    if k1_events is not None:   # (start, end) CUDA events around akv_profile (bench.py)
        k1_events[0].record()
    check(lib.akv_profile(C.byref(a), stream), ProfilerError)
    if k1_events is not None:
        k1_events[1].record()

    # Everything the compaction needs except the arena is prepared before the
    # session's single device->host read (the packed summary, which also
    # carries the arena size); after it only the arena allocation stands
    # between the read and the next launches, so the GPU idles briefly.
    seg_cap = torch.empty(G, dtype=i32, device=dev)
    seg_off = torch.empty(G, dtype=torch.int64, device=dev)
    cache = CompressedCache(B, H, d, q.dtype, N, int(max_new_tokens), dev)
    cache.status = torch.zeros(1, dtype=i32, device=dev)
    if pool is None:
        check(lib.akv_plan_segments(G, _ptr(out["kept_count"]), int(max_new_tokens),
                                    _ptr(seg_cap), _ptr(seg_off), _ptr(out["total"]), stream))
    else:
        if pool.d != d or pool.dtype != q.dtype or pool.device != dev:
            raise EngineError("arena pool does not match the cache's head dim / dtype / device")
        check(lib.akv_plan_segments_pool(G, _ptr(out["kept_count"]), int(max_new_tokens),
                                         _ptr(seg_cap), _ptr(seg_off), _ptr(out["total"]),
                                         _ptr(pool.used), pool.slots, _ptr(cache.status), stream))
    cache.head_atoms = torch.empty(G, dtype=torch.uint8, device=dev)
    cache.head_r_l = torch.empty(G, dtype=f64, device=dev)
    cache.head_r_f = torch.empty(G, dtype=f64, device=dev)
    cache.seg_cap, cache.seg_off = seg_cap, seg_off
    cache.max_cap = int(max(1, ((N + max_new_tokens + 7) // 8) * 8))
    cache.live_buf = [torch.empty(G, dtype=i32, device=dev), torch.empty(G, dtype=i32, device=dev)]
    cache.base_live = torch.empty(G, dtype=i32, device=dev)
    cache.out = out["out_last"]
    cache.evicted = torch.zeros(G, dtype=i32, device=dev)
    cache.classes = classes
    cache.slopes, cache.sinks = slopes, sinks
    cache.colsum = out["colsum"]
    cache.lastp = out["lastp"]
    c = CompactArgs()
    c.B, c.H, c.N, c.d, c.dtype = B, H, N, d, dt
    c.k_dev, c.v_dev, c.ld = _ptr(k), _ptr(v), ld
    c.cls_dev, c.cls_ld = _ptr(classes), classes.shape[1]
    c.kept_pos_dev, c.kept_count_dev, c.colsum_dev = (_ptr(out["kept_pos"]),
                                                      _ptr(out["kept_count"]), _ptr(out["colsum"]))
    c.choice_dev, c.choice_stride = _ptr(out["choice"]), nT
    c.topk_thr_key_dev, c.topk_thr_pos_dev = _ptr(out["thr_key"]), _ptr(out["thr_pos"])
    c.n_family = F
    for i, pol in enumerate(family):
        c.family_atoms[i], c.family_r_l[i], c.family_r_f[i] = pol.bits, pol.r_l, pol.r_f
    c.head_atoms_dev, c.head_r_l_dev, c.head_r_f_dev = (_ptr(cache.head_atoms),
                                                        _ptr(cache.head_r_l), _ptr(cache.head_r_f))
    c.seg_off_dev, c.seg_cap_dev = _ptr(seg_off), _ptr(seg_cap)
    c.live_dev = _ptr(cache.live_buf[0])

    if pool is None:
        hsum = summary.cpu()
        total_slots = int(view(hsum, "total")[0])
        cache.total_slots = max(total_slots, 1)
        cache.kc = torch.empty(cache.total_slots, d, dtype=q.dtype, device=dev)
        cache.vc = torch.empty(cache.total_slots, d, dtype=q.dtype, device=dev)
        cache.meta = torch.empty(cache.total_slots, dtype=i32, device=dev)
        cache.score = torch.empty(cache.total_slots, dtype=f64, device=dev)
    else:
        hsum = torch.empty(summary.numel(), dtype=torch.uint8, pin_memory=True)
        hsum.copy_(summary, non_blocking=True)
        summary_ready = torch.cuda.Event()
        summary_ready.record()
        cache.total_slots = pool.slots
        cache.kc, cache.vc, cache.meta, cache.score = pool.kc, pool.vc, pool.meta, pool.score
        cache.pool = pool
    c.kc_dev, c.vc_dev, c.meta_dev, c.score_dev = (_ptr(cache.kc), _ptr(cache.vc),
                                                   _ptr(cache.meta), _ptr(cache.score))
    check(lib.akv_compact(C.byref(c), stream), EngineError)
    cache.base_live.copy_(cache.live_buf[0])  # the decode's live-count bound anchor
    ws_bytes = lib.akv_decode_workspace_size(B, H, d, cache.max_cap, cache.total_slots)
    cache.workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib.akv_decode_workspace_init(_ptr(cache.workspace), ws_bytes, B, H, d, cache.max_cap,
                                        cache.total_slots, stream))

    def build():
        host = {name: view(hsum, name).numpy() for name, _, _ in sections}
        choice = host["choice"].reshape(G, nT).astype(np.int64)
        if (choice < 0).any():
            raise ProfilerError("no feasible policy met the threshold")
        return ProfileResult(
            family=family, thresholds=thresholds, recovery=host["recovery"].reshape(G, F),
            cost=host["cost"].reshape(G, F).astype(np.int64), cosine=host["cosine"].reshape(G, F),
            choice=choice, kept_count=host["kept_count"].astype(np.int64),
            last_row_recovery=host["lrr"], topk_gap=host["gap"])

    res = build() if pool is None else _PendingProfile(build, summary_ready)
    cache.profile_result = res
    cache._dargs = _decode_args(cache, dt)
    cache.track_recovery = bool(diagnostics)
    # per-head recovery of the latest step; before any decode step it is the
    # prompt's last-row recovery (engine.py:256-258, 362-363)
    cache.step_recovery = view(summary, "lrr")
    if diagnostics:
        cache.shadow = torch.empty(G, N + int(max_new_tokens), d, dtype=q.dtype, device=dev)
        cache.shadow.view(B, H, -1, d)[:, :, :N].copy_(k[:, :, :N])
        cache.cls_hist = torch.zeros(B, N + int(max_new_tokens), dtype=torch.uint8, device=dev)
        cache.cls_hist[:, :N].copy_(classes[:, :N])
        cache.step_recovery = cache.step_recovery.clone()
        shadow_ld = cache.shadow.shape[1]
        ws = lib.akv_decode_recovery_workspace_size(B, H, shadow_ld)
        cache.diag_ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        check(lib.akv_decode_recovery_workspace_init(_ptr(cache.diag_ws), ws, B, H, shadow_ld,
                                                     stream))
        g = _lib.DiagArgs()
        g.B, g.H, g.d, g.dtype = B, H, d, dt
        g.slope_dev, g.sink_dev = _ptr(slopes), _ptr(sinks)
        g.seg_off_dev, g.meta_dev = _ptr(cache.seg_off), _ptr(cache.meta)
        g.shadow_dev, g.shadow_ld = _ptr(cache.shadow), shadow_ld
        g.cls_hist_dev, g.cls_ld = _ptr(cache.cls_hist), cache.cls_hist.shape[1]
        g.recovery_dev = _ptr(cache.step_recovery)
        g.head_atoms_dev = _ptr(cache.head_atoms)
        g.workspace_dev, g.workspace_bytes = _ptr(cache.diag_ws), ws
        cache._diag_args = g
    return res, cache


def grow_cache(cache: CompressedCache, extra_steps: int) -> None:
    """Room for ``extra_steps`` more decode steps.  The reference's per-head
    lists grow without bound (engine.py:315-317); here every head's segment
    gains ``extra_steps`` slots (rounded up to 8), the segments move to a new
    private arena (a device-side gather of each old segment), and the decode
    workspace - plus, in diagnostics mode, the position-indexed shadow keys
    and class history - are rebuilt.  The session continues bit-identically.
    One device->host read (the new arena size); not for a cache whose decode
    is captured in a CUDA graph (its pointers change)."""
    if extra_steps <= 0:
        return
    cache.check()
    dev, G, d = cache.device, cache.G, cache.d
    i64 = torch.int64
    old_cap = cache.seg_cap.to(i64)
    old_off = cache.seg_off.to(i64)
    new_cap = ((old_cap + int(extra_steps) + 7) // 8) * 8
    new_off = torch.cumsum(new_cap, 0) - new_cap
    total = max(int(new_cap.sum().item()), 1)
    n_old = int(old_cap.sum().item())
    seg = torch.repeat_interleave(torch.arange(G, device=dev), old_cap, output_size=n_old)
    j = torch.arange(n_old, device=dev) - (torch.cumsum(old_cap, 0) - old_cap)[seg]
    src, dst = old_off[seg] + j, new_off[seg] + j
    for name, width in (("kc", d), ("vc", d), ("meta", None), ("score", None)):
        old = getattr(cache, name)
        new = torch.empty((total, width) if width else (total,), dtype=old.dtype, device=dev)
        new[dst] = old[src]
        setattr(cache, name, new)
    cache.pool = None
    cache.seg_cap = new_cap.to(torch.int32)
    cache.seg_off = new_off
    cache.total_slots = total
    cache.max_cap = int(((cache.max_cap + int(extra_steps) + 7) // 8) * 8)
    cache.capacity_steps += int(extra_steps)
    B, H = cache.B, cache.H
    ws_bytes = lib.akv_decode_workspace_size(B, H, d, cache.max_cap, cache.total_slots)
    cache.workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib.akv_decode_workspace_init(_ptr(cache.workspace), ws_bytes, B, H, d, cache.max_cap,
                                        cache.total_slots, _stream()), EngineError)
    dt = DTYPE_BF16 if cache.dtype == torch.bfloat16 else DTYPE_F32
    cache._dargs = _decode_args(cache, dt)
    if cache.track_recovery:
        old_ld = cache.shadow.shape[1]
        ld = old_ld + int(extra_steps)
        shadow = torch.empty(G, ld, d, dtype=cache.shadow.dtype, device=dev)
        shadow[:, :old_ld].copy_(cache.shadow)
        cls_hist = torch.zeros(B, ld, dtype=torch.uint8, device=dev)
        cls_hist[:, :old_ld].copy_(cache.cls_hist)
        cache.shadow, cache.cls_hist = shadow, cls_hist
        ws = lib.akv_decode_recovery_workspace_size(B, H, ld)
        cache.diag_ws = torch.empty(ws, dtype=torch.uint8, device=dev)
        check(lib.akv_decode_recovery_workspace_init(_ptr(cache.diag_ws), ws, B, H, ld, _stream()),
              EngineError)
        g = cache._diag_args
        g.seg_off_dev, g.meta_dev = _ptr(cache.seg_off), _ptr(cache.meta)
        g.shadow_dev, g.shadow_ld = _ptr(cache.shadow), ld
        g.cls_hist_dev, g.cls_ld = _ptr(cache.cls_hist), ld
        g.workspace_dev, g.workspace_bytes = _ptr(cache.diag_ws), ws


def _launch_recovery(cache, q, k, new_classes, live_in, pos=None, pos_dev=None):
    """Before the decode step of the same position (pre-eviction live set)."""
    g = cache._diag_args
    g.pos = 0 if pos is None else pos
    g.pos_dev = _ptr(pos_dev)
    g.q_dev, g.k_dev, g.bh_stride = _ptr(q), _ptr(k), q.stride(1)
    g.new_cls_dev = _ptr(new_classes)
    g.live_in_dev = _ptr(live_in)
    check(lib.akv_decode_recovery(C.byref(g), _stream()), EngineError)


def _decode_args(cache: CompressedCache, dt: int) -> DecodeArgs:
    a = DecodeArgs()
    a.B, a.H, a.d, a.dtype, a.prompt_len = cache.B, cache.H, cache.d, dt, cache.prompt_len
    a.slope_dev, a.sink_dev = _ptr(cache.slopes), _ptr(cache.sinks)
    a.head_atoms_dev, a.head_r_l_dev, a.head_r_f_dev = (_ptr(cache.head_atoms),
                                                        _ptr(cache.head_r_l), _ptr(cache.head_r_f))
    a.seg_off_dev, a.seg_cap_dev = _ptr(cache.seg_off), _ptr(cache.seg_cap)
    a.kc_dev, a.vc_dev, a.meta_dev, a.score_dev = (_ptr(cache.kc), _ptr(cache.vc),
                                                   _ptr(cache.meta), _ptr(cache.score))
    a.base_live_dev = _ptr(cache.base_live)
    a.out_dev, a.evicted_dev, a.status_dev = _ptr(cache.out), _ptr(cache.evicted), _ptr(cache.status)
    a.max_cap, a.total_slots = cache.max_cap, cache.total_slots
    a.workspace_dev, a.workspace_bytes = _ptr(cache.workspace), cache.workspace.numel()
    return a


def _check_rows(cache: CompressedCache, q, k, v, step_dim: bool):
    """The kernels read head g = b*H + h of q / k / v at g * q.stride(1)
    elements (d contiguous values; k and v with q's strides)."""
    nd = 4 if step_dim else 3
    for name, x in (("q", q), ("k", k), ("v", v)):
        if (x.dim() != nd or not x.is_cuda or x.dtype != cache.dtype or
                tuple(x.shape[:2]) != (cache.B, cache.H) or x.shape[-1] < cache.d or
                x.stride(-1) != 1 or (cache.B > 1 and x.stride(0) != cache.H * x.stride(1)) or
                x.stride()[1:] != q.stride()[1:]):
            raise EngineError(
                f"{name} must be a CUDA {cache.dtype} tensor [B={cache.B}, H={cache.H}"
                f"{', steps' if step_dim else ''}, >=d={cache.d}] with contiguous rows, batch "
                "stride H x head stride, and the same strides as q")


def decode_step_tensors(cache: CompressedCache, q, k, v, new_classes, out=None, *,
                        chained: bool = False) -> torch.Tensor:
    """One decode step for every head (Alg. 2 inner loop, engine.py:303-350):
    insert the new token's k/v, attend, update scores, evict.  q, k, v:
    CUDA tensors whose [B, H, :d] slices are the new token's rows (any
    head stride); new_classes: CUDA uint8 [B].  Returns the fp32 attention
    output [B, H, d]: ``out`` if given (contiguous fp32), else the cache's
    pending-output buffer (overwritten by the next step).

    ``chained=True`` promises that q/k/v/new_classes were not produced by the
    kernel launched just before on this stream (they were resident, or
    uploaded by a copy), which lets the step stream settled cache pages
    while the previous step drains (AKV_DECODE_CHAINED)."""
    if cache.seq_len - cache.prompt_len >= cache.capacity_steps:
        raise EngineError(
            f"cache capacity of {cache.capacity_steps} decode steps exhausted; "
            "encode with a larger max_new_tokens")
    _check_rows(cache, q, k, v, step_dim=False)
    a = cache._dargs
    a.pos = cache.seq_len
    a.q_dev, a.k_dev, a.v_dev = _ptr(q), _ptr(k), _ptr(v)
    a.bh_stride = q.stride(1)
    a.new_cls_dev = _ptr(new_classes)
    a.live_in_dev = _ptr(cache.live_buf[cache._parity])
    a.live_out_dev = _ptr(cache.live_buf[cache._parity ^ 1])
    dst = cache.out if out is None else out
    a.out_dev = _ptr(dst)
    a.pos_dev = None
    a.flags = _lib.DECODE_CHAINED if chained else 0
    if cache.track_recovery:
        _launch_recovery(cache, q, k, new_classes, cache.live_buf[cache._parity], pos=cache.seq_len)
        a.flags = 0  # the recovery kernel sits between two decode steps
    check(lib.akv_decode_step(C.byref(a), _stream()), EngineError)
    cache._parity ^= 1
    cache.seq_len += 1
    cache._latest_out = dst
    return dst


def decode_steps_tensors(cache: CompressedCache, q, k, v, new_classes, out=None, *,
                         chained: bool = False) -> torch.Tensor:
    """n teacher-forced decode steps in one library call (the step loop runs
    in C++, akv_decode_steps): q, k, v are [B, H, n, >=d] CUDA tensors whose
    [:, :, t] slices are step t's new-token rows (the same strides for all
    three), ``new_classes`` is uint8 [n, B] (contiguous rows: step t's
    classes).  Returns the fp32 outputs: ``out`` [n, B, H, d] if given
    (contiguous), else the last step's output in the cache's pending-output
    buffer.  Same results as n calls of decode_step_tensors; ``chained``
    applies to the first step (later steps are chained by construction).
    Diagnostics-mode caches step one at a time (the recovery kernel runs
    between steps)."""
    n = int(q.shape[2])
    if new_classes.dim() != 2 or tuple(new_classes.shape) != (n, cache.B) or \
            (cache.B > 1 and new_classes.stride(1) != 1) or new_classes.dtype != torch.uint8:
        raise EngineError(f"new_classes must be a contiguous uint8 [{n}, {cache.B}] tensor")
    if k.shape[2] != n or v.shape[2] != n:
        raise EngineError("q, k and v must have the same number of steps")
    _check_rows(cache, q, k, v, step_dim=True)
    if out is not None and (tuple(out.shape) != (n, cache.B, cache.H, cache.d) or
                            not out.is_contiguous() or out.dtype != torch.float32):
        raise EngineError(f"out must be a contiguous float32 [{n}, {cache.B}, {cache.H}, {cache.d}]")
    if cache.track_recovery:
        for t in range(n):
            decode_step_tensors(cache, q[:, :, t], k[:, :, t], v[:, :, t], new_classes[t],
                                None if out is None else out[t], chained=chained)
        return cache.out if out is None else out
    if n == 0:
        return cache.out if out is None else out
    if cache.seq_len + n - cache.prompt_len > cache.capacity_steps:
        raise EngineError(
            f"cache capacity of {cache.capacity_steps} decode steps exhausted; "
            "encode with a larger max_new_tokens")
    a = cache._dargs
    a.pos = cache.seq_len
    a.q_dev, a.k_dev, a.v_dev = _ptr(q), _ptr(k), _ptr(v)
    a.bh_stride = q.stride(1)
    a.new_cls_dev = _ptr(new_classes)
    a.live_in_dev = _ptr(cache.live_buf[cache._parity])
    a.live_out_dev = _ptr(cache.live_buf[cache._parity ^ 1])
    a.out_dev = _ptr(cache.out)
    a.pos_dev = None
    a.flags = _lib.DECODE_CHAINED if chained else 0
    check(lib.akv_decode_steps(C.byref(a), n, q.stride(2), new_classes.stride(0),
                               _ptr(out), 0 if out is None else out[0].numel(), _stream()),
          EngineError)
    cache._parity ^= n & 1
    cache.seq_len += n
    cache._latest_out = cache.out if out is None else out[n - 1]
    return cache.out if out is None else out


def decode_step_launch(cache: CompressedCache, q, k, v, new_classes, out, parity: int, pos_dev):
    """Launch one decode step whose insert position is read from the device
    (int32 ``pos_dev``) and whose live-count buffers are those of ``parity``,
    without touching the host bookkeeping: the building block of a captured
    CUDA graph that is replayed for successive steps.  The caller advances
    ``pos_dev`` and, per replay, calls ``advance_host_state``."""
    a = cache._dargs
    a.pos = cache.prompt_len
    a.q_dev, a.k_dev, a.v_dev = _ptr(q), _ptr(k), _ptr(v)
    a.bh_stride = q.stride(1)
    a.new_cls_dev = _ptr(new_classes)
    a.live_in_dev = _ptr(cache.live_buf[parity])
    a.live_out_dev = _ptr(cache.live_buf[parity ^ 1])
    a.out_dev = _ptr(out)
    a.pos_dev = _ptr(pos_dev)
    a.flags = 0
    if cache.track_recovery:
        _launch_recovery(cache, q, k, new_classes, cache.live_buf[parity], pos_dev=pos_dev)
    check(lib.akv_decode_step(C.byref(a), _stream()), EngineError)
    cache._latest_out = out
    return out


def advance_host_state(cache: CompressedCache):
    """Host bookkeeping of one replayed decode step (see decode_step_launch);
    the caller has checked the capacity before the replay."""
    cache._parity ^= 1
    cache.seq_len += 1


# ---------------------------------------------------------------------------
# reference-protocol drop-ins (engine.py:203-502)

@dataclass
class StepRecord:
    step: int
    token_id: int
    head_retained: dict
    total_cache_tokens: int
    mean_recovery: float | None
    retained_positions: dict | None = None


@dataclass
class GenerationResult:
    tokens: list
    profile: HeadProfile
    records: list
    cache: CompressedCache


def _model_rows(model, grid, positions, klass_of, prompt_len):
    d = model.config.head_dim
    G, n = len(grid), len(positions)
    q = np.empty((1, G, n, d), dtype=np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    for gi, (layer, head) in enumerate(grid):
        for i, pos in enumerate(positions):
            k[0, gi, i] = model.k_row(layer, head, pos, klass_of(pos), prompt_len)
            v[0, gi, i] = model.v_row(layer, head, pos)
            q[0, gi, i] = model.q_row(layer, head, pos, prompt_len)
    return q, k, v


def encode_model_rows(model, tokens, profiler_cfg: ProfilerConfig | None,
                      fixed_policy: CompressionPolicy | None = None, *, prompt_len=None,
                      max_new_tokens: int = 0, diagnostics: bool = False,
                      extra_thresholds=()):
    """The GPU counterpart of prompt_head_data + profiling (engine.py:161-200):
    gather every head's rows for ``tokens`` from the duck-typed model (rows
    anchored to ``prompt_len``, default len(tokens), which also anchors the
    local budget), then profile (K1) and compact (K2).  Returns
    (ProfileResult, CompressedCache, sorted grid, annotations)."""
    tokens = list(tokens)
    if not tokens:
        raise EngineError("empty prompt")
    n = len(tokens)
    p = n if prompt_len is None else int(prompt_len)
    if not 1 <= p <= n:
        raise EngineError(f"prompt_len {p} out of range for {n} tokens")
    grid = sorted(model.config.head_grid())
    annotations = classify_tokens(tokens, model.vocab)
    q, k, v = _model_rows(model, grid, range(n), lambda i: annotations[i].klass, p)
    dev = torch.device("cuda")
    cls = torch.tensor([[CLASS_CODE[a.klass] for a in annotations]], dtype=torch.uint8)
    res, cache = encode_prompt_tensors(
        torch.from_numpy(q).to(dev), torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev),
        cls.to(dev), profiler_cfg, fixed_policy, max_new_tokens=max_new_tokens,
        diagnostics=diagnostics, local_len=p if p != n else 0,
        extra_thresholds=extra_thresholds)
    return res, cache, grid, annotations


def profile_of(res: ProfileResult, grid, t: int = 0) -> HeadProfile:
    """HeadProfile (profiler.py:181-228) of threshold column ``t`` of a
    ProfileResult whose heads are ``grid`` in order."""
    decisions = {}
    for gi, key in enumerate(grid):
        c = int(res.choice[gi, t])
        decisions[key] = HeadDecision(res.family[c], float(res.recovery[gi, c]),
                                      int(res.cost[gi, c]))
    return HeadProfile(decisions)


def encode_prompt(model, prompt_tokens, profiler_cfg: ProfilerConfig | None,
                  fixed_policy: CompressionPolicy | None = None, threads=None,
                  diagnostics: bool = True, max_new_tokens: int = 256):
    """Drop-in for engine.py:203-272 over the duck-typed model protocol.

    Rows are gathered from the model (float64 -> float32) into one [1, G, n,
    d] batch whose heads are the model's sorted (layer, head) grid, then
    profiled and compacted on the GPU.  ``threads`` is accepted for API
    compatibility (the GPU processes all heads at once).
    """
    if profiler_cfg is None and fixed_policy is None:
        raise EngineError("need a profiler config or a fixed policy")
    res, cache, grid, annotations = encode_model_rows(
        model, prompt_tokens, profiler_cfg, fixed_policy, max_new_tokens=max_new_tokens,
        diagnostics=diagnostics)
    dev = cache.device
    profile = profile_of(res, grid)
    cache.profile = profile
    cache.keys = grid
    cache.annotations = list(annotations)
    cache.diagnostics = diagnostics
    cache._model_new_cls = torch.empty(1, dtype=torch.uint8, device=dev)
    return profile, cache


def _check_cache(model, cache: CompressedCache):
    expected = set(model.config.head_grid())
    if set(cache.keys) != expected or (cache.profile is not None and
                                       set(cache.profile.decisions) != expected):
        raise EngineError("cache/profile mismatch: head grid does not match the model")


def generate_step(model, cache: CompressedCache, last_token=None, sampler=None):
    """Drop-in for engine.py:283-371: insert ``last_token`` (if given) into
    every head's cache on the GPU, then sample the next token from
    ``model.head_logits`` over the concatenated head outputs."""
    _check_cache(model, cache)
    if not isinstance(sampler, _Sampler):
        sampler = _Sampler(sampler if sampler is not None else GreedyArgmax())
    if last_token is not None:
        pos = cache.seq_len
        klass = model.vocab.classify_id(last_token)
        cache.annotations.append(TokenAnnotation(pos, int(last_token), klass))
        q, k, v = _model_rows(model, cache.keys, [pos], lambda p: klass, cache.prompt_len)
        dev = cache.device
        qd = torch.from_numpy(q[:, :, 0]).to(dev)
        kd = torch.from_numpy(k[:, :, 0]).to(dev)
        vd = torch.from_numpy(v[:, :, 0]).to(dev)
        cache._model_new_cls.fill_(CLASS_CODE[klass])
        if cache.seq_len - cache.prompt_len >= cache.capacity_steps:
            # the reference's cache is unbounded: double the decode room
            grow_cache(cache, max(cache.capacity_steps, 16))
        decode_step_tensors(cache, qd.to(cache.dtype), kd.to(cache.dtype), vd.to(cache.dtype),
                            cache._model_new_cls)
    concat = cache.pending_output.reshape(-1).double().cpu().numpy()
    next_token = sampler(model.head_logits(concat))
    live = cache.head_retained()
    cache.last_record = StepRecord(
        step=0, token_id=next_token,
        head_retained={key: int(live[i]) for i, key in enumerate(cache.keys)},
        total_cache_tokens=int(live.sum()),
        mean_recovery=(float(cache.step_recovery.mean().item()) if cache.diagnostics else None),
        retained_positions=(
            {key: tuple(int(x) for x in p)
             for key, p in zip(cache.keys, cache.retained_positions())}
            if cache.diagnostics else None))
    return next_token, cache


def _run_decode(model, cache, profile, gen_cfg):
    sampler = _Sampler(gen_cfg.sampling)
    tokens, records, last = [], [], None
    for step in range(1, gen_cfg.max_new_tokens + 1):
        tok, cache = generate_step(model, cache, last, sampler)
        rec = cache.last_record
        rec.step = step
        tokens.append(tok)
        records.append(rec)
        last = tok
    return GenerationResult(tokens, profile, records, cache)


def generate(model, prompt_tokens, profiler_cfg: ProfilerConfig, gen_cfg: GenerationConfig,
             threads=None, diagnostics: bool = True) -> GenerationResult:
    """Encode once, then ``max_new_tokens`` decoding steps (engine.py:382-394)."""
    profile, cache = encode_prompt(model, prompt_tokens, profiler_cfg, threads=threads,
                                   diagnostics=diagnostics,
                                   max_new_tokens=max(1, gen_cfg.max_new_tokens))
    return _run_decode(model, cache, profile, gen_cfg)


def generate_fixed_baseline(model, prompt_tokens, policy: CompressionPolicy,
                            gen_cfg: GenerationConfig, diagnostics: bool = True):
    """One imposed policy on every head, no profiling (engine.py:397-408)."""
    profile, cache = encode_prompt(model, prompt_tokens, None, fixed_policy=policy,
                                   diagnostics=diagnostics,
                                   max_new_tokens=max(1, gen_cfg.max_new_tokens))
    return _run_decode(model, cache, profile, gen_cfg)


def reference_generate(model, prompt_tokens, gen_cfg: GenerationConfig) -> GenerationResult:
    """Uncompressed baseline (engine.py:428-502): the full policy on every
    head through the same kernels (no eviction ever happens)."""
    res = generate_fixed_baseline(model, prompt_tokens, full_policy(), gen_cfg, diagnostics=False)
    for rec in res.records:
        rec.mean_recovery = 1.0
    return GenerationResult(res.tokens, HeadProfile({}), res.records, res.cache)


def records_to_ndjson(records, num_layers: int, num_heads: int) -> str:
    """One JSON object per step, retained counts in layer-major order
    (engine.py:505-525)."""
    lines = []
    for rec in records:
        grid = [[rec.head_retained[(layer, head)] for head in range(num_heads)]
                for layer in range(num_layers)]
        lines.append(json.dumps({"step": rec.step, "token_id": rec.token_id,
                                 "head_retained": grid,
                                 "total_cache_tokens": rec.total_cache_tokens,
                                 "mean_recovery": rec.mean_recovery}, sort_keys=True))
    return "\n".join(lines) + ("\n" if lines else "")
