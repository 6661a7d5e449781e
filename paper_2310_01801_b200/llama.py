"""Multi-layer caller of the adaptive-KV path: a random-init Llama decoder
whose every layer profiles, compacts and decodes through K1/K2/K3
(BASELINE.json configs 2 and 3).

The reference's engine consumes per-(layer, head) q/k/v rows from a model
object (model.py:219-286) and hands the concatenated head outputs to a
linear head (engine.py:354-357).  Here the model is a Llama stack (RMSNorm,
RoPE, SwiGLU; weights ~N(0, 0.02), seeded) whose projections are cuBLAS
GEMMs and whose glue is the caller kernels of ``csrc/akv_caller.cu``:

prefill, per layer  add_rmsnorm -> QKV GEMM -> rope_scatter (head-major
                    [B, Hl, N, d]) -> causal attention outputs of every
                    prompt row (library SDPA; FastGen does not compress the
                    prefill) -> K1 profile + K2 compaction into this layer's
                    ragged arena -> O GEMM -> add_rmsnorm -> gate|up GEMM ->
                    swiglu -> down GEMM
decode, per layer   the same with one row per sequence and K3 (insert ->
                    attend -> score update -> evict) in place of attention
                    + profiling; the next token is chosen on the device
                    (``akv_greedy_next``: argmax, class lookup, embedding),
                    so a decode step never waits on the host.

Sharding (one process per GPU, ``torch.distributed`` over NCCL):

* ``gather`` (config 2): heads are split into contiguous blocks, the QKV
  projection is column-sliced to the local heads, everything else is
  replicated; the attention outputs [rows, Hl*d] are all-gathered (the
  cross-shard gather of BASELINE's north star) before the O projection.
* ``tp`` (config 3, whose weights do not fit one GPU replicated): Megatron
  tensor parallelism - QKV and gate|up column-sliced, O and down
  row-sliced, each followed by an all-reduce of the partial sums.
* batch rows are independent sessions: data-parallel ranks simply run the
  model on their own rows (world 1 from the model's point of view).

Weights are generated per full matrix from a seeded CUDA generator and then
sliced, so any sharding of one seed describes the same network.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import DTYPE_BF16, DTYPE_F32, RopeArgs, check, lib
from .engine import (EngineError, advance_host_state, decode_step_launch, decode_step_tensors,
                     encode_prompt_tensors)
from .parallel import all_reduce_partial, gather_head_blocks, shard_layer_weights
from .profiler import ProfilerConfig
from .workloads import PUNCT_IDS, SPECIAL_IDS, class_lut


@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int
    d_model: int
    n_heads: int
    ffn: int
    vocab: int = 32000
    rope_theta: float = 10000.0
    eps: float = 1e-5
    init_std: float = 0.02

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


LLAMA_7B = LlamaConfig(n_layers=32, d_model=4096, n_heads=32, ffn=11008)
LLAMA_65B = LlamaConfig(n_layers=80, d_model=8192, n_heads=64, ffn=22016)


@dataclass(frozen=True)
class ShardPlan:
    """Which heads / FFN columns this rank owns (``mode``: gather | tp)."""

    rank: int = 0
    world: int = 1
    mode: str = "gather"
    # False: this process computes rank `rank`'s shard but issues no
    # collective (single-GPU measurement of one rank's compute; the outputs
    # are then not those of the full model)
    comm: bool = True

    def heads(self, H: int) -> tuple:
        if H % self.world:
            raise EngineError(f"{H} heads do not split evenly over {self.world} ranks")
        n = H // self.world
        return self.rank * n, (self.rank + 1) * n

    def ffn(self, F: int) -> tuple:
        if self.mode != "tp":
            return 0, F
        if F % self.world:
            raise EngineError(f"ffn {F} does not split evenly over {self.world} ranks")
        n = F // self.world
        return self.rank * n, (self.rank + 1) * n


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(dtype) -> int:
    if dtype == torch.float32:
        return DTYPE_F32
    if dtype == torch.bfloat16:
        return DTYPE_BF16
    raise EngineError(f"unsupported dtype {dtype}")


@dataclass
class _Layer:
    attn_norm: torch.Tensor
    wqkv: torch.Tensor      # [3*Hl*d, dm]: q heads | k heads | v heads
    wo: torch.Tensor        # gather: [dm, H*d]; tp: [dm, Hl*d]
    mlp_norm: torch.Tensor
    wgu: torch.Tensor       # [2*Fl, dm]: gate | up
    wdown: torch.Tensor     # [dm, Fl]


@dataclass
class _PeerPartials:
    """Pending tensor-parallel reduction: slot of the symmetric buffers that
    hold every rank's partial product (consumed by _rmsnorm)."""
    slot: int


@dataclass
class PrefillResult:
    profiles: list                     # per layer: ProfileResult (local heads)
    next_tokens: torch.Tensor          # [B] int64 (device)
    events: list = field(default_factory=list)  # per layer (start, end) CUDA events of K1+K2

    def profiling_ms(self) -> list:
        """Per-layer profile + compaction time (ms); synchronises."""
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in self.events]


class FastGenLlama:
    """Random-init Llama decoder over the FastGen compressed KV cache.

    ``prefill(tokens, profiler_cfg, max_new_tokens)`` profiles every layer's
    heads on the prompt and builds the per-layer compressed caches;
    ``decode_step()`` generates one token per sequence (greedy) through K3.
    """

    def __init__(self, cfg: LlamaConfig, *, dtype=torch.bfloat16, device=None, seed: int = 0,
                 plan: ShardPlan | None = None, group=None, max_positions: int = 8192,
                 special_ids=SPECIAL_IDS, punct_ids=PUNCT_IDS):
        _lib.require_device()
        self.cfg = cfg
        self.dtype = dtype
        self.dt = _dt(dtype)
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.plan = plan or ShardPlan()
        self.group = group
        d = cfg.head_dim
        if d * cfg.n_heads != cfg.d_model:
            raise EngineError("d_model must be n_heads * head_dim")
        self.h0, self.h1 = self.plan.heads(cfg.n_heads)
        self.Hl = self.h1 - self.h0
        self.f0, self.f1 = self.plan.ffn(cfg.ffn)
        self.Fl = self.f1 - self.f0
        self.max_positions = max_positions
        self.lut = torch.from_numpy(class_lut(cfg.vocab, special_ids, punct_ids)).to(self.device)
        self._rope_tables(max_positions)
        self._init_weights(seed)
        self.caches: list = []
        self.record = False
        self.use_graphs = True
        self._graphs = None
        self._ar_bufs = None      # tensor-parallel decode reduction buffers (_setup_tp_reduce)
        self.pos_dev = None
        self.trace: dict = {}

    # -- weights ------------------------------------------------------------
    def _randn(self, gen, rows, cols):
        w = torch.empty(rows, cols, dtype=torch.float32, device=self.device)
        w.normal_(0.0, self.cfg.init_std, generator=gen)
        return w.to(self.dtype)

    def _init_weights(self, seed: int):
        cfg, dm, d = self.cfg, self.cfg.d_model, self.cfg.head_dim
        gen = torch.Generator(device=self.device)
        ones = torch.ones(dm, dtype=self.dtype, device=self.device)
        self.layers = []
        for layer in range(cfg.n_layers):
            mats = {}
            for i, (name, rows, cols) in enumerate(
                    [("wq", dm, dm), ("wk", dm, dm), ("wv", dm, dm), ("wo", dm, dm),
                     ("wg", cfg.ffn, dm), ("wu", cfg.ffn, dm), ("wd", dm, cfg.ffn)]):
                gen.manual_seed((seed * 100003 + layer) * 16 + i)
                mats[name] = self._randn(gen, rows, cols)
            wqkv, wo, wgu, wdown = shard_layer_weights(mats, self.h0, self.h1, d, self.f0,
                                                       self.f1, self.plan.mode)
            del mats
            self.layers.append(_Layer(ones.clone(), wqkv, wo, ones.clone(), wgu, wdown))
        gen.manual_seed(seed * 100003 + 99991)
        self.embed = self._randn(gen, cfg.vocab, dm)
        gen.manual_seed(seed * 100003 + 99989)
        self.lm_head = self._randn(gen, cfg.vocab, dm)
        self.final_norm = ones.clone()

    def _rope_tables(self, max_pos: int):
        d = self.cfg.head_dim
        inv = self.cfg.rope_theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
        ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = torch.from_numpy(np.cos(ang).astype(np.float32)).to(self.device)
        self.sin = torch.from_numpy(np.sin(ang).astype(np.float32)).to(self.device)

    # -- caller kernels -----------------------------------------------------
    def _rmsnorm(self, residual, w, x=None, out=None):
        rows, dim = residual.shape
        out = torch.empty_like(residual) if out is None else out
        if isinstance(x, _PeerPartials):   # tensor-parallel reduction fused into the norm
            ptrs = self._ar_ptrs[x.slot]
            check(lib.akv_add_rmsnorm_peers(rows, dim, self.dt, _ptr(ptrs), ptrs.numel(),
                                            self._ar_bufs[x.slot].stride(0), _ptr(residual),
                                            _ptr(w), self.cfg.eps, _ptr(out), _stream()),
                  EngineError)
            return out
        check(lib.akv_add_rmsnorm(rows, dim, self.dt, _ptr(x), _ptr(residual), _ptr(w),
                                  self.cfg.eps, _ptr(out), _stream()), EngineError)
        return out

    def _rope(self, qkv, n, pos0, q, k, v, out_ld, pos_dev=None):
        a = RopeArgs()
        a.T, a.n, a.Hl, a.d, a.dtype = qkv.shape[0], n, self.Hl, self.cfg.head_dim, self.dt
        a.qkv_dev, a.qkv_ld = _ptr(qkv), qkv.stride(0)
        a.pos0, a.max_pos = pos0, self.max_positions
        a.cos_dev, a.sin_dev = _ptr(self.cos), _ptr(self.sin)
        a.q_dev, a.k_dev, a.v_dev = _ptr(q), _ptr(k), _ptr(v)
        a.out_ld, a.row0 = out_ld, 0
        a.pos_dev = _ptr(pos_dev)
        check(lib.akv_rope_scatter(C.byref(a), _stream()), EngineError)

    def _swiglu(self, gu):
        rows = gu.shape[0]
        out = torch.empty(rows, self.Fl, dtype=self.dtype, device=self.device)
        check(lib.akv_swiglu(rows, self.Fl, self.dt, _ptr(gu), _ptr(out), _stream()), EngineError)
        return out

    def _greedy(self, logits):
        B = logits.shape[0]
        check(lib.akv_greedy_next(B, self.cfg.vocab, self.dt, _ptr(logits), logits.stride(0),
                                  _ptr(self.lut), _ptr(self.embed), self.cfg.d_model,
                                  _ptr(self.next_tok), _ptr(self.next_cls), _ptr(self.x_next),
                                  _stream()), EngineError)

    # -- collectives --------------------------------------------------------
    def _setup_decode_gather(self, B):
        """Decode-time attention outputs go straight from K3's combine into
        the O projection's input [B, width] (cache dtype): the local buffer,
        or - head-sharded over ranks (gather mode) - every rank's
        symmetric-memory buffer at this rank's column block, followed by a
        device-side barrier (the cross-shard gather fused into the decode
        kernel; no NCCL call and no cast on the decode path).  Two buffers
        alternate between layers so one barrier per layer suffices."""
        d = self.cfg.head_dim
        sharded = self.plan.mode == "gather" and self.plan.world > 1
        width = (self.plan.world * self.Hl * d) if sharded else self.Hl * d
        col0 = self.plan.rank * self.Hl * d if sharded else 0
        self._gather_hdl = [None, None]
        if sharded and self.plan.comm:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            group = self.group if self.group is not None else dist.group.WORLD
            bufs, ptrs = [], []
            for i in range(2):
                t = symm_mem.empty((B, width), dtype=self.dtype, device=self.device)
                hdl = symm_mem.rendezvous(t, group.group_name)
                bufs.append(t)
                ptrs.append(torch.tensor(list(hdl.buffer_ptrs), dtype=torch.int64,
                                         device=self.device))
                self._gather_hdl[i] = hdl
        else:
            bufs = [torch.zeros(B, width, dtype=self.dtype, device=self.device) for _ in range(2)]
            ptrs = [torch.tensor([t.data_ptr()], dtype=torch.int64, device=self.device) for t in bufs]
        self._gather_bufs, self._gather_ptrs = bufs, ptrs
        for li, c in enumerate(self.caches):
            a = c._dargs
            a.peer_out_dev = C.c_void_p(ptrs[li & 1].data_ptr())
            a.n_peers = ptrs[li & 1].numel()
            a.peer_ld, a.peer_col0 = width, col0

    def _decode_gathered(self, li):
        """The O projection's input of layer li after its decode step."""
        hdl = self._gather_hdl[li & 1]
        if hdl is not None:
            hdl.barrier(channel=li & 1)
        return self._gather_bufs[li & 1]

    def _gather_heads(self, o):
        """[rows, Hl*d] local head outputs -> [rows, H*d] (rank-ordered head
        blocks = global head order)."""
        if self.plan.mode == "tp":
            return o
        if not self.plan.comm:   # compute-only shard: the local block in place, zeros elsewhere
            full = torch.zeros(o.shape[0], self.plan.world * o.shape[1], dtype=o.dtype,
                               device=o.device)
            full[:, self.plan.rank * o.shape[1]:(self.plan.rank + 1) * o.shape[1]] = o
            return full
        return gather_head_blocks(o, self.plan.world, self.group)

    def _reduce(self, x):
        if self.plan.mode != "tp" or not self.plan.comm:
            return x
        return all_reduce_partial(x, self.plan.world, self.group)

    def _setup_tp_reduce(self, B, local=False):
        """Decode-time row-parallel reductions (tp mode) fused into the norm
        that consumes them: each rank's O / down projection writes its
        partial product into its own symmetric-memory buffer [B, dm] (two
        alternating, so one barrier per reduction also orders the reuse),
        a device-side barrier, then akv_add_rmsnorm_peers sums every rank's
        partial over NVLink loads (rank order: identical bits everywhere),
        adds the residual and normalises - no NCCL call on the decode path.
        ``local`` builds the same plumbing over this process's buffers only
        (world 1; tests)."""
        self._ar_bufs = None
        multi = self.plan.mode == "tp" and self.plan.comm and self.plan.world > 1
        if not (multi or local):
            return
        dm = self.cfg.d_model
        bufs, ptrs, hdls = [], [], []
        for i in range(2):
            if multi:
                import torch.distributed as dist
                import torch.distributed._symmetric_memory as symm_mem

                group = self.group if self.group is not None else dist.group.WORLD
                t = symm_mem.empty((B, dm), dtype=self.dtype, device=self.device)
                hdl = symm_mem.rendezvous(t, group.group_name)
                p = list(hdl.buffer_ptrs)
            else:
                t = torch.zeros(B, dm, dtype=self.dtype, device=self.device)
                hdl, p = None, [t.data_ptr()]
            bufs.append(t)
            hdls.append(hdl)
            ptrs.append(torch.tensor(p, dtype=torch.int64, device=self.device))
        self._ar_bufs, self._ar_ptrs, self._ar_hdls, self._ar_next = bufs, ptrs, hdls, 0

    def _reduce_linear(self, x, w):
        """x @ w.T summed over the tensor-parallel ranks: a _PeerPartials
        handle for the fused decode path, else the all-reduced tensor."""
        if self._ar_bufs is not None and x.shape[0] == self._ar_bufs[0].shape[0]:
            slot = self._ar_next
            self._ar_next ^= 1
            torch.matmul(x, w.t(), out=self._ar_bufs[slot])
            if self._ar_hdls[slot] is not None:
                self._ar_hdls[slot].barrier(channel=slot)
            return _PeerPartials(slot)
        return self._reduce(torch.nn.functional.linear(x, w))

    def _mlp(self, L, residual, attn_out):
        """residual += attn_out; MLP; returns (mlp delta)."""
        xn = self._rmsnorm(residual, L.mlp_norm, x=attn_out)
        gu = torch.nn.functional.linear(xn, L.wgu)
        return self._reduce_linear(self._swiglu(gu), L.wdown)

    # -- prefill ------------------------------------------------------------
    def prefill(self, tokens: torch.Tensor, profiler_cfg: ProfilerConfig | None = None,
                max_new_tokens: int = 0, fixed_policy=None, extra_thresholds=(),
                diagnostics: bool = False):
        """Run the prompt ``tokens`` [B, N] (int64, device) through every
        layer: full causal attention for the prompt rows, K1 profiling and
        K2 compaction of each layer's heads.  Returns a PrefillResult; the
        next token per sequence is left on the device for decode_step.
        ``diagnostics`` keeps every layer's shadow keys so that each decode
        step also reports its heads' recovery against uncompressed attention
        (``mean_recovery``; engine.py:341-349)."""
        cfg, d, dm = self.cfg, self.cfg.head_dim, self.cfg.d_model
        if tokens.dim() != 2 or not tokens.is_cuda:
            raise EngineError("tokens must be a CUDA tensor [B, N]")
        B, N = tokens.shape
        if N < 1:
            raise EngineError("empty prompt")
        if N + max_new_tokens > self.max_positions:
            raise EngineError(f"{N + max_new_tokens} positions exceed the RoPE table "
                              f"({self.max_positions})")
        if int(tokens.min()) < 0 or int(tokens.max()) >= cfg.vocab:
            raise EngineError("token id out of range")
        T = B * N
        tokens = tokens.contiguous()
        self.B, self.N, self.seq_len = B, N, N
        self.capacity = max_new_tokens
        residual = torch.empty(T, dm, dtype=self.dtype, device=self.device)
        cls = torch.empty(B, N + max_new_tokens, dtype=torch.uint8, device=self.device)
        check(lib.akv_embed_classify(T, _ptr(tokens), cfg.vocab, _ptr(self.lut), _ptr(self.embed),
                                     dm, self.dt, _ptr(residual), None, _stream()), EngineError)
        cls_prompt = torch.empty(B, N, dtype=torch.uint8, device=self.device)
        check(lib.akv_embed_classify(T, _ptr(tokens), cfg.vocab, _ptr(self.lut), None, dm, self.dt,
                                     None, _ptr(cls_prompt), _stream()), EngineError)
        cls[:, :N] = cls_prompt
        self.classes = cls
        q = torch.empty(B, self.Hl, N, d, dtype=self.dtype, device=self.device)
        k, v = torch.empty_like(q), torch.empty_like(q)
        self.caches, profiles, prof_events = [], [], []
        self._graphs = None
        self._ar_bufs = None      # prefill reduces through NCCL
        self.trace = {"prompt": [], "steps": []} if self.record else {}
        delta = None
        for li, L in enumerate(self.layers):
            xn = self._rmsnorm(residual, L.attn_norm, x=delta)
            qkv = torch.nn.functional.linear(xn, L.wqkv)
            self._rope(qkv, N, 0, q, k, v, N)
            if self.record:
                self.trace["prompt"].append((q.clone(), k.clone(), v.clone()))
            o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            res, cache = encode_prompt_tensors(
                q, k, v, cls_prompt, profiler_cfg, fixed_policy, prompt_len=N,
                max_new_tokens=max_new_tokens, extra_thresholds=extra_thresholds,
                diagnostics=diagnostics)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record()
            prof_events.append((ev0, ev1))
            self.caches.append(cache)
            profiles.append(res)
            o = self._gather_heads(o.transpose(1, 2).reshape(T, self.Hl * d))
            attn = self._reduce(torch.nn.functional.linear(o, L.wo))
            delta = self._mlp(L, residual, attn)
        last = residual.view(B, N, dm)[:, N - 1]
        dl = delta.view(B, N, dm)[:, N - 1]
        r_last = last.contiguous()
        xf = self._rmsnorm(r_last, self.final_norm, x=dl.contiguous())
        logits = torch.nn.functional.linear(xf, self.lm_head)
        self.next_tok = torch.empty(B, dtype=torch.int64, device=self.device)
        self.next_cls = torch.empty(B, dtype=torch.uint8, device=self.device)
        self.x_next = torch.empty(B, dm, dtype=self.dtype, device=self.device)
        self._greedy(logits)
        self.last_logits = logits
        self.q1 = torch.empty(B, self.Hl, d, dtype=self.dtype, device=self.device)
        self.k1, self.v1 = torch.empty_like(self.q1), torch.empty_like(self.q1)
        self.o_dec = torch.empty(len(self.layers), B, self.Hl, d, dtype=torch.float32,
                                 device=self.device)
        self._setup_decode_gather(B)
        self._setup_tp_reduce(B)
        out = PrefillResult(profiles, self.next_tok)
        out.events = prof_events
        return out

    # -- decode -------------------------------------------------------------
    def decode_step(self) -> torch.Tensor:
        """Insert the pending token of every sequence into every layer's
        compressed cache and produce the next one (greedy).  Returns the
        inserted tokens [B] (device, int64; a copy).

        Unless ``record`` is set or ``use_graphs`` is off, the first step
        runs eagerly and captures the whole step (every layer's kernels and
        GEMMs) into two CUDA graphs - one per parity of the double-buffered
        live counts - whose K3 and RoPE launches read the insert position
        from the device; later steps are graph replays."""
        if not self.caches:
            raise EngineError("decode_step before prefill")
        if self.seq_len - self.N >= self.capacity:
            raise EngineError(f"cache capacity of {self.capacity} decode steps exhausted")
        if self.record or not self.use_graphs:
            return self._step_eager()
        if self._graphs is None:
            out = self._step_eager()
            self._capture()
            return out
        parity = self.caches[0]._parity
        self._graphs[parity].replay()
        self.last_logits = self._graph_logits[parity]
        for c in self.caches:
            advance_host_state(c)
        self.seq_len += 1
        return self.ins_buf.clone()

    def _layers_step(self, residual, new_cls, pos=None, parity=None, rec=None):
        """Every layer of one decode step; host ``pos`` (eager, through
        decode_step_tensors) or the device position (graph capture)."""
        d, B = self.cfg.head_dim, self.B
        delta = None
        for li, L in enumerate(self.layers):
            xn = self._rmsnorm(residual, L.attn_norm, x=delta)
            qkv = torch.nn.functional.linear(xn, L.wqkv)
            if pos is None:
                self._rope(qkv, 1, 0, self.q1, self.k1, self.v1, 1, pos_dev=self.pos_dev)
                o = decode_step_launch(self.caches[li], self.q1, self.k1, self.v1, new_cls,
                                       self.o_dec[li], parity, self.pos_dev)
            else:
                self._rope(qkv, 1, pos, self.q1, self.k1, self.v1, 1)
                if rec is not None:
                    rec.append((self.q1.clone(), self.k1.clone(), self.v1.clone()))
                o = decode_step_tensors(self.caches[li], self.q1, self.k1, self.v1, new_cls,
                                        out=self.o_dec[li])
            attn = self._reduce_linear(self._decode_gathered(li), L.wo)
            delta = self._mlp(L, residual, attn)
        xf = self._rmsnorm(residual, self.final_norm, x=delta)
        logits = torch.nn.functional.linear(xf, self.lm_head)
        self._greedy(logits)
        self.last_logits = logits

    def _step_eager(self) -> torch.Tensor:
        pos = self.seq_len
        inserted = self.next_tok.clone()
        new_cls = self.next_cls.clone()
        self.classes[:, pos] = new_cls
        rec = [] if self.record else None
        self._layers_step(self.x_next.clone(), new_cls, pos=pos, rec=rec)
        if rec is not None:
            self.trace["steps"].append((rec, new_cls.clone(), self.o_dec.clone()))
        self.seq_len += 1
        return inserted

    def _capture(self):
        """Capture one decode step per live-count parity (see decode_step).
        The graph snapshots the pending token / class / embedding row, runs
        every layer, picks the next token and advances the device position."""
        self.pos_dev = torch.full((1,), self.seq_len, dtype=torch.int32, device=self.device)
        # every buffer a captured graph touches must outlive the graphs
        self.ins_buf = torch.empty_like(self.next_tok)
        cls_buf = self._g_cls = torch.empty_like(self.next_cls)
        res_buf = self._g_res = torch.empty_like(self.x_next)
        col = self._g_col = torch.empty(1, dtype=torch.int64, device=self.device)
        parity0 = self.caches[0]._parity
        if any(c._parity != parity0 for c in self.caches):
            raise EngineError("layer caches out of step")
        torch.cuda.synchronize()
        graphs, self._graph_logits = {}, {}
        eager_logits = self.last_logits
        pool = None
        for parity in (parity0, parity0 ^ 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool):
                self.ins_buf.copy_(self.next_tok)
                cls_buf.copy_(self.next_cls)
                res_buf.copy_(self.x_next)
                col.copy_(self.pos_dev)
                self.classes.index_copy_(1, col, cls_buf[:, None])
                self._layers_step(res_buf, cls_buf, parity=parity)
                self.pos_dev.add_(1)
            pool = g.pool()
            graphs[parity] = g
            self._graph_logits[parity] = self.last_logits
        self.last_logits = eager_logits
        self._graphs = graphs

    def generate(self, tokens, profiler_cfg=None, max_new_tokens: int = 16, fixed_policy=None):
        """Prefill then ``max_new_tokens`` greedy tokens; returns [B, D]
        (device int64): the tokens sampled after the prompt, in order."""
        self.prefill(tokens, profiler_cfg, max_new_tokens, fixed_policy)
        out = torch.empty(self.B, max_new_tokens, dtype=torch.int64, device=self.device)
        for t in range(max_new_tokens):
            out[:, t] = self.decode_step()
        return out

    def mean_recovery(self) -> float:
        """Mean over layers and heads of the latest step's recovery (the
        reference's StepRecord.mean_recovery); needs prefill(diagnostics=True)."""
        if not self.caches or not self.caches[0].track_recovery:
            raise EngineError("mean_recovery needs prefill(..., diagnostics=True)")
        return float(torch.stack([c.step_recovery for c in self.caches]).mean())

    def check(self):
        for c in self.caches:
            c.check()

    def cache_tokens(self) -> int:
        return int(sum(int(c.live.sum()) for c in self.caches))
