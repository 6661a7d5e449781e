"""Run the CUDA path (through the package's tensor API, i.e. the C-ABI) on a
golden case and collect results in the golden layout."""

from __future__ import annotations

import numpy as np
import torch

import cases as C
from helpers import NAME_BIT, parse_fixed
from paper_2310_01801_b200 import (CompressionPolicy, ProfilerConfig, RowAveraging,
                                   SelectionCriterion, decode_step_tensors, encode_prompt_tensors,
                                   feasible_set, parse_policy)
from paper_2310_01801_b200.policies import PolicyAtom
from paper_2310_01801_b200.workloads import class_lut

ATOM_NAME = {"special": PolicyAtom.SPECIAL, "punct": PolicyAtom.PUNCTUATION,
             "frequent": PolicyAtom.FREQUENT, "local": PolicyAtom.LOCAL}


def case_config(w, opts, T):
    order = [ATOM_NAME[a] for a in opts.get("order", C.ORDER_DEFAULT)]
    drop = [ATOM_NAME[a] for a in opts.get("drop", ())]
    fam = feasible_set(r_l=w.r_l, r_f=w.r_f, atom_order=order, drop=drop)
    return ProfilerConfig(recovery_threshold=T, feasible=fam,
                          criterion=SelectionCriterion(opts.get("criterion", "recovery")),
                          rows=RowAveraging(opts.get("rows", "all")))


def torch_dtype(w):
    return torch.bfloat16 if w.dtype == "bf16" else torch.float32


def run_arrays(q, k, v, cls, N, D, slopes, sinks, cfg=None, fixed=None, extra=(),
               dtype=torch.float32, record_steps=True, pool=None):
    """q,k,v numpy float [B,H,T,d] (values exactly representable in dtype),
    cls uint8 [B,T].  Returns a dict in the golden layout."""
    dev = torch.device("cuda")
    B, H, T, d = q.shape
    qt = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float32)).to(dev).to(dtype)
    kt = torch.from_numpy(np.ascontiguousarray(k, dtype=np.float32)).to(dev).to(dtype)
    vt = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(dev).to(dtype)
    ct = torch.from_numpy(np.ascontiguousarray(cls, dtype=np.uint8)).to(dev)
    sl = None if slopes is None else torch.tensor(slopes, dtype=torch.float32, device=dev)
    sk = None if sinks is None else torch.tensor(sinks, dtype=torch.float32, device=dev)
    res, cache = encode_prompt_tensors(qt, kt, vt, ct, cfg, fixed, prompt_len=N,
                                       max_new_tokens=D, extra_thresholds=extra, slopes=sl,
                                       sinks=sk, diagnostics=True, pool=pool)
    G = B * H
    out = dict(res=res, cache=cache)
    enc_kept = np.zeros((G, N), bool)
    for g, pos in enumerate(cache.retained_positions()):
        enc_kept[g, pos] = True
    out["enc_kept"] = enc_kept
    out["enc_out"] = cache.out.reshape(G, d).cpu().numpy().astype(np.float64)
    out["colsum"] = cache.colsum.cpu().numpy()
    out["lastrow"] = cache.lastp.cpu().numpy().astype(np.float64)
    dec_kept = np.zeros((D, G, N + D), bool)
    dec_out = np.zeros((D, G, d))
    dec_rec = np.zeros((D + 1, G))
    dec_rec[0] = cache.step_recovery.cpu().numpy()
    cls_cols = [ct[:, N + t].contiguous() for t in range(D)]
    for t in range(D):
        pos = N + t
        o = decode_step_tensors(cache, qt[:, :, pos], kt[:, :, pos], vt[:, :, pos],
                                cls_cols[t], chained=True)
        if record_steps:
            dec_out[t] = o.reshape(G, d).cpu().numpy()
            dec_rec[t + 1] = cache.step_recovery.cpu().numpy()
            for g, p in enumerate(cache.retained_positions()):
                dec_kept[t, g, p] = True
    torch.cuda.synchronize()
    cache.check()
    out["dec_kept"] = dec_kept
    out["dec_out"] = dec_out
    out["dec_rec"] = dec_rec
    return out


def run_case(name, pool=None):
    """CUDA path on a workload golden case, heads in golden order."""
    w, opts = C.case_workload(name)
    heads = C.case_heads(w, opts)
    bs = sorted({b for b, _ in heads})
    hs = sorted({h for _, h in heads})
    assert [(b, h) for b in bs for h in hs] == heads
    lut = class_lut()
    T = w.total_len
    q = np.zeros((len(bs), len(hs), T, w.d), np.float32)
    k = np.zeros_like(q)
    v = np.zeros_like(q)
    cls = np.zeros((len(bs), T), np.uint8)
    for i, b in enumerate(bs):
        cls[i] = lut[w.tokens(b)]
        for j, h in enumerate(hs):
            q[i, j], k[i, j], v[i, j] = w.head_qkv(b, h)
    dec_T = opts.get("decode_T", w.thresholds[0])
    if "fixed" in opts:
        cfg, fixed, extra = None, parse_policy(opts["fixed"]), ()
    else:
        cfg, fixed, extra = case_config(w, opts, dec_T), None, tuple(w.thresholds)
    return run_arrays(q, k, v, cls, w.N, w.D, w.slopes[hs], w.sinks[hs], cfg, fixed, extra,
                      torch_dtype(w), pool=pool)
