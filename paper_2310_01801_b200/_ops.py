"""Device helpers behind the single-context API functions (attention.py,
policies.py, profiler.py mirrors): numpy in, numpy out, every computation
in a libakv kernel (float64)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import KeepArgs, check, lib


def _dev():
    _lib.require_device()
    return torch.device("cuda")


def to_dev(x, dtype=torch.float64):
    a = np.ascontiguousarray(x)
    if not a.flags.writeable:
        a = a.copy()
    return torch.as_tensor(a).to(device=_dev(), dtype=dtype)


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def softmax_rows(m: np.ndarray, lengths=None, exc=None) -> np.ndarray:
    x = to_dev(m)
    out = torch.empty_like(x)
    ln = None if lengths is None else to_dev(np.asarray(lengths, dtype=np.int32), torch.int32)
    check(lib.akv_softmax_rows_f64(x.shape[0], x.shape[1], ptr(x), ptr(ln), ptr(out), stream()), exc)
    return out.cpu().numpy()


def causal_attention(q, k, v, scale, exc=None):
    qd, kd, vd = to_dev(q), to_dev(k), to_dev(v)
    n = qd.shape[0]
    A = torch.empty(n, n, dtype=torch.float64, device=qd.device)
    O = torch.empty(n, vd.shape[1], dtype=torch.float64, device=qd.device)
    check(lib.akv_causal_attention_f64(n, qd.shape[1], vd.shape[1], ptr(qd), ptr(kd), ptr(vd),
                                       float(scale), ptr(A), ptr(O), stream()), exc)
    return A.cpu().numpy(), O.cpu().numpy()


def keep_masks(items, exc=None):
    """items: list of dicts with keys cls (uint8 [L]), scores (float64 [L]),
    cand (bool [L] or None), prompt_len, current_len, atoms, r_l, r_f.
    Returns (keep bool [G, stride], counts int [G])."""
    G = len(items)
    stride = max(1, max(it["current_len"] for it in items))
    cls = np.zeros((G, stride), np.uint8)
    sc = np.zeros((G, stride), np.float64)
    cand = np.zeros((G, stride), np.uint8)
    any_cand = any(it["cand"] is not None for it in items)
    for g, it in enumerate(items):
        L = it["current_len"]
        cls[g, :L] = it["cls"][:L]
        sc[g, :L] = it["scores"][:L]
        cand[g, :L] = 1 if it["cand"] is None else it["cand"][:L]
    dev = _dev()
    t = lambda x, dt: torch.as_tensor(x).to(device=dev, dtype=dt)
    plen = t(np.array([it["prompt_len"] for it in items], np.int32), torch.int32)
    clen = t(np.array([it["current_len"] for it in items], np.int32), torch.int32)
    atoms = t(np.array([it["atoms"] for it in items], np.uint8), torch.uint8)
    rl = t(np.array([it["r_l"] for it in items], np.float64), torch.float64)
    rf = t(np.array([it["r_f"] for it in items], np.float64), torch.float64)
    clsd, scd = t(cls, torch.uint8), t(sc, torch.float64)
    candd = t(cand, torch.uint8) if any_cand else None
    keep = torch.empty(G, stride, dtype=torch.uint8, device=dev)
    cnt = torch.empty(G, dtype=torch.int32, device=dev)
    scratch = torch.empty(G, stride, dtype=torch.int32, device=dev)
    a = KeepArgs(G, stride, ptr(plen), ptr(clen), ptr(clsd), ptr(scd), ptr(candd), ptr(atoms),
                 ptr(rl), ptr(rf), ptr(keep), ptr(cnt), ptr(scratch))
    check(lib.akv_keep_mask(C.byref(a), stream()), exc)
    return keep.cpu().numpy().astype(bool), cnt.cpu().numpy().astype(np.int64)


def map_recovery(maps: np.ndarray, masks: np.ndarray, rows: int, exc=None):
    """maps [G, n, n] float64, masks [G, F, n] bool -> (recovery [G, F], cosine [G, F])."""
    A = to_dev(maps)
    G, n, _ = A.shape
    F = masks.shape[1]
    m = to_dev(masks.astype(np.uint8), torch.uint8)
    ws1 = torch.empty(G, n, dtype=torch.float64, device=A.device)
    ws2 = torch.empty_like(ws1)
    rec = torch.empty(G, F, dtype=torch.float64, device=A.device)
    cos = torch.empty_like(rec)
    check(lib.akv_map_recovery_f64(G, n, ptr(A), F, ptr(m), rows, ptr(ws1), ptr(ws2), ptr(rec),
                                   ptr(cos), stream()), exc)
    return rec.cpu().numpy(), cos.cpu().numpy()


def update_scores(scores: np.ndarray, retained: np.ndarray, row: np.ndarray, exc=None):
    L = scores.shape[0]
    s = to_dev(scores if L else np.zeros(1))
    idx = to_dev(retained.astype(np.int32), torch.int32) if retained.size else None
    r = to_dev(row) if retained.size else None
    out = torch.empty(L + 1, dtype=torch.float64, device=s.device)
    check(lib.akv_update_scores_f64(L, ptr(s), int(retained.size), ptr(idx), ptr(r), ptr(out),
                                    stream()), exc)
    return out.cpu().numpy()


def gather_rows(K: np.ndarray, V: np.ndarray, idx: np.ndarray, exc=None):
    m = idx.size
    dk, dv = K.shape[1], V.shape[1]
    if m == 0:
        return np.zeros((0, dk)), np.zeros((0, dv))
    Kd, Vd = to_dev(K), to_dev(V)
    ix = to_dev(idx.astype(np.int32), torch.int32)
    Kc = torch.empty(m, dk, dtype=torch.float64, device=Kd.device)
    Vc = torch.empty(m, dv, dtype=torch.float64, device=Kd.device)
    check(lib.akv_gather_rows_f64(dk, dv, ptr(Kd), ptr(Vd), m, ptr(ix), ptr(Kc), ptr(Vc), stream()),
          exc)
    return Kc.cpu().numpy(), Vc.cpu().numpy()


def tv_distance(p: np.ndarray, mask: np.ndarray, exc=None) -> float:
    pd = to_dev(p)
    md = to_dev(mask.astype(np.uint8), torch.uint8)
    out = torch.empty(1, dtype=torch.float64, device=pd.device)
    check(lib.akv_tv_distance_f64(pd.shape[0], ptr(pd), ptr(md), ptr(out), stream()), exc)
    return float(out.item())
