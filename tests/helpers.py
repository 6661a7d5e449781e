"""Shared test helpers: run the CPU oracle on a golden case and compare
results (CUDA path or oracle) against the golden vectors."""

from __future__ import annotations

import numpy as np

import cases as C
from oracle import akv_oracle as O
from paper_2310_01801_b200.workloads import class_lut

NAME_BIT = {"special": O.ATOM_SPECIAL, "punct": O.ATOM_PUNCT,
            "frequent": O.ATOM_FREQUENT, "local": O.ATOM_LOCAL}


def case_family(w, opts):
    order = [NAME_BIT[a] for a in opts.get("order", C.ORDER_DEFAULT)
             if a not in opts.get("drop", ())]
    return O.default_family(w.r_l, w.r_f, order)


def parse_fixed(text):
    """Minimal parse of the fixed-policy strings used in cases.py."""
    atoms, r_l, r_f = 0, 0.3, 0.3
    for tok in text.split("+"):
        name = tok.split("(")[0]
        if name == "full":
            atoms |= O.ATOM_FULL
            continue
        atoms |= NAME_BIT[name]
        if "r_f=" in tok:
            r_f = float(tok.split("=")[1].rstrip(")"))
        if "r_l=" in tok:
            r_l = float(tok.split("=")[1].rstrip(")"))
    return O.Member(atoms, r_l, r_f)


def case_inputs(name):
    """Per-head float64 inputs of a golden workload case, in golden order."""
    w, opts = C.case_workload(name)
    heads = C.case_heads(w, opts)
    lut = class_lut()
    toks = {b: w.tokens(b) for b, _ in heads}
    out = []
    for b, h in heads:
        q, k, v = (x.astype(np.float64) for x in w.head_qkv(b, h))
        out.append(dict(b=b, h=h, q=q, k=k, v=v, cls=lut[toks[b]].astype(np.int64),
                        slope=w.slopes[h], sink=w.sinks[h]))
    return w, opts, out


def oracle_case(name):
    """Run the oracle head by head on a golden case."""
    w, opts, heads = case_inputs(name)
    rows = O.ROWS_LAST if opts.get("rows") == "last" else O.ROWS_ALL
    crit = O.CRIT_COSINE if opts.get("criterion") == "cosine" else O.CRIT_RECOVERY
    fixed = parse_fixed(opts["fixed"]) if "fixed" in opts else None
    fam = [fixed] if fixed else case_family(w, opts)
    N, D = w.N, w.D
    res = dict(R=[], cost=[], cos=[], choice=[], colsum=[], lastrow=[], enc_kept=[], enc_out=[],
               dec_kept=np.zeros((D, len(heads), N + D), bool),
               dec_out=np.zeros((D, len(heads), w.d)), dec_choice=[],
               dec_rec=np.zeros((D + 1, len(heads))))
    thr = [-1.0] if fixed else list(w.thresholds)
    dec_T = opts.get("decode_T", w.thresholds[0])
    for gi, hd in enumerate(heads):
        N_ = N
        prof = O.profile_head(hd["q"][:N_], hd["k"][:N_], hd["v"][:N_], hd["cls"], hd["slope"],
                              hd["sink"], fam, thr + ([dec_T] if not fixed else []), rows, crit)
        res["R"].append(prof.recoveries)
        res["cost"].append(prof.costs)
        res["cos"].append(prof.cosine)
        res["choice"].append(prof.choice[:len(thr)])
        res["colsum"].append(prof.colsum)
        res["lastrow"].append(prof.lastp)
        dchoice = prof.choice[-1] if not fixed else 0
        res["dec_choice"].append(dchoice)
        member = fam[dchoice]
        kept = O.keep_positions(member.atoms, np.arange(N_), hd["cls"], prof.colsum, N_, N_,
                                member.r_l, member.r_f)
        m = np.zeros(N_, bool)
        m[kept] = True
        res["enc_kept"].append(m)
        res["enc_out"].append(prof.out_last)
        prof.kept = kept
        st = O.compact_head(prof, hd["k"][:N_], hd["v"][:N_], member, N_, hd["slope"], hd["sink"])
        res["dec_rec"][0, gi] = st.recovery
        for t in range(D):
            pos = N_ + t
            o = O.decode_head(st, hd["q"][pos], hd["k"][pos], hd["v"][pos], pos, hd["cls"], N_)
            res["dec_kept"][t, gi, st.positions] = True
            res["dec_out"][t, gi] = o
            res["dec_rec"][t + 1, gi] = st.recovery
    for k in ("R", "cost", "cos", "choice", "colsum", "lastrow", "enc_kept", "enc_out", "dec_choice"):
        res[k] = np.asarray(res[k])
    return res


def load_golden(name):
    z = dict(np.load(C.golden_path(name)))
    w, opts = C.case_workload(name)
    z["enc_kept"] = C.unpack_kept(z["enc_kept"], w.N)
    z["dec_kept"] = C.unpack_kept(z["dec_kept"], w.N + w.D)
    return z
