"""Summarise a widened randomised parity sweep (tests/test_gpu_fuzz.py run
with AKV_FUZZ_SEEDS / AKV_FUZZ_STATS) into profiles/<tag>_fuzz.md.

    AKV_FUZZ_SEEDS=96:5096 AKV_FUZZ_STATS=gpurun_out/fz python -m pytest tests/test_gpu_fuzz.py -n 12
    python tools/fuzz_report.py r1 gpurun_out/fz "<command>" [more stats prefixes]
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag, prefixes = sys.argv[1], sys.argv[2:]
    rows = []
    for p in prefixes:
        for f in glob.glob(p + ".*"):
            rows += [json.loads(l) for l in open(f)]
    out = [f"# {tag}: randomised parity sweep, CUDA path vs the CPU oracle", "",
           "`tests/test_gpu_fuzz.py` widened with `AKV_FUZZ_SEEDS` on a B200 "
           "(`tools/fuzz_report.py`).  Seeds < 100000 draw prompts of 1-300 positions, "
           "seeds 100000-199999 of 255-1500 (multi-page segments), seeds >= 200000 batch 8-24 x "
           "16-32 heads with prompts of 16-130; head dims 16-128, fp32/bf16, "
           "random family orders / drops, ratios, thresholds in [0, 1], planted biases, "
           "0-24 decode steps; 20 % of seeds select by the cosine criterion and 25 % average "
           "recovery over the last row only.  Bar per seed: policies and kept-index sets "
           "bit-exact after encode and after every decode step for every compared head; "
           "recoveries (and cosine similarities) within 5e-5 (fp32) / 2e-4 (bf16); outputs "
           "within rtol 1e-4 (fp32) / 2e-2 (bf16) with an absolute floor of rtol * max|o| "
           "over the step's heads.", "",
           "Two kinds of heads are not compared, and they are listed apart:", "",
           "* **near-T** (the north star's exemption): a family member up to the chosen one "
           "has recovery within 1e-4 of T (cosine criterion: the two chosen members' "
           "similarities lie within 1e-4);",
           "* **near tie** (beyond the north star): the frequent top-k boundary is a near "
           "tie of scores - relative gap < 1e-6 at encode, < 2e-4 at a decode step - where "
           "fp32 logits vs float64 may order two scores differently.  This sweep ran with the "
           "exemption armed and met no such head; the test has since dropped it (a kept-set "
           "difference now fails whatever the gap).", "",
           "| sweep | seeds | heads compared | near-T heads | near-tie heads (encode / decode) | "
           "decode head-steps compared | of which the head's live set did not grow | "
           "max rel. output error fp32 / bf16 |", "|---|---:|---:|---:|---:|---:|---:|---|"]
    for name, sel in (("small (N <= 300)", lambda r: r["seed"] < 100000),
                      ("large (N 255-1500)", lambda r: 100000 <= r["seed"] < 200000),
                      ("wide (128-768 heads per launch)", lambda r: r["seed"] >= 200000)):
        rs = [r for r in rows if sel(r)]
        if not rs:
            continue
        e32 = max([r["max_rel_out_err"] for r in rs if r["dtype"] == "f32"] or [0])
        e16 = max([r["max_rel_out_err"] for r in rs if r["dtype"] == "bf16"] or [0])
        out.append(f"| {name} | {len(rs)} | {sum(r['compared'] for r in rs)} | "
                   f"{sum(len(r.get('near_t_heads', [])) for r in rs)} | "
                   f"{sum(len(r.get('near_tie_encode_heads', [])) for r in rs)} / "
                   f"{sum(r.get('decode_ties', 0) for r in rs)} | "
                   f"{sum(r['head_steps'] for r in rs)} | "
                   f"{sum(r['evict_steps'] for r in rs)} | {e32:.1e} / {e16:.1e} |")
    crit = [r for r in rows if r.get("criterion") == "cosine"]
    last = [r for r in rows if r.get("rows") == "last"]
    tc = [r for r in rows if r["dtype"] == "bf16" and r["d"] == 128]
    out += ["", f"Criterion / rows coverage: {len(crit)} seeds with the cosine criterion "
                f"({sum(1 for r in crit if r['dtype'] == 'bf16' and r['d'] == 128)} on the tcgen05 "
                f"path, bf16 d=128), {len(last)} with last-row recovery "
                f"({sum(1 for r in last if r['dtype'] == 'bf16' and r['d'] == 128)} on the tcgen05 "
                f"path); {len(tc)} seeds in all ran the tcgen05 profiling kernel."]
    t1 = [r for r in rows if r["T"] == 1.0]
    nt = sum(len(r.get("near_t_heads", [])) for r in rows)
    out += ["", f"Near-T heads: {nt}, of which {sum(len(r.get('near_t_heads', [])) for r in t1)} at "
                "T = 1, where every member that keeps all positions has R = 1 up to rounding."]
    listed = [(r["seed"], g) for r in rows for g in r.get("near_t_heads", []) if r["T"] != 1.0]
    if listed:
        out += ["", "Near-T heads at T < 1 (seed, head): " + ", ".join(map(str, listed[:200]))]
    ties = [(r["seed"], g) for r in rows for g in r.get("near_tie_encode_heads", [])]
    dties = [(r["seed"], g, t, f"{gap:.1e}") for r in rows for g, t, gap in r.get("near_tie_decode", [])]
    out += ["", f"Near-tie heads at encode (seed, head): {ties if ties else 'none'}",
            "", f"Near-tie heads at a decode step (seed, head, step, relative gap): "
                f"{dties if dties else 'none'}"]
    path = os.path.join(ROOT, "profiles", f"{tag}_fuzz.md")
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
