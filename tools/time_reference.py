"""Time the UNMODIFIED reference (importable only in the build container,
/root/reference) on a bounded config-1 sample: batch row 0, 8 of the 32
heads (2 planted + 6 plain), prompt 1024, 512 teacher-forced decode steps,
diagnostics off, through the reference's own encode_prompt / generate_step
(ArrayModel from tests/golden/make_golden.py folds the planted bias).
Prints tok/s of the full row (heads are independent: x32/8 of the sample time).

    python tools/time_reference.py [n_heads] [decode_steps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [os.path.join(ROOT, "tests", "golden"), ROOT]
import make_golden as MG  # noqa: E402  (puts /root/reference/pkg/src on the path)
from adaptive_kv import ProfilerConfig, encode_prompt, generate_step  # noqa: E402
from adaptive_kv.tokens import VocabMetadata  # noqa: E402

from paper_2310_01801_b200.workloads import PUNCT_IDS, SPECIAL_IDS, config1  # noqa: E402


def main():
    nh = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    D = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    w = config1()
    planted = [h for h in range(w.H) if w.slopes[h] or w.sinks[h]][:2]
    heads = planted + [h for h in range(w.H) if h not in planted][: nh - len(planted)]
    tok = w.tokens(0)
    qs, ks, vs = zip(*(w.head_qkv(0, h) for h in heads))
    vocab = VocabMetadata(special_ids=frozenset(SPECIAL_IDS), punctuation_ids=frozenset(PUNCT_IDS))
    model = MG.ArrayModel(np.stack(qs).astype(np.float64), np.stack(ks).astype(np.float64),
                          np.stack(vs).astype(np.float64), w.slopes[heads], w.sinks[heads], vocab)
    t0 = time.perf_counter()
    _, cache = encode_prompt(model, list(tok[: w.N]), ProfilerConfig(recovery_threshold=0.95),
                             diagnostics=False)
    t1 = time.perf_counter()
    generate_step(model, cache, None)
    for t in range(D):
        generate_step(model, cache, int(tok[w.N + t]))
    t2 = time.perf_counter()
    scale = w.H / len(heads)
    row_s = (t2 - t0) * scale
    print(f"reference, batch row 0, {len(heads)} heads: encode {t1 - t0:.2f} s, {D} steps "
          f"{t2 - t1:.2f} s; full row (x{scale:g}) {row_s:.1f} s -> {D / row_s:.2f} tok/s; "
          f"profiling {1e3 * (t1 - t0) * scale:.0f} ms/layer-row")


if __name__ == "__main__":
    main()
