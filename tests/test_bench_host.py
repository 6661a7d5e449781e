"""bench.py's host-side accounting on CPU: the algorithmic bytes behind the
K3 roofline (live K/V rows + the new row + 4-byte metadata,
16 bytes of score traffic per FREQUENT slot, q/k/v in and o out) and the
exponential-rate roofline; a tiny run of the CPU legs' oracle session."""

import numpy as np


class _Fam:
    def __init__(self, bits, full):
        self.bits, self.is_full = bits, full


class _Res:
    def __init__(self, choice):
        self.choice = np.asarray(choice)[:, None]
        # member 0: special+frequent (bits 1 | 4), member 1: full
        self.family = [_Fam(1 | 4, False), _Fam(8, True)]


class _W:
    d, dtype, B, H, N, D = 128, "bf16", 1, 2, 10, 3


def test_decode_bytes_formula():
    import bench

    w = _W()
    res = _Res([0, 1])                      # head 0 FREQUENT, head 1 full
    lives = [np.array([4, 10]), np.array([5, 11]), np.array([5, 12])]
    got = bench.decode_bytes(w, res, lives)
    es, d = 2, 128
    want = []
    for L in lives[:-1]:
        b = ((L + 1) * (2 * d * es + 4)).sum() + L[0] * 16 + 2 * (3 * d * es + d * 4)
        want.append(int(b))
    assert got == want


def test_exp_roofline():
    import bench

    class Clk:
        def summary(self):
            return {"sm_mhz": 1000.0}

    class W:
        B, H, N = 2, 4, 8

    import torch

    if not torch.cuda.is_available():   # the SM count needs a device; check the arithmetic
        orig = torch.cuda.get_device_properties
        torch.cuda.get_device_properties = lambda i: type("P", (), {"multi_processor_count": 148})
        try:
            r = bench._exp_roofline(W(), 1.0, Clk())
        finally:
            torch.cuda.get_device_properties = orig
    else:
        r = bench._exp_roofline(W(), 1.0, Clk())
    exps = 2 * 4 * 8 * 9
    assert r["exps_per_launch"] == exps
    assert abs(r["achieved"] - exps / 1e-3 / 1e9) < 1e-9
    sms = 148 if not torch.cuda.is_available() else torch.cuda.get_device_properties(0).multi_processor_count
    assert abs(r["peak"] - 16 * sms * 1000e6 / 1e9) < 1e-6


def test_cpu_legs_run_on_a_tiny_workload():
    import bench

    for kind in ("port", "reference"):
        if kind == "reference" and not bench._reference_available():
            continue
        secs = bench._cpu_job((1, [(0, [0, 1])], 0.95, 1, 2, 16, 2, kind))
        assert secs > 0


def test_reference_arm_does_not_map_the_product_library():
    """The CPU legs load the workload generator by path: the product
    package (whose import maps libakv_sm100a.so) stays unimported."""
    import subprocess
    import sys

    import bench

    code = ("import sys, bench; bench._cpu_job((1, [(0, [0])], 0.95, 1, 2, 16, 2, bench._cpu_kind())); "
            "assert 'paper_2310_01801_b200' not in sys.modules, 'product package imported'; "
            "maps = open('/proc/self/maps').read(); assert 'libakv_sm100a' not in maps; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=bench.ROOT, capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_reference_leg_matches_the_oracle_port_on_a_small_session():
    """The folded model drives the unmodified reference to the same kept
    sets the oracle port computes (planted sink head, evictions)."""
    import bench

    if not bench._reference_available():
        import pytest

        pytest.skip("baseline/_ref not installed")
    import numpy as np
    from adaptive_kv import ProfilerConfig, encode_prompt, generate_step

    from oracle import akv_oracle as O

    W = bench._workloads()
    w = W.config1(seed=1, B=1, H=32, N=96, D=6)
    heads = [h for h in range(w.H) if w.sinks[h]][:2] + [0]
    m = bench._FoldedModel(w, 0, heads)
    N = w.N
    _, cache = encode_prompt(m, [int(x) for x in m.tokens[:N]], ProfilerConfig(recovery_threshold=0.99),
                             diagnostics=False)
    generate_step(m, cache, None)
    for t in range(w.D):
        generate_step(m, cache, int(m.tokens[N + t]))
    cls = W.class_lut()[w.tokens(0)].astype(np.int64)
    fam = O.default_family(w.r_l, w.r_f)
    for i, h in enumerate(heads):
        q, k, v = (x.astype(np.float64) for x in w.head_qkv(0, h))
        prof = O.profile_head(q[:N], k[:N], v[:N], cls, w.slopes[h], w.sinks[h], fam, [0.99])
        st = O.compact_head(prof, k[:N], v[:N], fam[prof.choice[0]], N, w.slopes[h], w.sinks[h])
        for t in range(w.D):
            O.decode_head(st, q[N + t], k[N + t], v[N + t], N + t, cls, N)
        assert list(np.sort(st.positions)) == cache.heads[(0, i)].positions
