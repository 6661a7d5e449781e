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


def test_oracle_leg_runs_on_a_tiny_workload():
    import bench

    secs = bench._oracle_heads((1, 0, [0, 1], 0.95, 1, 2, 16, 2))
    assert secs > 0
