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


def _ranks_worker(rank, world, port, q):
    import os

    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import bench

    R = bench.Ranks(cpu=True)
    mx = R.max(float(rank), 10.0 - rank)
    got = R.gather({"rank": rank})
    # each rank's decode costs of its head shard of a B=2 x H=4 workload
    from paper_2310_01801_b200.parallel import head_shard

    sh = head_shard(2, 4, world, rank)
    costs = [100 * (b + 1) + h for b in range(2) for h in range(sh.h0, sh.h1)]
    bal = bench.shard_balance(2, 4, R.gather(costs))
    R.barrier()
    q.put((rank, mx, got, bal))
    R.dist.destroy_process_group()


def test_bench_ranks_and_balance_under_gloo():
    """bench.py's multi-rank plumbing (max over ranks, gather, the head-shard
    balance report) with world size 2 over gloo on CPU."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ranks_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    for rank, mx, got, bal in out:
        assert mx == [1.0, 10.0]
        assert got == [{"rank": 0}, {"rank": 1}]
        # heads 0-1 on rank 0: 100+101+200+201 = 602; heads 2-3: 102+103+202+203 = 610
        assert abs(bal["contiguous_max_over_mean"] - 610 / 606) < 1e-12
        assert bal["lpt_max_over_mean"] <= bal["contiguous_max_over_mean"] + 1e-12
