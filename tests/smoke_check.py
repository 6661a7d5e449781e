"""smoke(): one small profile + compact + decode session on cuda:0 (config 0
with planted sinks), checked against the CPU oracle."""

import time

import numpy as np


def run_smoke():
    import torch

    from gpu_runner import run_case
    from helpers import oracle_case
    import cases as C
    from test_gpu_parity import _compare

    assert torch.cuda.is_available(), "smoke() needs a CUDA device"
    name = "c0_sink"
    t0 = time.time()
    r = run_case(name)
    o = oracle_case(name)
    w, opts = C.case_workload(name)
    g = dict(R=o["R"], cost=o["cost"], colsum=o["colsum"], dec_choice=o["dec_choice"],
             choice=o["choice"], enc_kept=o["enc_kept"], enc_out=o["enc_out"],
             dec_kept=o["dec_kept"], dec_out=o["dec_out"], dec_rec=o["dec_rec"])
    excluded = _compare(name, g, r, w, opts)
    print(f"smoke ok: {name} on {torch.cuda.get_device_name(0)} in {time.time() - t0:.2f}s; "
          f"policies {np.bincount(r['res'].choice[:, 0], minlength=5).tolist()}, "
          f"near-T heads {excluded}")
