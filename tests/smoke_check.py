"""smoke(): two small profile + compact + decode sessions on cuda:0, each
checked against the CPU oracle:

* config 0 with planted sinks (fp32, d=64: the SIMT profiling passes and
  the SIMT decode kernel);
* a config-1 slice (bf16, d=128, B=2 x 32 heads, N=256, 48 steps: the
  tcgen05/TMA profiling passes k1tc_rowlse / k1tc_colsum and the TMA +
  mma.sync decode kernel k3_decode_mma)."""

import time

import numpy as np


def run_smoke():
    import torch

    from gpu_runner import run_case
    from helpers import oracle_case
    import cases as C
    from test_gpu_parity import _compare

    assert torch.cuda.is_available(), "smoke() needs a CUDA device"
    for name in ("c0_sink", "c1_small"):
        t0 = time.time()
        r = run_case(name)
        o = oracle_case(name)
        w, opts = C.case_workload(name)
        g = dict(R=o["R"], cost=o["cost"], cos=o["cos"], colsum=o["colsum"], lastrow=o["lastrow"],
                 dec_choice=o["dec_choice"], choice=o["choice"], enc_kept=o["enc_kept"],
                 enc_out=o["enc_out"], dec_kept=o["dec_kept"], dec_out=o["dec_out"],
                 dec_rec=o["dec_rec"])
        excluded = _compare(name, g, r, w, opts)
        print(f"smoke ok: {name} ({w.dtype}, d={w.d}) on {torch.cuda.get_device_name(0)} in "
              f"{time.time() - t0:.2f}s; policies "
              f"{np.bincount(r['res'].choice[:, 0], minlength=5).tolist()}, "
              f"near-T heads {excluded}")
