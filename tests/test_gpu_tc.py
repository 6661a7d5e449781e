"""Tensor-core (tcgen05/TMA/TMEM) profiling passes vs. the SIMT passes on
the same inputs: ragged N (not a multiple of the 128 tile), planted biases,
batch > 1.  Both run through the C-ABI; the SIMT passes are themselves
pinned to the reference goldens by test_gpu_parity.py."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors
from paper_2310_01801_b200._lib import lib
from paper_2310_01801_b200.workloads import round_bf16

pytestmark = pytest.mark.gpu

lib.akv_debug_set_tc.argtypes = [ctypes.c_int]


def _run(q, k, v, cls, N, sl, sk, tc):
    lib.akv_debug_set_tc(1 if tc else 0)
    try:
        res, cache = encode_prompt_tensors(q, k, v, cls, ProfilerConfig(recovery_threshold=0.95),
                                           prompt_len=N, max_new_tokens=4, slopes=sl, sinks=sk,
                                           extra_thresholds=(0.98, 0.99))
        torch.cuda.synchronize()
        return res, cache
    finally:
        lib.akv_debug_set_tc(1)


@pytest.mark.parametrize("N", [1, 77, 128, 300, 1024])
def test_tc_profile_matches_simt(N):
    rng = np.random.default_rng(N)
    B, H, d = 2, 3, 128
    ld = N + 5
    x = round_bf16(rng.standard_normal((3, B, H, ld, d)).astype(np.float32))
    dev = torch.device("cuda")
    q, k, v = (torch.from_numpy(x[i]).to(dev).to(torch.bfloat16) for i in range(3))
    cls = rng.choice([0, 0, 0, 0, 2, 1], size=(B, ld)).astype(np.uint8)
    cls[:, 0] = 1
    cls_t = torch.from_numpy(cls).to(dev)
    sl = torch.tensor([0.0, 0.05, 0.0], device=dev)
    sk = torch.tensor([0.0, 0.0, 9.0], device=dev)
    rt, ct = _run(q, k, v, cls_t, N, sl, sk, True)
    rs, cs = _run(q, k, v, cls_t, N, sl, sk, False)
    np.testing.assert_allclose(ct.colsum.cpu().numpy(), cs.colsum.cpu().numpy(), rtol=2e-4, atol=1e-6)
    np.testing.assert_allclose(ct.lastp.cpu().numpy(), cs.lastp.cpu().numpy(), rtol=2e-4, atol=1e-7)
    np.testing.assert_allclose(ct.out.cpu().numpy(), cs.out.cpu().numpy(), rtol=1e-3, atol=1e-5)
    np.testing.assert_allclose(rt.recovery, rs.recovery, rtol=0, atol=5e-5)
    near = rt.near_threshold() | rs.near_threshold()
    ok = ~near.any(axis=1)
    np.testing.assert_array_equal(rt.choice[ok], rs.choice[ok])
