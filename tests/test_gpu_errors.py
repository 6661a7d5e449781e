"""Error behaviour of the GPU path, mirroring the reference's exceptions and
messages (engine.py:173-280, profiler.py:112-145) and the
C-ABI status codes (include/akv.h): invalid input raises the reference's
EngineError / ProfilerError, unsupported shapes or exhausted capacity raise
AkvError with the library's message - never a silent CPU fallback."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _qkv(B=1, H=2, T=40, d=64, dtype=torch.float32):
    g = torch.Generator(device="cuda").manual_seed(0)
    return tuple(torch.randn(B, H, T, d, device="cuda", generator=g).to(dtype) for _ in range(3))


def test_encode_argument_errors():
    from paper_2310_01801_b200 import EngineError, ProfilerConfig, encode_prompt_tensors

    q, k, v = _qkv()
    cls = torch.zeros(1, 40, dtype=torch.uint8, device="cuda")
    with pytest.raises(EngineError, match="need a profiler config or a fixed policy"):
        encode_prompt_tensors(q, k, v, cls, None)
    with pytest.raises(EngineError, match="empty prompt"):
        encode_prompt_tensors(q, k, v, cls, ProfilerConfig(), prompt_len=0)
    with pytest.raises(EngineError, match="out of range"):
        encode_prompt_tensors(q, k, v, cls, ProfilerConfig(), prompt_len=41)
    with pytest.raises(EngineError, match="unsupported dtype"):
        encode_prompt_tensors(q.half(), k.half(), v.half(), cls, ProfilerConfig())
    with pytest.raises(EngineError, match="one shape"):
        encode_prompt_tensors(q, k[:, :, :30], v, cls, ProfilerConfig())
    with pytest.raises(EngineError, match="CUDA"):
        encode_prompt_tensors(q.cpu(), k.cpu(), v.cpu(), cls.cpu(), ProfilerConfig())


def test_unsupported_head_dim_is_a_library_error():
    from paper_2310_01801_b200 import ProfilerConfig, encode_prompt_tensors
    from paper_2310_01801_b200._lib import AKV_ERR_UNSUPPORTED, AkvError

    q, k, v = _qkv(d=48)
    cls = torch.zeros(1, 40, dtype=torch.uint8, device="cuda")
    with pytest.raises(AkvError, match="head dim") as e:
        encode_prompt_tensors(q, k, v, cls, ProfilerConfig())
    assert e.value.code == AKV_ERR_UNSUPPORTED


def test_decode_capacity_is_enforced():
    from paper_2310_01801_b200 import EngineError, ProfilerConfig, decode_step_tensors, \
        encode_prompt_tensors

    q, k, v = _qkv()
    cls = torch.zeros(1, 40, dtype=torch.uint8, device="cuda")
    _, cache = encode_prompt_tensors(q, k, v, cls, ProfilerConfig(), prompt_len=36,
                                     max_new_tokens=2)
    for t in range(2):
        decode_step_tensors(cache, q[:, :, 36 + t], k[:, :, 36 + t], v[:, :, 36 + t],
                            cls[:, 36 + t].contiguous())
    with pytest.raises(EngineError, match="capacity"):
        decode_step_tensors(cache, q[:, :, 38], k[:, :, 38], v[:, :, 38], cls[:, 38].contiguous())
    cache.check()


def test_decode_input_shapes_are_checked():
    """Rows the kernels would misread are refused before any launch: wrong
    head count, wrong dtype, q / k / v strides that differ, short rows, and
    for the multi-step call a wrong class layout or step count."""
    from paper_2310_01801_b200 import (EngineError, ProfilerConfig, decode_step_tensors,
                                       decode_steps_tensors, encode_prompt_tensors)

    q, k, v = _qkv()
    cls = torch.zeros(1, 40, dtype=torch.uint8, device="cuda")
    _, cache = encode_prompt_tensors(q, k, v, cls, ProfilerConfig(), prompt_len=30,
                                     max_new_tokens=8)
    row = lambda x, p: x[:, :, p]  # noqa: E731
    c = cls[:, 30].contiguous()
    with pytest.raises(EngineError, match="H="):
        decode_step_tensors(cache, row(q, 30)[:, :1], row(k, 30)[:, :1], row(v, 30)[:, :1], c)
    with pytest.raises(EngineError, match="q must be"):
        decode_step_tensors(cache, row(q, 30).double(), row(k, 30), row(v, 30), c)
    with pytest.raises(EngineError, match="k must be"):
        decode_step_tensors(cache, row(q, 30), row(k, 30).contiguous(), row(v, 30), c)
    with pytest.raises(EngineError, match="q must be"):
        decode_step_tensors(cache, row(q, 30)[..., :8], row(k, 30)[..., :8], row(v, 30)[..., :8], c)
    seq = lambda x: x[:, :, 30:34]  # noqa: E731
    with pytest.raises(EngineError, match="new_classes"):
        decode_steps_tensors(cache, seq(q), seq(k), seq(v), cls[:, 30:34])
    with pytest.raises(EngineError, match="steps"):
        decode_steps_tensors(cache, seq(q), k[:, :, 30:33], seq(v),
                             cls[:, 30:34].t().contiguous())
    # the valid calls still run, and the cache is intact
    decode_steps_tensors(cache, seq(q), seq(k), seq(v), cls[:, 30:34].t().contiguous())
    decode_step_tensors(cache, row(q, 34), row(k, 34), row(v, 34), cls[:, 34].contiguous())
    torch.cuda.synchronize()
    cache.check()
    assert cache.seq_len == 35


def test_profiler_config_and_threshold_errors():
    from paper_2310_01801_b200 import (ProfilerConfig, ProfilerError, encode_prompt_tensors,
                                       feasible_set, parse_policy)

    with pytest.raises(ProfilerError):
        ProfilerConfig(recovery_threshold=1.5)
    with pytest.raises(ProfilerError):
        ProfilerConfig(feasible=())
    with pytest.raises(ProfilerError):   # the last feasible entry must be full (profiler.py:129-132)
        ProfilerConfig(feasible=tuple(feasible_set())[:-1])
    q, k, v = _qkv()
    cls = torch.zeros(1, 40, dtype=torch.uint8, device="cuda")
    too_many = tuple(np.linspace(0.1, 0.9, 9))
    with pytest.raises(ProfilerError, match="thresholds"):
        encode_prompt_tensors(q, k, v, cls, ProfilerConfig(), extra_thresholds=too_many)
    res, _ = encode_prompt_tensors(q, k, v, cls, None,
                                   fixed_policy=parse_policy("special+frequent(r_f=0.5)"))
    assert res.choice.shape[1] == 1


def test_model_protocol_grid_mismatch():
    from paper_2310_01801_b200 import EngineError, ProfilerConfig, encode_prompt, generate_step
    from paper_2310_01801_b200.trace import ModelConfig
    from paper_2310_01801_b200.tokens import VocabMetadata

    class M:
        def __init__(self, heads):
            self.config = ModelConfig(1, heads, 16, 32, 0)
            self.vocab = VocabMetadata(frozenset({1}), frozenset({2}))
            self._r = np.random.default_rng(0).standard_normal((heads, 64, 16))

        def k_row(self, layer, head, pos, klass, prompt_len):
            return self._r[head, pos]

        def q_row(self, layer, head, pos, prompt_len):
            return self._r[head, pos] * 0.5

        def v_row(self, layer, head, pos):
            return self._r[head, pos] * 2.0

        def head_logits(self, concat):
            return np.zeros(32)

    prof, cache = encode_prompt(M(2), [1, 5, 6, 2, 7], ProfilerConfig(), max_new_tokens=4)
    with pytest.raises(EngineError, match="cache/profile mismatch"):
        generate_step(M(3), cache, None)
    with pytest.raises(EngineError, match="empty prompt"):
        encode_prompt(M(2), [], ProfilerConfig())
