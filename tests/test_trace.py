"""AKVT trace I/O (paper_2310_01801_b200/trace.py).

CPU: the reference's own trace tests (pkg/tests/test_trace.py:1-121)
restated against this package, plus cross-implementation checks on files
the unmodified reference wrote (tests/golden/replay.akvt / .ndjson, made by
make_golden.make_trace): our reader reproduces them and our writer emits
byte-identical binary.  GPU: replaying the reference's recorded run through
K1/K2/K3 (TraceModel + generate, and the bulk trace_tensors path) gives the
reference's tokens, per-head policies and per-step retained counts."""

import io
import json
import os

import numpy as np
import pytest

import cases as C
from paper_2310_01801_b200.tokens import TokenAnnotation, TokenClass
from paper_2310_01801_b200.trace import (AttentionTrace, ModelConfig, TraceBlock,
                                         TraceDimensionError, TraceHeaderError, TraceModel,
                                         TraceTruncatedError, read_trace, write_trace,
                                         write_trace_ndjson)

REPLAY_AKVT = os.path.join(C.HERE, "replay.akvt")
REPLAY_NDJSON = os.path.join(C.HERE, "replay.ndjson")


def build_trace(rng, positions=5):
    config = ModelConfig(num_layers=2, num_heads=2, head_dim=4, vocab_size=16, seed=-3)
    classes = [TokenClass.SPECIAL] + [TokenClass.OTHER] * (positions - 1)
    tokens = [TokenAnnotation(p, int(rng.integers(0, 16)), classes[p]) for p in range(positions)]
    blocks = {key: [TraceBlock(step=p, k=rng.normal(size=4), v=rng.normal(size=4),
                               q=rng.normal(size=4)) for p in range(positions)]
              for key in config.head_grid()}
    return AttentionTrace(config, tokens, blocks)


def assert_same(a, b):
    assert a.config == b.config
    assert a.tokens == b.tokens
    assert sorted(a.blocks) == sorted(b.blocks)
    for key in a.blocks:
        assert len(a.blocks[key]) == len(b.blocks[key])
        for x, y in zip(a.blocks[key], b.blocks[key]):
            assert x.step == y.step
            for r in ("k", "v", "q"):
                assert getattr(x, r).tobytes() == getattr(y, r).tobytes()


def test_binary_round_trip_lossless(tmp_path):
    t = build_trace(np.random.default_rng(0))
    write_trace(t, tmp_path / "t.akvt")
    assert_same(t, read_trace(tmp_path / "t.akvt"))


def test_binary_round_trip_is_byte_stable(tmp_path):
    t = build_trace(np.random.default_rng(1))
    write_trace(t, tmp_path / "a.akvt")
    write_trace(read_trace(tmp_path / "a.akvt"), tmp_path / "b.akvt")
    assert (tmp_path / "a.akvt").read_bytes() == (tmp_path / "b.akvt").read_bytes()


def test_ndjson_round_trip_lossless(tmp_path):
    t = build_trace(np.random.default_rng(2))
    write_trace_ndjson(t, tmp_path / "t.ndjson")
    assert_same(t, read_trace(tmp_path / "t.ndjson"))


def test_truncated_payload_distinct_error():
    buf = io.BytesIO()
    write_trace(build_trace(np.random.default_rng(3)), buf)
    data = buf.getvalue()
    for cut in (len(data) - 7, len(data) // 2, 8, 36, 40):
        with pytest.raises(TraceTruncatedError, match="truncated payload"):
            read_trace(io.BytesIO(data[:cut]))


def test_bad_magic_is_header_error():
    with pytest.raises(TraceHeaderError, match="magic"):
        read_trace(io.BytesIO(b"NOPE" + b"\x00" * 40))


def test_zero_layer_header_rejected():
    buf = io.BytesIO()
    write_trace(build_trace(np.random.default_rng(4)), buf)
    data = bytearray(buf.getvalue())
    data[6:10] = (0).to_bytes(4, "little")
    with pytest.raises(TraceHeaderError, match="num_layers"):
        read_trace(io.BytesIO(bytes(data)))


def test_unknown_class_code_and_version():
    buf = io.BytesIO()
    write_trace(build_trace(np.random.default_rng(5)), buf)
    data = bytearray(buf.getvalue())
    data[4:6] = (2).to_bytes(2, "little")
    with pytest.raises(TraceHeaderError, match="unsupported version 2"):
        read_trace(io.BytesIO(bytes(data)))
    data = bytearray(buf.getvalue())
    data[34 + 5 * 1 + 4] = 9   # class code of token 1
    with pytest.raises(TraceHeaderError, match="token 1: unknown class code 9"):
        read_trace(io.BytesIO(bytes(data)))


def test_dimension_mismatch_rejected():
    config = ModelConfig(num_layers=1, num_heads=1, head_dim=4, vocab_size=16, seed=0)
    tokens = [TokenAnnotation(0, 1, TokenClass.SPECIAL)]
    bad = [TraceBlock(step=0, k=np.zeros(3), v=np.zeros(4), q=np.zeros(4))]
    with pytest.raises(TraceDimensionError, match="K row"):
        AttentionTrace(config, tokens, {(0, 0): bad})


def test_irregular_row_in_file_is_dimension_error():
    """A file whose block carries a short row takes the sequential scan and
    fails validation like the reference."""
    t = build_trace(np.random.default_rng(6))
    buf = io.BytesIO()
    write_trace(t, buf)
    good = buf.getvalue()
    t.blocks[(1, 1)][2] = TraceBlock(2, np.zeros(3), np.zeros(4), np.zeros(4))
    object.__setattr__(t, "blocks", t.blocks)
    from paper_2310_01801_b200.trace import _encode

    with pytest.raises(TraceDimensionError, match="K row at \\(layer=1, head=1, step=2\\)"):
        read_trace(io.BytesIO(_encode(t)))
    assert read_trace(io.BytesIO(good)).config.head_dim == 4


def test_steps_strictly_increasing_enforced():
    config = ModelConfig(num_layers=1, num_heads=1, head_dim=2, vocab_size=16, seed=0)
    tokens = [TokenAnnotation(0, 1, TokenClass.SPECIAL)]
    rows = dict(k=np.zeros(2), v=np.zeros(2), q=np.zeros(2))
    with pytest.raises(TraceDimensionError, match="strictly increasing"):
        AttentionTrace(config, tokens, {(0, 0): [TraceBlock(1, **rows), TraceBlock(1, **rows)]})


def test_trace_model_requires_complete_grid():
    t = build_trace(np.random.default_rng(5))
    del t.blocks[(1, 1)]
    with pytest.raises(TraceDimensionError, match=r"\(layer=1, head=1\)"):
        TraceModel(t)


def test_reads_reference_written_files_and_writes_them_back_identically(tmp_path):
    a = read_trace(REPLAY_AKVT)
    b = read_trace(REPLAY_NDJSON)
    assert_same(a, b)
    write_trace(a, tmp_path / "ours.akvt")
    with open(REPLAY_AKVT, "rb") as fh:
        assert (tmp_path / "ours.akvt").read_bytes() == fh.read()
    write_trace_ndjson(a, tmp_path / "ours.ndjson")
    with open(REPLAY_NDJSON, encoding="utf-8") as fh:
        assert (tmp_path / "ours.ndjson").read_text(encoding="utf-8") == fh.read()
    k, v, q = a.dense_rows()
    assert k.shape == (4, len(a.tokens), 16)


@pytest.mark.gpu
def test_replay_through_gpu_matches_reference():
    from paper_2310_01801_b200 import (GenerationConfig, ProfilerConfig, generate, read_trace,
                                       replay_tensors)

    z = dict(np.load(C.golden_path("replay")))
    P, S = int(z["prompt_len"]), int(z["steps"])
    trace = read_trace(REPLAY_AKVT)
    model = TraceModel(trace)
    prompt = model.prompt_token_ids(P)
    res = generate(model, prompt, ProfilerConfig(recovery_threshold=0.95),
                   GenerationConfig(max_new_tokens=S))
    assert res.tokens == z["tokens"].tolist()
    got = [r.split(",") for r in res.profile.to_csv().splitlines()]
    ref = [r.split(",") for r in str(z["profile_csv"]).splitlines()]
    assert [g[:3] + g[4:] for g in got] == [r[:3] + r[4:] for r in ref]
    for g, r in zip(got[1:], ref[1:]):
        assert abs(float(g[3]) - float(r[3])) < 5e-5
    grid = trace.config.head_grid()
    np.testing.assert_array_equal([[rec.head_retained[k] for k in grid] for rec in res.records],
                                  z["retained"])
    np.testing.assert_allclose([rec.mean_recovery for rec in res.records], z["mean_rec"],
                               rtol=0, atol=5e-5)
    for rec, ref_pos in zip(res.records, z["retained_pos"]):
        ref_pos = json.loads(str(ref_pos))
        for k in grid:
            assert list(rec.retained_positions[k]) == ref_pos[f"{k[0]},{k[1]}"]
    # bulk path: the whole recorded run teacher-forced through the tensor API
    pres, cache, outs = replay_tensors(trace, P, ProfilerConfig(recovery_threshold=0.95))
    choice = [pres.family[c] for c in pres.choice[:, 0]]
    assert [str(p) for p in choice] == [r[2] for r in ref[1:]]
    last = res.records[len(trace.tokens) - P]
    np.testing.assert_array_equal(cache.head_retained(), [last.head_retained[k] for k in grid])


@pytest.mark.gpu
def test_generate_with_nucleus_sampling_matches_reference():
    """generate() with the reference's Nucleus sampler (engine.py:71-90,
    382-394) on the recorded trace: the same sampled tokens as the
    reference's own run (tests/golden/nucleus.npz)."""
    from paper_2310_01801_b200 import GenerationConfig, Nucleus, ProfilerConfig, generate, read_trace

    z = dict(np.load(C.golden_path("replay")))
    n = dict(np.load(C.golden_path("nucleus")))
    P, S = int(z["prompt_len"]), int(z["steps"])
    model = TraceModel(read_trace(REPLAY_AKVT))
    prompt = model.prompt_token_ids(P)
    for (temp, top_p, seed), want in zip(n["params"], n["gen_tokens"]):
        res = generate(model, prompt, ProfilerConfig(recovery_threshold=0.95),
                       GenerationConfig(max_new_tokens=S, sampling=Nucleus(
                           temperature=float(temp), top_p=float(top_p), seed=int(seed))))
        assert res.tokens == want.tolist(), (temp, top_p, seed)
