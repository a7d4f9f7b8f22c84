"""The CPU oracle itself: weight generator spec, decoder contract, and the
installed reference's loop on the oracle decoder reproducing the config c1
golden logs (tests/golden/tiny_turns.json)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import weights as W
from oracle.decoder import CpuDecoderLM, DecoderOracle
from paper_2506_15556_b200 import SyntheticVocabulary, specstream
from paper_2506_15556_b200.shapes import TINY, small_shape

LatencyModel = specstream.LatencyModel

TINY_TURNS = json.loads((GOLDEN / "tiny_turns.json").read_text())


def test_weight_generator_spec():
    a = W.uniform_f32(0, 5, 1000)
    b = W.uniform_f32(0, 5, 1000, chunk=37)
    assert np.array_equal(a, b)
    assert abs(a.std() - 0.02) < 0.002 and abs(a.mean()) < 0.003
    assert np.abs(a).max() <= 0.02 * np.sqrt(3) + 1e-6
    assert not np.array_equal(a, W.uniform_f32(1, 5, 1000))
    assert not np.array_equal(a, W.uniform_f32(0, 6, 1000))
    # values are k * scale with integer k: fp32-exact spec
    k = np.round(a / W.scale_f32(0.02)).astype(np.float32)
    assert np.array_equal(k * W.scale_f32(0.02), a)


def test_bf16_rounding_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5e-3], dtype=np.float32)
    r = W.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[2] == 1.0 + 2 ** -7
    assert abs(r[3] + 2.5e-3) < 2.5e-3 * 2 ** -8


def test_decoder_cache_transparency_and_causality():
    shape = small_shape(mode=0).as_dict()
    m = DecoderOracle(shape, seed=3)
    toks = [int(t) for t in np.random.default_rng(0).integers(4, 2048, 20)]
    _, full = m.extend(toks)
    m.reset()
    _, a = m.extend(toks[:7])
    _, b = m.extend(toks[7:])
    np.testing.assert_allclose(np.concatenate([a, b]), full, rtol=1e-12, atol=1e-12)


def test_cpu_lm_contract():
    vocab = SyntheticVocabulary(TINY.vocab)
    lm = CpuDecoderLM(TINY.as_dict(), vocab, seed=0)
    ctx = [5, 6, 7, 8]
    block, handle, cost = lm.forward(ctx)
    assert block.rows.shape == (4, TINY.vocab) and cost == LatencyModel().pass_cost(4)
    block2, h2, cost2 = lm.forward(ctx + [9], handle)
    assert block2.first_position == 4 and cost2 == LatencyModel().pass_cost(1)
    np.testing.assert_array_equal(block2.rows[0], lm.forward(ctx + [9])[0].rows[4])
    with pytest.raises(specstream.PrefixViolationError):
        lm.forward(ctx, h2.truncated(4))


@pytest.mark.parametrize("i", range(len(TINY_TURNS["turns"])))
def test_tiny_turn_replay_matches_reference(i):
    """The installed reference + oracle decoder reproduces the golden turn logs."""
    rec = TINY_TURNS["turns"][i]
    vocab = SyntheticVocabulary(TINY.vocab)
    cfg = specstream.PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32)
    for arm, run in (("speculative", specstream.run_turn), ("baseline", specstream.run_baseline)):
        lm = CpuDecoderLM(TINY_TURNS["shape"], vocab, seed=TINY_TURNS["seed"], latency=LatencyModel())
        res = run([], specstream.make_stream(rec["prompt"], cfg.rate_chars_per_min, cfg.chunk_words), cfg, lm)
        assert res.final_text == rec[arm]["final_text"]
        assert [e.to_dict() for e in res.events] == rec[arm]["events"]
    assert rec["speculative"]["final_text"] == rec["baseline"]["final_text"]  # lossless


def test_judge_tokens_and_reflection_on_the_oracle():
    """Self-judgment (verify_reflection, verify.py:116-158) on the decoder oracle:
    judge text maps to one id per split word (so a pass costs `judge_cost`),
    known surfaces keep their ids, unknown words hash into the word ids, and the
    verdict is yes > no on the last row of the judge pass."""
    format_judge_prompt = specstream.lm.format_judge_prompt
    verify_reflection = specstream.verify_reflection
    split_words = specstream.text.split_words

    vocab = SyntheticVocabulary(TINY.vocab)
    ids = vocab.judge_ids("Partial Prompt: w12 w13 . yes")
    assert ids[3:6] == [12, 13, 1] and all(4 <= i < TINY.vocab for i in ids[:3] + ids[6:])
    assert ids == vocab.judge_ids("Partial Prompt: w12 w13 . yes")  # deterministic
    lm = CpuDecoderLM(TINY.as_dict(), vocab, seed=0, latency=LatencyModel())
    verdict, cost = lm.judge_consistency("w10 w11 w12", "w40 w41 .")
    text = format_judge_prompt("w10 w11 w12", "w40 w41 .")
    assert cost == lm.latency.pass_cost(len(split_words(text)))
    block, _, _ = lm.forward(vocab.judge_ids(text))
    row = block.last_row
    assert verdict.yes_score == float(row[vocab.judge_ids("yes")[0]])
    assert verdict.consistent == (verdict.yes_score > verdict.no_score)
    out = verify_reflection([5, 6, 7, 8], [40, 41, 1, 50], lm)
    assert out.judge_fallback in (None, "judge_rejected")
    if out.judge_fallback is None:
        assert out.accepted_count == 3 and out.first_sentence_accepted


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("tied", [False, True])
def test_streamed_oracle_equals_resident(mode, tied):
    """The layer-streamed oracle (weights fetched per layer, embedding gathered per
    token, LM head in row blocks) computes exactly what the resident one does."""
    shape = small_shape(mode=mode, vocab=700, tied_embeddings=tied).as_dict()
    toks = [int(t) for t in np.random.default_rng(1).integers(4, 700, 24)]
    a = DecoderOracle(shape, seed=5)
    b = DecoderOracle(shape, seed=5, stream=True)
    b.HEAD_BLOCK = 256  # several head blocks, one partial
    _, la = a.extend(toks[:10])
    _, lb = b.extend(toks[:10])
    np.testing.assert_array_equal(la, lb)
    _, la = a.extend(toks[10:])
    _, lb = b.extend(toks[10:])
    np.testing.assert_array_equal(la, lb)


def test_generator_offset_rows():
    full = W.uniform_f32(3, 9, 5000)
    np.testing.assert_array_equal(W.uniform_f32(3, 9, 1200, first=1700), full[1700:2900])
