"""The reference's own loop, unmodified, on `B200LM`.

Everything the algorithm layer does here is `specstream` code — installed
into baseline/_ref, never copied — calling `B200LM.forward` and `np.argmax`
on its lazy rows:

* `run_turn` / `run_baseline` (pipeline.py:270-413) reproduce the event logs
  the reference produced on the float64 oracle decoder (tests/golden/);
* `verify_greedy` (verify.py:86-97), `greedy_decode` (lm.py:350-382) and
  `ar_generate` (generate.py:129-178) match the goldens and their pass
  accounting (test_generate.py:76-86, 112-124);
* the reference's backend-agnostic properties hold on the bf16 path:
  brute-force LCP (test_verify.py:64-79), decode/forward consistency
  (test_lm.py:175-183), cache transparency (test_lm.py:98-105, bitwise),
  splice soundness (test_generate.py:66-74), top-1 == greedy and monotone k
  (test_acceptance.py:122-136);
* criteria 5 and 6 (test_acceptance.py:139-168): a full-accept scene has
  NFETFS 1 and TTFS = one verify pass; a zero-accept final verify costs
  exactly one pass over the baseline;
* the ctypes stub of INTEGRATION.md §2 — the binding a maintainer would add
  to `specstream` — is executed as written and reproduces a golden turn.
"""

import dataclasses
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2506_15556_b200 import B200LM, SyntheticVocabulary, fused, specstream
from paper_2506_15556_b200 import _native
from paper_2506_15556_b200.backend import ps_config
from paper_2506_15556_b200.shapes import TINY, small_shape

pytestmark = pytest.mark.gpu

TINY_TURNS = json.loads((GOLDEN / "tiny_turns.json").read_text())
C1_CFG = specstream.PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32)


@pytest.fixture(scope="module")
def tiny():
    lm = B200LM(TINY, seed=0, max_seq=1024)
    yield lm
    lm.close()


@pytest.fixture(scope="module")
def small():
    lm = B200LM(small_shape(), seed=1, max_seq=1024)
    yield lm
    lm.close()


def _stream(text, cfg=C1_CFG):
    return specstream.make_stream(text, cfg.rate_chars_per_min, cfg.chunk_words)


def _events(res):
    return [e.to_dict() for e in res.events]


@pytest.mark.parametrize("i", range(len(TINY_TURNS["turns"])))
def test_reference_run_turn_on_b200_equals_golden(tiny, i):
    rec = TINY_TURNS["turns"][i]
    for arm, run in (("speculative", specstream.run_turn), ("baseline", specstream.run_baseline)):
        res = run([], _stream(rec["prompt"]), C1_CFG, tiny)
        assert res.final_text == rec[arm]["final_text"]
        assert res.nfe_total == rec[arm]["nfe_total"]
        assert _events(res) == rec[arm]["events"]
    # the fused verifier binding gives the same log
    assert _events(fused.run_turn([], _stream(rec["prompt"]), C1_CFG, tiny)) == rec["speculative"]["events"]


def test_reference_verify_greedy_on_b200_equals_golden(tiny):
    g = np.load(GOLDEN / "tiny_verify.npz")
    P, R = json.loads(str(g["prompts"])), json.loads(str(g["cands"]))
    for i, (p, r) in enumerate(zip(P, R)):
        out = specstream.verify_greedy(p, r, tiny)
        assert out.accepted_count == int(g["k"][i]), i
        assert out.first_sentence_accepted == bool(g["first_sentence"][i])
        assert out.cache.prefix == tuple(p + r[: out.accepted_count])
        assert (out.nfe, out.uncached_positions) == (1, len(p) + len(r))
        f = fused.verify_greedy(p, r, tiny)
        assert dataclasses.asdict(f) == dataclasses.asdict(out)


def test_reference_generation_on_b200(tiny):
    from oracle.decoder import CpuDecoderLM

    ref = CpuDecoderLM(TINY.as_dict(), SyntheticVocabulary(TINY.vocab), seed=0)
    rng = np.random.default_rng(11)
    budget = specstream.GenerationBudget(max_new_tokens=12)
    for _ in range(4):
        p = [int(t) for t in rng.integers(4, TINY.vocab, int(rng.integers(2, 30)))]
        want = specstream.greedy_decode(ref, p, max_new=12)
        assert specstream.greedy_decode(tiny, p, max_new=12) == want
        out = specstream.ar_generate(0, p, [], tiny, budget=budget)
        assert p + out.response == want
        kinds = [x.kind for x in out.passes]
        assert kinds.count("prefill") == 1 and kinds.count("decode") == len(out.response)
        assert out.passes[0].uncached == len(p) - 1 and all(x.uncached == 1 for x in out.passes[1:])
        assert out.nfe == len(out.response) + 1
        # a cache from the caller skips the prefill (test_generate.py:112-117)
        _, handle, _ = tiny.forward(p)
        again = specstream.ar_generate(0, p, [], tiny, cache=handle, budget=budget)
        assert not [x for x in again.passes if x.kind == "prefill"] and again.response == out.response
        # the one-call device decode loop gives the same tokens
        assert [t for t, _ in tiny.decode_greedy_fused(p, len(want) - len(p))] == want[len(p):]


def test_reference_properties_on_bf16_path(small):
    lm = small
    rng = np.random.default_rng(5)
    V = lm.vocab_size
    for trial in range(12):
        p = [int(t) for t in rng.integers(4, V, int(rng.integers(1, 40)))]
        greedy = specstream.greedy_decode(lm, p, max_new=10)[len(p):]
        cut = int(rng.integers(0, len(greedy) + 1))
        r = greedy[:cut] + [int(t) for t in rng.integers(1, V, int(rng.integers(0, 6)))]
        # brute-force LCP (test_verify.py:64-79)
        out = specstream.verify_greedy(p, r, lm)
        expect = 0
        for a, b in zip(r, greedy):
            if a != b:
                break
            expect += 1
        assert out.accepted_count == expect
        # top-1 == greedy and monotone in k (test_acceptance.py:122-136), fused top-k
        t1 = fused.verify_topk(p, r, lm, 1)
        assert (t1.accepted_count, t1.first_sentence_accepted) == (out.accepted_count, out.first_sentence_accepted)
        counts = [fused.verify_topk(p, r, lm, k).accepted_count for k in (1, 2, 3, 5, 10)]
        assert counts == sorted(counts)
        # splice soundness (test_generate.py:66-74)
        k = int(rng.integers(0, len(r) + 1))
        res = specstream.ar_generate(k, p, r, lm, budget=specstream.GenerationBudget(max_new_tokens=5))
        assert res.response[:k] == r[:k]
    # decode/forward consistency (test_lm.py:175-183)
    p = [int(t) for t in rng.integers(4, V, 20)]
    seq = specstream.greedy_decode(lm, p, max_new=8)
    block, _, _ = lm.forward(seq)
    for pos in range(len(p), len(seq)):
        assert seq[pos] == specstream.argmax_token(block.row_for(pos - 1))
    # cache transparency, bitwise (test_lm.py:98-105)
    full, _, _ = lm.forward(seq)
    _, handle, _ = lm.forward(seq[:7])
    part, _, _ = lm.forward(seq, handle)
    assert part.first_position == 7
    a = np.stack([np.asarray(full.row_for(i)) for i in range(7, len(seq))])
    b = np.stack([np.asarray(part.row_for(i)) for i in range(7, len(seq))])
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _criteria_turns(lm, cfg, seed, trials):
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        text = " ".join(f"w{int(t)}" for t in rng.integers(4, lm.vocab_size, 16))
        pred = specstream.run_turn([], _stream(text, cfg), cfg, lm)
        base = specstream.run_baseline([], _stream(text, cfg), cfg, lm)
        assert pred.final_text == base.final_text  # lossless
        last = [e for e in pred.events if e.kind == "verify"][-1].payload
        pm, bm = specstream.compute_metrics(pred.events), specstream.compute_metrics(base.events)
        yield last, pm, bm, cfg.lm_latency.pass_cost(last["uncached"])


CRIT_CFG = specstream.PipelineConfig(system_prompt="", chunk_words=4, max_response_tokens=8)


def test_acceptance_criterion_5_full_accept_on_device():
    """Criterion 5: a final verify that accepts the first sentence gives NFETFS 1 and
    TTFS = audio latency = that verify pass (modeled cost, exact). Scene: the
    terminator ids carry a large logit bias, so every candidate is a run of
    terminators, the first sentence is its first token, and the final prompt keeps
    it (the B200 analogue of the reference's scripted full-accept scene,
    test_pipeline.py:44-69; the buffered-TTS resume path of generate.py:365-380)."""
    shape = dataclasses.replace(TINY, name="tiny-terminators", term_bias_sigma=40.0)
    lm = B200LM(shape, seed=0, max_seq=1024)
    full = 0
    try:
        for last, pm, bm, verify_pass in _criteria_turns(lm, CRIT_CFG, 17, 8):
            if last["first_sentence_accepted"]:
                full += 1
                assert pm.nfetfs == 1
                assert pm.ttfs_ms == verify_pass and pm.audio_latency_ms == verify_pass
    finally:
        lm.close()
    assert full >= 4, full


def test_acceptance_criterion_6_zero_accept_on_device(tiny):
    """Criterion 6: a zero-accept final verify costs exactly one verify pass over
    the baseline, in TTFS and in audio latency (modeled cost, exact)."""
    zero = 0
    for last, pm, bm, verify_pass in _criteria_turns(tiny, CRIT_CFG, 23, 8):
        if last["k"] == 0:
            zero += 1
            assert pm.ttfs_ms - bm.ttfs_ms == verify_pass
            assert pm.audio_latency_ms - bm.audio_latency_ms == verify_pass
    assert zero >= 2, zero


def _integration_stub():
    text = (ROOT / "INTEGRATION.md").read_text()
    section = text[text.index("## 2."):text.index("## 3.")]
    return re.search(r"```python\n(.*?)```", section, re.S).group(1)


def test_integration_stub_runs_the_reference_loop():
    os.environ["PREDGEN_B200_LIB"] = str(_native.LIB_PATH)
    ns: dict = {}
    exec(compile(_integration_stub(), "INTEGRATION.md#2", "exec"), ns)
    ours = ps_config(TINY, seed=0, max_seq=1024)
    cfg = ns["PsConfig"]()
    for name, _ in _native.PsConfig._fields_:
        if name != "reserved":
            setattr(cfg, name, getattr(ours, name))
    backend = ns["B200Backend"](SyntheticVocabulary(TINY.vocab), cfg)
    rec = TINY_TURNS["turns"][0]
    for arm, run in (("speculative", specstream.run_turn), ("baseline", specstream.run_baseline)):
        res = run([], _stream(rec["prompt"]), C1_CFG, backend)
        assert _events(res) == rec[arm]["events"]
    ns["_lib"].ps_destroy(backend._h)
