"""The package's host-side loop replays the reference's event logs exactly.

Golden logs come from the reference itself (tests/golden/make_golden.py runs
`specstream.run_turn` / `run_baseline`, pipeline.py:270-413, over its own
`NGramLM`); here the same conversations run through this package's
`run_conversation` with the restated n-gram backend (oracle/ngram.py). Every
event — timestamps, pass kinds, uncached counts, k, TTS jobs — must match.
Unit checks below mirror the reference's module tests.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.ngram import NGramOracleLM
from paper_2506_15556_b200 import (
    PipelineConfig,
    SimClock,
    TtsSimulator,
    build_vocabulary,
    compute_metrics,
    first_sentence,
    make_stream,
    read_events_jsonl,
    run_conversation,
    write_events_jsonl,
)
from paper_2506_15556_b200.generation import GenerationBudget, ar_generate
from paper_2506_15556_b200.model_api import JudgeUnsupportedError, argmax_token, greedy_decode, topk_tokens
from paper_2506_15556_b200.turn_metrics import percentile, summarize_percentiles
from paper_2506_15556_b200.verifier import verify_greedy, verify_topk
from paper_2506_15556_b200.vocab import SyntheticVocabulary, Vocabulary, VocabularyError, split_words

NGRAM = json.loads((GOLDEN / "ngram_turns.json").read_text())


def test_greedy_decode_golden_sequence():
    g = NGRAM["greedy_decode"]
    vocab = build_vocabulary([g["corpus"]])
    lm = NGramOracleLM(vocab, seed=g["seed"])
    assert greedy_decode(lm, vocab.tokenize(g["prompt"]), max_new=g["max_new"]) == g["tokens"]
    # the reference's own test asserts this literal (test_lm.py:161-168)
    assert g["tokens"] == [9, 10, 10, 10, 9, 10, 3, 6, 11, 3]


@pytest.mark.parametrize("idx", range(len(NGRAM["cases"])))
def test_event_logs_match_reference(idx):
    case = NGRAM["cases"][idx]
    cfg = PipelineConfig.from_dict(dict(case["cfg"]))
    texts = ([cfg.system_prompt] if cfg.system_prompt else []) + case["turns"]
    vocab = build_vocabulary(texts)
    for arm, baseline in (("speculative", False), ("baseline", True)):
        lm = NGramOracleLM(vocab, seed=case["seed"], latency=cfg.lm_latency, judge_error=JudgeUnsupportedError)
        results = run_conversation(case["turns"], cfg, lm, conversation_id="g", baseline=baseline)
        want = case[arm]
        assert len(results) == len(want)
        for got, exp in zip(results, want):
            assert got.final_text == exp["final_text"]
            assert got.nfe_total == exp["nfe_total"]
            assert [e.to_dict() for e in got.events] == exp["events"]


def test_lossless_greedy_on_golden_cases():
    for case in NGRAM["cases"]:
        if case["cfg"].get("verifier", "greedy") != "greedy":
            continue
        spec = [t["final_text"] for t in case["speculative"]]
        base = [t["final_text"] for t in case["baseline"]]
        assert spec == base


def test_split_words_rules():
    assert split_words("Hello, world. 3.5 is a.b! end?") == ["Hello", ",", "world", ".", "3.5", "is", "a", ".", "b",
                                                          "!", "end", "?"]
    assert split_words('.5 "x" 1.') == [".", "5", '"', "x", '"', "1", "."]


def test_vocabulary_roundtrip_and_freeze():
    v = Vocabulary()
    ids = v.tokenize("a b , c . a")
    assert ids == [1, 2, 3, 4, 5, 1]
    assert v.tokenize(v.detokenize(ids)) == ids
    v.freeze()
    with pytest.raises(VocabularyError):
        v.tokenize("zzz")


def test_synthetic_vocabulary():
    v = SyntheticVocabulary(1000)
    ids = [0, 1, 2, 3, 4, 999]
    assert v.surface(0) == "<eos>" and v.surface(1) == "." and v.surface(999) == "w999"
    text = v.detokenize([5, 6, 1, 7, 3])
    assert text == "w5 w6. w7!"
    assert v.tokenize(text) == [5, 6, 1, 7, 3]
    with pytest.raises(VocabularyError):
        v.tokenize("w1000")
    with pytest.raises(VocabularyError):
        v.id_of("w04")
    span = first_sentence([5, 6, 2, 7], v)
    assert (span.end, span.terminator) == (3, "?")
    assert len(v) == 1000 and ids[-1] == 999


def test_stream_timing():
    s = make_stream("a" * 30, 600.0, 2)
    assert s.chunks[-1].arrival_ms == 3000.0
    s = make_stream("one two three four five", 600.0, 2)
    assert [c.text for c in s.chunks] == ["one two", "one two three four", "one two three four five"]
    assert s.poll(0.0)[0].index == -1


def test_tts_timing():
    clock = SimClock()
    tts = TtsSimulator(clock)
    job = tts.synthesize_buffer("x" * 200, 0.0)
    clock.drain()
    assert job.chunk_times[0] == 200.0 and job.chunk_times[16] == 1480.0
    assert job.state == "buffered"


def test_argmax_topk_ties():
    assert argmax_token(np.array([0.5, 0.5, 0.1])) == 0
    assert topk_tokens(np.array([9.0, 3.0, 7.0, 7.0]), 3) == {0, 2, 3}


def test_verify_lcp_brute_force():
    vocab = build_vocabulary(["tell me a story about the old tree . it grew tall and wise ? ! extra junk words"])
    lm = NGramOracleLM(vocab, seed=11)
    rng = np.random.default_rng(5)
    ids = list(range(1, len(vocab)))
    for _ in range(50):
        p = [int(rng.choice(ids)) for _ in range(int(rng.integers(1, 8)))]
        r = [int(rng.choice(ids)) for _ in range(int(rng.integers(0, 10)))]
        out = verify_greedy(p, r, lm)
        oracle = greedy_decode(lm, p, max_new=len(r))[len(p):]
        expect = 0
        while expect < min(len(r), len(oracle)) and r[expect] == oracle[expect]:
            expect += 1
        assert out.accepted_count == expect
        assert verify_topk(p, r, lm, 1).accepted_count == expect


def test_ar_generate_accounting():
    vocab = build_vocabulary(["How many apples will Alice and Bob have ?"])
    lm = NGramOracleLM(vocab, seed=9)
    p = vocab.tokenize("How many apples will Alice")
    out = ar_generate(0, p, [], lm, budget=GenerationBudget(max_new_tokens=6))
    assert [x.kind for x in out.passes].count("prefill") == 1
    assert out.nfe == len(out.response) + 1


def test_metrics_roundtrip_and_percentiles(tmp_path):
    case = NGRAM["cases"][0]
    cfg = PipelineConfig.from_dict(dict(case["cfg"]))
    vocab = build_vocabulary(([cfg.system_prompt] if cfg.system_prompt else []) + case["turns"])
    lm = NGramOracleLM(vocab, seed=case["seed"], latency=cfg.lm_latency)
    res = run_conversation(case["turns"], cfg, lm)[0]
    m = compute_metrics(res.events)
    path = tmp_path / "ev.jsonl"
    write_events_jsonl(res.events, path)
    assert compute_metrics(read_events_jsonl(path)) == m
    assert percentile([1, 2, 3, 4], 50) == 2.5
    assert summarize_percentiles([m, m])["p50_ttfs_ms"] == m.ttfs_ms
