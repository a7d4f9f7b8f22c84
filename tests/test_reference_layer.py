"""The installed reference (baseline/_ref) is the one the goldens came from,
and this package's additions compose with it (CPU, no GPU).

The algorithm layer — `run_turn`, `run_baseline`, `verify_*`, `ar_generate`,
`jacobi_generate`, the clock, the TTS model, `compute_metrics` — is the
reference's own code, used unmodified (paper_2506_15556_b200/_specstream.py).
tests/golden/ngram_turns.json holds event logs the reference produced over
its own `NGramLM` (tests/golden/make_golden.py); replaying them pins the
installed copy. The fused-verifier binding (`paper_2506_15556_b200.fused`)
must give identical logs on a backend without fused entry points.
"""

import json

import pytest

from conftest import GOLDEN
from paper_2506_15556_b200 import SyntheticVocabulary, fused, percentile, specstream, summarize_percentiles

NGRAM = json.loads((GOLDEN / "ngram_turns.json").read_text())


def _vocab_for(case):
    cfg = specstream.PipelineConfig.from_dict(dict(case["cfg"]))
    texts = ([cfg.system_prompt] if cfg.system_prompt else []) + case["turns"]
    return cfg, specstream.build_vocabulary(texts)


def test_installed_reference_greedy_golden():
    g = NGRAM["greedy_decode"]
    vocab = specstream.build_vocabulary([g["corpus"]])
    lm = specstream.NGramLM(vocab, seed=g["seed"])
    assert specstream.greedy_decode(lm, vocab.tokenize(g["prompt"]), max_new=g["max_new"]) == g["tokens"]
    # the reference's own test asserts this literal (test_lm.py:161-168)
    assert g["tokens"] == [9, 10, 10, 10, 9, 10, 3, 6, 11, 3]


@pytest.mark.parametrize("idx", range(len(NGRAM["cases"])))
@pytest.mark.parametrize("runner", ["reference", "fused-binding"])
def test_event_logs_match_golden(idx, runner):
    case = NGRAM["cases"][idx]
    cfg, vocab = _vocab_for(case)
    run_conversation = specstream.run_conversation if runner == "reference" else fused.run_conversation
    for arm, baseline in (("speculative", False), ("baseline", True)):
        lm = specstream.NGramLM(vocab, seed=case["seed"], latency=cfg.lm_latency)
        results = run_conversation(case["turns"], cfg, lm, conversation_id="g", baseline=baseline)
        want = case[arm]
        assert len(results) == len(want)
        for got, exp in zip(results, want):
            assert got.final_text == exp["final_text"]
            assert got.nfe_total == exp["nfe_total"]
            assert [e.to_dict() for e in got.events] == exp["events"]


def test_fused_binding_is_scoped():
    original = specstream.pipeline.make_verifier
    with fused.fused_verifiers():
        assert specstream.pipeline.make_verifier is fused.make_verifier
    assert specstream.pipeline.make_verifier is original


def test_synthetic_vocabulary_is_a_reference_vocabulary():
    v = SyntheticVocabulary(1000)
    assert isinstance(v, specstream.text.Vocabulary) and v.frozen and len(v) == 1000
    assert v.surface(0) == "<eos>" and v.surface(1) == "." and v.surface(999) == "w999"
    text = v.detokenize([5, 6, 1, 7, 3])
    assert text == "w5 w6. w7!"
    assert v.tokenize(text) == [5, 6, 1, 7, 3]
    with pytest.raises(specstream.VocabularyError):
        v.tokenize("w1000")
    with pytest.raises(specstream.VocabularyError):
        v.id_of("w04")
    span = specstream.first_sentence([5, 6, 2, 7], v)
    assert (span.end, span.terminator) == (3, "?")
    judge = v.judge_ids(specstream.lm.format_judge_prompt("w5 w6", "w7."))
    assert len(judge) == len(specstream.text.split_words(specstream.lm.format_judge_prompt("w5 w6", "w7.")))
    assert all(0 <= t < 1000 for t in judge)


def test_percentiles():
    case = NGRAM["cases"][0]
    cfg, vocab = _vocab_for(case)
    lm = specstream.NGramLM(vocab, seed=case["seed"], latency=cfg.lm_latency)
    res = specstream.run_conversation(case["turns"], cfg, lm)[0]
    m = specstream.compute_metrics(res.events)
    assert percentile([1, 2, 3, 4], 50) == 2.5
    assert percentile([5], 90) == 5
    with pytest.raises(ValueError):
        percentile([], 50)
    s = summarize_percentiles([m, m])
    assert s["p50_ttfs_ms"] == m.ttfs_ms and s["turns"] == 2


def test_annotate_events_joins_calls_in_order():
    from paper_2506_15556_b200.report import annotate_events
    from paper_2506_15556_b200.shapes import TINY

    case = NGRAM["cases"][0]
    cfg, vocab = _vocab_for(case)
    lm = specstream.NGramLM(vocab, seed=case["seed"], latency=cfg.lm_latency)
    res = specstream.run_conversation(case["turns"][:1], cfg, lm)[0]
    n = sum(1 for e in res.events if e.kind in ("verify", "generate_step"))
    calls = [(10 + i, i % 3, 0.5 * i) for i in range(n)]
    out = annotate_events(res.events, calls, TINY)
    passes = [e for e in out if e.kind in ("verify", "generate_step")]
    assert [(e.payload["rows_computed"], e.payload["gpu_ms"]) for e in passes] == [(r, ms) for _, r, ms in calls]
    assert all((e.payload["algorithmic_bytes"] > 0) == (e.payload["rows_computed"] > 0) for e in passes)
    assert [e.to_dict()["kind"] for e in out] == [e.kind for e in res.events]
    assert "gpu_ms" not in res.events[0].payload  # the reference's events are not modified
    with pytest.raises(ValueError):
        annotate_events(res.events, calls[1:], TINY)
