"""Reflection verification on a B200: the self-consistency
judge (one pass over the judge prompt, yes/no scores of the last row) against
the CPU oracle, and whole reflection turns against the oracle's event logs.

fp32 mode (TINY): scores within the stated logits tolerance (atol 2e-4);
verdicts equal whenever |yes - no| > 1e-3 (all cases here); event logs exact.
"""

import numpy as np
import pytest

from conftest import GOLDEN  # noqa: F401
from oracle.decoder import CpuDecoderLM
from paper_2506_15556_b200 import B200LM, PipelineConfig, make_stream, run_turn
from paper_2506_15556_b200 import LatencyModel
from paper_2506_15556_b200.shapes import TINY
from paper_2506_15556_b200 import SyntheticVocabulary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    lm = B200LM(TINY, seed=0, max_seq=1024)
    ref = CpuDecoderLM(TINY.as_dict(), SyntheticVocabulary(TINY.vocab), seed=0, latency=LatencyModel())
    yield lm, ref
    lm.close()


def test_judge_scores_match_oracle(pair):
    lm, ref = pair
    rng = np.random.default_rng(0)
    for _ in range(6):
        prompt = " ".join(f"w{int(t)}" for t in rng.integers(4, TINY.vocab, int(rng.integers(3, 20))))
        answer = " ".join(f"w{int(t)}" for t in rng.integers(4, TINY.vocab, int(rng.integers(2, 9)))) + " ."
        a, ca = lm.judge_consistency(prompt, answer)
        b, cb = ref.judge_consistency(prompt, answer)
        assert ca == cb
        assert abs(a.yes_score - b.yes_score) <= 2e-4 and abs(a.no_score - b.no_score) <= 2e-4
        if abs(b.yes_score - b.no_score) > 1e-3:
            assert a.consistent == b.consistent


def test_reflection_turns_match_oracle(pair):
    lm, ref = pair
    cfg = PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32, verifier="reflection")
    rng = np.random.default_rng(3)
    verdicts = 0
    for _ in range(3):
        words = " ".join(f"w{int(t)}" for t in rng.integers(4, TINY.vocab, 40))
        stream = make_stream(words, cfg.rate_chars_per_min, cfg.chunk_words)
        got = run_turn([], stream, cfg, lm)
        want = run_turn([], stream, cfg, ref)
        assert [e.to_dict() for e in got.events] == [e.to_dict() for e in want.events]
        verdicts += sum(1 for e in got.events if e.to_dict().get("judge_fallback") != "judge_unsupported")
    assert verdicts > 0
