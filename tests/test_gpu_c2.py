"""Config c2 (Qwen2.5-0.5B shape, fp32 bit-exact mode): the B200 run of a
128-token query streamed in 16 chunks with a 64-token candidate cap
reproduces the event log the reference's algorithm layer produced on the
float64 oracle decoder (tests/golden/c2_turns.json) — every verify k, every
pass, every timestamp."""

import json

import pytest

from conftest import GOLDEN
from paper_2506_15556_b200 import B200LM, PipelineConfig, make_stream, run_baseline, run_turn
from paper_2506_15556_b200.shapes import QWEN_05B

pytestmark = pytest.mark.gpu

C2 = json.loads((GOLDEN / "c2_turns.json").read_text())


def test_c2_turn_matches_reference_golden():
    lm = B200LM(QWEN_05B, seed=C2["seed"], max_seq=1024)
    try:
        cfg = PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=64)
        for rec in C2["turns"]:
            for arm, run in (("speculative", run_turn), ("baseline", run_baseline)):
                res = run([], make_stream(rec["prompt"], cfg.rate_chars_per_min, cfg.chunk_words), cfg, lm)
                assert res.final_text == rec[arm]["final_text"]
                assert [e.to_dict() for e in res.events] == rec[arm]["events"]
    finally:
        lm.close()
