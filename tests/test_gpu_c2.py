"""Config c2 (Qwen2.5-0.5B shape, fp32 bit-exact mode): 128-token queries streamed
in 16 chunks with a 64-token candidate cap, some conversations with a second
turn whose history holds the first reply. The reference's own
`run_conversation` (pipeline.py:416-434) on B200LM reproduces the event logs
the reference produced on the float64 oracle decoder (tests/golden/c2_turns.json)
— every verify k, every pass, every timestamp — in both arms; so does the
fused-verifier binding."""

import json

import pytest

from conftest import GOLDEN
from paper_2506_15556_b200 import B200LM, fused, specstream
from paper_2506_15556_b200.shapes import QWEN_05B

pytestmark = pytest.mark.gpu

C2 = json.loads((GOLDEN / "c2_turns.json").read_text())
CFG = specstream.PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=64)


@pytest.fixture(scope="module")
def c2lm():
    lm = B200LM(QWEN_05B, seed=C2["seed"], max_seq=2048)
    yield lm
    lm.close()


@pytest.mark.parametrize("i", range(len(C2["conversations"])))
def test_c2_conversation_matches_reference_golden(c2lm, i):
    rec = C2["conversations"][i]
    for arm, baseline in (("speculative", False), ("baseline", True)):
        res = specstream.run_conversation(rec["turns"], CFG, c2lm, conversation_id=f"c2-{rec['trial']}",
                                          baseline=baseline)
        assert len(res) == len(rec[arm])
        for got, want in zip(res, rec[arm]):
            assert got.final_text == want["final_text"]
            assert got.nfe_total == want["nfe_total"]
            assert [e.to_dict() for e in got.events] == want["events"]


def test_c2_fused_binding_matches(c2lm):
    rec = C2["conversations"][0]
    res = fused.run_conversation(rec["turns"], CFG, c2lm, conversation_id=f"c2-{rec['trial']}")
    assert [[e.to_dict() for e in r.events] for r in res] == [t["events"] for t in rec["speculative"]]
