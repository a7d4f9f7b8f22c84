"""Fused top-k verification (`ps_verify_topk`) and exact materialised rows, on a B200.

* Rows materialised by `ps_logits_rows` are the LM phase's own fp32 logits, so
  `np.argmax(row)` equals the device argmax on every row (bf16 and fp32).
* Known-answer top-k: the candidate is built token by token from the model's
  own rows at chosen ranks (ties broken by the lower id, `topk_tokens`,
  lm.py:139-145), so for every k the accepted length is the first position
  whose rank is >= k (`verify_topk`, verify.py:100-113). Device ranks must equal
  the ranks of the materialised rows exactly; k = 1 must equal greedy.
* A whole turn with the top-k verifier gives identical event logs through the
  fused path and the reference-style generic path (forward + topk_tokens).
"""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2506_15556_b200 import B200LM, PipelineConfig, make_stream, run_turn, specstream
from paper_2506_15556_b200.shapes import MODE_BF16, TINY, small_shape
from paper_2506_15556_b200.fused import verify_greedy, verify_topk

pytestmark = pytest.mark.gpu

SHAPES = {"bf16": small_shape(), "f32": TINY}


def rank_of(row, tok):
    row = np.asarray(row, dtype=np.float32)
    st = row[tok]
    return int(np.sum(row > st) + np.sum(row[:tok] == st))


@pytest.fixture(scope="module", params=["bf16", "f32"])
def lm(request):
    m = B200LM(SHAPES[request.param], seed=3, max_seq=1024)
    yield m
    m.close()


def test_materialised_rows_argmax_equals_device_argmax(lm):
    rng = np.random.default_rng(0)
    toks = [int(t) for t in rng.integers(4, lm.vocab_size, 90)]
    block, _, _ = lm.forward(toks)
    dev = [int(block.row_for(p).argmax()) for p in range(len(toks))]  # device argmax (LazyRow)
    rows = [np.asarray(block.row_for(p)) for p in range(len(toks))]  # ps_logits_rows
    assert [int(np.argmax(r)) for r in rows] == dev


def test_topk_known_answer_and_ranks(lm):
    rng = np.random.default_rng(1)
    vocab = lm.vocab_size
    prompt = [int(t) for t in rng.integers(4, vocab, 40)]
    want_ranks = [int(r) for r in rng.choice([0, 0, 0, 1, 2, 3, 4, 6], size=18)]
    cand = []
    for r in want_ranks:  # the token of rank r in the row that scores it
        block, _, _ = lm.forward(prompt + cand)
        row = np.asarray(block.row_for(len(prompt) + len(cand) - 1), dtype=np.float32)
        order = sorted(range(len(row)), key=lambda i: (-row[i], i))
        cand.append(int(order[r]))
        assert rank_of(row, cand[-1]) == r
    for k in (1, 2, 3, 5, 7, 9):
        d = lm.verify_topk_detail(prompt, cand, k)
        # bf16, k <= 8: ranks from the fused best-k lists, exact below k and k past it
        fused = lm.shape.mode == MODE_BF16 and k <= 8
        assert d["rank"] == ([min(r, k) for r in want_ranks] if fused else want_ranks)
        expect = next((i for i, r in enumerate(want_ranks) if r >= k), len(cand))
        assert d["k"] == expect, (k, d["k"], expect)
        # the KV was rolled back to |P| + k
        assert lm.resident() == prompt + cand[:expect]
    g = lm.verify_greedy_detail(prompt, cand)
    assert g["k"] == lm.verify_topk_detail(prompt, cand, 1)["k"]


def test_fused_topk_lists_rank_wide_window(lm):
    """One wide verify pass (bf16: ranks from the per-tile best-k lists merged
    in FINAL, no logits rows; fp32: counted over materialised rows): a rank
    below k is exact, anything else reads k on the bf16 path."""
    rng = np.random.default_rng(4)
    vocab = lm.vocab_size
    prompt = [int(t) for t in rng.integers(4, vocab, 24)]
    want = [int(r) for r in rng.choice([0, 1, 2, 5, 7, 8, 9, 30, 500], size=40)]
    cand = []
    for r in want:
        block, _, _ = lm.forward(prompt + cand)
        row = np.asarray(block.row_for(len(prompt) + len(cand) - 1), dtype=np.float32)
        order = sorted(range(len(row)), key=lambda i: (-row[i], i))
        cand.append(int(order[r]))
    lm.truncate(len(prompt) - 6)  # the verify pass recomputes 6 prompt rows + the 40 candidate rows
    d = lm.verify_topk_detail(prompt, cand, 8)
    cap = 8 if lm.shape.mode == MODE_BF16 else None
    assert d["rank"] == [min(r, cap) if cap else r for r in want]
    assert d["k"] == next((i for i, r in enumerate(want) if r >= 8), len(cand))


def test_topk_verifier_fused_equals_generic(lm):
    class Generic:  # no fused entry points: forward + topk_tokens on materialised rows
        def __init__(self, inner):
            self._lm = inner
            self.vocab, self.latency, self._backend_id = inner.vocab, inner.latency, inner._backend_id

        eos_id = 0

        def forward(self, context, cache=None):
            return self._lm.forward(context, cache)

    rng = np.random.default_rng(2)
    for trial in range(4):
        prompt = [int(t) for t in rng.integers(4, lm.vocab_size, 30)]
        cand = [t for t, _ in lm.decode_greedy_fused(prompt, 12)]
        for i in rng.choice(len(cand), size=3, replace=False):  # perturb a few tokens
            cand[int(i)] = int(rng.integers(4, lm.vocab_size))
        for k in (1, 3):
            a = verify_topk(prompt, cand, lm, k)
            b = verify_topk(prompt, cand, Generic(lm), k)
            assert (a.accepted_count, a.first_sentence_accepted, a.nfe, a.uncached_positions) == \
                (b.accepted_count, b.first_sentence_accepted, b.nfe, b.uncached_positions)
            assert a.cache.prefix == b.cache.prefix
        assert verify_topk(prompt, cand, lm, 1).accepted_count == verify_greedy(prompt, cand, lm).accepted_count


def test_topk_turn_event_logs_fused_equals_generic():
    cfg = PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32, verifier="topk", topk_k=3)
    lm = B200LM(TINY, seed=0, max_seq=1024)
    try:
        words = " ".join(f"w{int(t)}" for t in np.random.default_rng(5).integers(4, TINY.vocab, 48))
        stream = make_stream(words, cfg.rate_chars_per_min, cfg.chunk_words)
        fused = run_turn([], stream, cfg, lm)
        generic = specstream.run_turn([], stream, cfg, lm)  # the reference's topk_tokens on materialised rows
        assert [e.to_dict() for e in fused.events] == [e.to_dict() for e in generic.events]
    finally:
        lm.close()


def test_topk_contract_errors():
    lm = B200LM(small_shape(), seed=0, max_seq=256)
    try:
        with pytest.raises(ValueError):
            lm.verify_topk_detail([5, 6, 7], [8, 9], 0)
        with pytest.raises(ValueError):
            lm.verify_topk_detail([5, 6, 7], [lm.vocab_size + 3], 2)
    finally:
        lm.close()


TOPK_TURNS = __import__("json").loads((GOLDEN / "tiny_topk_turns.json").read_text())


@pytest.mark.parametrize("i", range(len(TOPK_TURNS["turns"])))
def test_topk_turns_equal_reference_golden(i):
    """Top-k (k = 3) turns pinned to the reference: tests/golden/tiny_topk_turns.json
    holds the event logs the reference's run_turn produced with its own
    verify_topk / topk_tokens on the float64 oracle decoder. The fused device
    verifier (ranks counted on the device) reproduces every event — including
    the accept-heavy rounds (k = 32, the whole candidate) whose first sentence
    resumes from the buffered TTS job."""
    rec = TOPK_TURNS["turns"][i]
    cfg = PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32, verifier="topk", topk_k=3)
    lm = B200LM(TINY, seed=TOPK_TURNS["seed"], max_seq=1024)
    try:
        res = run_turn([], make_stream(rec["prompt"], cfg.rate_chars_per_min, cfg.chunk_words), cfg, lm)
        assert res.final_text == rec["speculative"]["final_text"]
        assert [e.to_dict() for e in res.events] == rec["speculative"]["events"]
    finally:
        lm.close()
