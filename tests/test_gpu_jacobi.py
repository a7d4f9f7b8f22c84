"""Jacobi decoding (generate.py:181-291) on a B200.

Each Jacobi iteration is a verify-shaped pass over base + window with a
rollback to b-1, served by `B200LM.forward` + device argmax rows. Fixed-point
property (the reference's criterion 2, test_acceptance.py:82-101): the
converged window equals the greedy continuation, within <= window-length
iterations. Exact here because every pass is batch-invariant (a row's argmax
does not depend on how many rows the pass scored).
"""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2506_15556_b200 import B200LM, greedy_decode, jacobi_generate, specstream
from paper_2506_15556_b200.shapes import TINY, small_shape

pytestmark = pytest.mark.gpu
GenerationBudget = specstream.GenerationBudget


@pytest.mark.parametrize("shape", [TINY, small_shape()], ids=["f32", "bf16"])
def test_jacobi_fixed_point_equals_greedy(shape):
    lm = B200LM(shape, seed=2, max_seq=1024)
    try:
        rng = np.random.default_rng(7)
        for _ in range(12):
            p = [int(t) for t in rng.integers(4, shape.vocab, int(rng.integers(1, 24)))]
            r = [int(t) for t in rng.integers(4, shape.vocab, int(rng.integers(1, 20)))]
            k = int(rng.integers(0, len(r) + 1))
            window = len(r) - k
            out = jacobi_generate(k, p, r, lm, budget=GenerationBudget(max_new_tokens=0))
            want = greedy_decode(lm, p + r[:k], max_new=window)[len(p) + k:]
            assert out.response[k:] == want
            assert sum(1 for x in out.passes if x.kind == "jacobi") <= max(1, window)
    finally:
        lm.close()


JACOBI_TURNS = __import__("json").loads((GOLDEN / "tiny_jacobi_turns.json").read_text())


@pytest.mark.parametrize("i", range(len(JACOBI_TURNS["turns"])))
def test_jacobi_turns_equal_reference_golden(i):
    """Whole c1 turns with the reference's Jacobi generator (generate.py:181-291) on
    B200LM reproduce the event logs the reference produced on the float64 oracle
    decoder (tests/golden/tiny_jacobi_turns.json): every jacobi / prefill / decode
    pass, every verify k, every timestamp."""
    rec = JACOBI_TURNS["turns"][i]
    cfg = specstream.PipelineConfig(system_prompt="", chunk_words=8, max_response_tokens=32, generator="jacobi")
    lm = B200LM(TINY, seed=JACOBI_TURNS["seed"], max_seq=1024)
    try:
        res = specstream.run_turn([], specstream.make_stream(rec["prompt"], cfg.rate_chars_per_min, cfg.chunk_words),
                                  cfg, lm)
        assert res.final_text == rec["speculative"]["final_text"]
        assert [e.to_dict() for e in res.events] == rec["speculative"]["events"]
    finally:
        lm.close()
