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

from conftest import GOLDEN  # noqa: F401
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
