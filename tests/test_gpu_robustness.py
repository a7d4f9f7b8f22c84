"""Edge cases of the C-ABI runtime on the device: the KV capacity, the staging
ring bound, and recovery after errors."""

import numpy as np
import pytest

from conftest import GOLDEN  # noqa: F401  (registers the markers)
from paper_2506_15556_b200 import B200LM, specstream
from paper_2506_15556_b200._native import CapacityError
from paper_2506_15556_b200.shapes import small_shape

pytestmark = pytest.mark.gpu


def test_fused_decode_stops_at_the_kv_capacity():
    """ps_decode_greedy never asks for steps past max_seq: near the capacity it
    returns the tokens that fit (what the reference's per-pass loop produces up
    to that point) instead of failing a request EOS could have ended early."""
    lm = B200LM(small_shape(), seed=1, max_seq=256)
    try:
        ctx = [int(t) for t in np.random.default_rng(3).integers(4, lm.vocab_size, 253)]
        got = [t for t, _ in lm.decode_greedy_fused(ctx, 64)]
        assert len(got) == 4  # the resident row's argmax + 3 steps at positions 253..255
        assert got == specstream.greedy_decode(lm, ctx, max_new=4)[len(ctx):]
        with pytest.raises(CapacityError):
            lm.forward(ctx + got + [5])
        assert lm.forward(ctx[:10])[2] > 0  # the backend recovers
    finally:
        lm.close()


def test_max_seq_beyond_the_staging_ring_is_rejected():
    with pytest.raises(ValueError):
        B200LM(small_shape(), seed=1, max_seq=62 * 256 + 64)
