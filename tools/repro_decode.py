"""Decode a few steps of the small bf16 shape after a long context (NaN / bounds repro under compute-sanitizer)."""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import small_shape
shape = small_shape()
ctxlen = int(sys.argv[1])
lm = B200LM(shape, seed=0, max_seq=2048, cost_mode="measured")
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, shape.vocab, ctxlen)]
print(lm.decode_greedy_fused(ctx, 3))
