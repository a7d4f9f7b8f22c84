"""Verify-window and decode-step latency of the fp32 bit-exact path (config c2,
Qwen2.5-0.5B shape) next to its HBM floor: python tools/c2_time.py"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import QWEN_05B

shape = QWEN_05B
lm = B200LM(shape, seed=0, max_seq=1024, cost_mode="measured")
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, shape.vocab, 128)]
lm.decode_greedy_fused(ctx, 4)
dec = []
for _ in range(3):
    lm.truncate(128)
    dec += [c for _, c in lm.decode_greedy_fused(ctx, 24)[1:]]
cand = [int(t) for t in rng.integers(4, shape.vocab, 64)]
ver = []
for _ in range(5):
    lm.truncate(120)
    ver.append(lm.verify_greedy_detail(ctx, cand)["gpu_ms"])
wb = shape.weight_bytes_per_pass()
print(f"c2 fp32: weights/pass {wb/1e9:.3f} GB, HBM floor {wb/6531.9e9*1e3:.3f} ms")
print(f"decode step p50 {statistics.median(dec):.3f} ms; verify (72 rows) p50 {statistics.median(ver):.3f} ms")
