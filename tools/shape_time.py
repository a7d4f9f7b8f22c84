"""Decode-step and 72-row verify latency of any registered shape against its
HBM floor (weights streamed once per pass):

    python tools/shape_time.py mistral-7b
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import SHAPES

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "mistral-7b"]
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
floor = shape.weight_bytes_per_pass() / 6531.9e9 * 1e3
d, v = statistics.median(dec), statistics.median(ver)
print(f"{shape.name}: weights/pass {shape.weight_bytes_per_pass()/1e9:.3f} GB, HBM floor {floor:.3f} ms")
print(f"decode step p50 {d:.3f} ms ({floor/d:.2f} of roofline); verify (72 rows) p50 {v:.3f} ms ({floor/v:.2f})")
