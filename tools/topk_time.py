"""Fused top-k verify vs greedy verify at the 8B shape (same prompt/candidate, device ms).

    python tools/topk_time.py [--ctx 128] [--cand 64] [--k 3]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2506_15556_b200 import B200LM  # noqa: E402
from paper_2506_15556_b200.shapes import SHAPES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama-3-8b")
ap.add_argument("--ctx", type=int, default=128)
ap.add_argument("--cand", type=int, default=64)
ap.add_argument("--k", type=int, default=3)
a = ap.parse_args()
shape = SHAPES[a.shape]
lm = B200LM(shape, seed=0, max_seq=2048)
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, shape.vocab, a.ctx)]
cand = [int(t) for t in rng.integers(4, shape.vocab, a.cand)]
g, t = [], []
for i in range(9):
    lm.truncate(a.ctx - 8)
    g.append(lm.verify_greedy_detail(ctx, cand)["gpu_ms"])
    lm.truncate(a.ctx - 8)
    t.append(lm.verify_topk_detail(ctx, cand, a.k)["gpu_ms"])
mg, mt = statistics.median(g[1:]), statistics.median(t[1:])
print(f"{shape.name}: greedy verify {mg:.4f} ms, top-{a.k} verify {mt:.4f} ms (+{100 * (mt / mg - 1):.1f}%)")
