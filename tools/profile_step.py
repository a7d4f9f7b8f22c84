"""Drive a few 8B-shape passes for ncu: prefill a context, one verify pass,
then decode steps (graph replays). Usage under gpurun:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/profile_step.py
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import SHAPES

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama-3-8b")
ap.add_argument("--ctx", type=int, default=128)
ap.add_argument("--window", type=int, default=72)
ap.add_argument("--decode", type=int, default=3)
a = ap.parse_args()
shape = SHAPES[a.shape]
lm = B200LM(shape, seed=0, max_seq=2048)
import numpy as np
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, shape.vocab, a.ctx)]
lm.forward(ctx)                                   # prefill
cand = [int(t) for t in rng.integers(4, shape.vocab, a.window - 8)]
new = [int(t) for t in rng.integers(4, shape.vocab, 8)]
lm.verify_greedy_detail(ctx + new, cand)          # verify pass: 72 rows
lm.decode_greedy_fused(ctx + new, a.decode + 1)   # graph capture + replays
lm.decode_greedy_fused(ctx + new, a.decode + 1)
print("done", lm.stats())
