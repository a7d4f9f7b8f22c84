"""Decode-step / verify time for values of one environment knob.

    python tools/sweep_splits.py [--var NAME] value...   (default NAME: PS_SK_G; also PS_MAX_STAGES, PS_PF_WIDE, ...)
"""
import os, subprocess, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
code = r'''
import sys, statistics, numpy as np
sys.path.insert(0, "%s")
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import LLAMA3_8B
lm = B200LM(LLAMA3_8B, seed=0, max_seq=2048, cost_mode="measured")
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, LLAMA3_8B.vocab, 128)]
lm.decode_greedy_fused(ctx, 8)
ms = []
for i in range(3):
    lm.truncate(128)
    ms += [c for _, c in lm.decode_greedy_fused(ctx, 40)[1:]]
cand = [int(t) for t in rng.integers(4, LLAMA3_8B.vocab, 64)]
v = []
for i in range(5):
    lm.truncate(120)
    v.append(lm.verify_greedy_detail(ctx, cand)["gpu_ms"])
print("RESULT", statistics.median(ms), statistics.median(v))
''' % ROOT
args = sys.argv[1:]
var = "PS_SK_G"
if args[:1] == ["--var"]:
    var, args = args[1], args[2:]
for combo in args:
    env = dict(os.environ, **{var: combo})
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(var, combo, line[0] if line else out.stderr[-500:], flush=True)
