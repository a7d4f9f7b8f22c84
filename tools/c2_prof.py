"""Drive the fp32 c2 path (Qwen2.5-0.5B shape) through a prefill, a 72-row
verify and a few decode steps, for an ncu launch list:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/c2_launches.csv python tools/c2_prof.py
"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import QWEN_05B
lm = B200LM(QWEN_05B, seed=0, max_seq=1024)
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, QWEN_05B.vocab, 128)]
lm.forward(ctx[:120])
cand = [int(t) for t in rng.integers(4, QWEN_05B.vocab, 64)]
lm.verify_greedy_detail(ctx, cand)
lm.decode_greedy_fused(ctx, 3)
