"""One c2 (Qwen2.5-0.5B shape, fp32) 72-row verify pass between cudaProfilerStart/Stop,
for a per-kernel launch list:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/c2_verify.csv python tools/c2_verify_prof.py
  python tools/summarize_launches.py gpurun_out/c2_verify.csv
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_15556_b200 import B200LM  # noqa: E402
from paper_2506_15556_b200.shapes import QWEN_05B  # noqa: E402

lm = B200LM(QWEN_05B, seed=0, max_seq=1024)
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, QWEN_05B.vocab, 128)]
cand = [int(t) for t in rng.integers(4, QWEN_05B.vocab, 64)]
lm.forward(ctx[:120])
lm.verify_greedy_detail(ctx, cand)  # warm
lm.truncate(120)
torch.cuda.profiler.start()
lm.verify_greedy_detail(ctx, cand)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
