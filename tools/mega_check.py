"""Megakernel vs legacy multi-kernel path: argmax agreement, batch invariance, timing."""
import os, sys, statistics, subprocess
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
code = r'''
import sys, statistics, numpy as np, time
sys.path.insert(0, "%s")
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import LLAMA3_8B, small_shape
shape = {"small": small_shape(), "8b": LLAMA3_8B}[sys.argv[1]]
lm = B200LM(shape, seed=1, max_seq=1024, cost_mode="measured")
rng = np.random.default_rng(0)
toks = [int(t) for t in rng.integers(4, shape.vocab, 100)]
t0 = time.time()
b, _, ms = lm.forward(toks)
am = [int(np.argmax(b.row_for(p))) for p in range(len(toks))]
print("FWD", round(ms, 3), "wall", round(time.time() - t0, 3), flush=True)
dec = lm.decode_greedy_fused(toks, 24)
print("DEC", [t for t, _ in dec][:12], "ms", [round(c, 3) for _, c in dec[1:6]], flush=True)
print("AM", am[:16], flush=True)
v = lm.verify_greedy_detail(toks[:80], toks[80:100] + [5] * 40)
print("VER k", v["k"], "ms", round(v["gpu_ms"], 3), flush=True)
''' % ROOT
for shape in sys.argv[1:]:
    for legacy in ("1", "0"):
        env = dict(os.environ, PS_LEGACY=legacy)
        try:
            out = subprocess.run([sys.executable, "-c", code, shape], env=env, capture_output=True, text=True, timeout=150)
            print(shape, "legacy" if legacy == "1" else "mega", "\n", out.stdout, out.stderr[-1500:], flush=True)
        except subprocess.TimeoutExpired:
            print(shape, legacy, "TIMEOUT", flush=True)
