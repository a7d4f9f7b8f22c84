"""Same-box A/B of decode-step and verify times for package copies.

    python tools/ab_time.py ROOT_A ROOT_B[@VAR=val,VAR2=val] [--rounds 2] [--ctx 128]

Each ROOT holds a built `paper_2506_15556_b200/` (e.g. `_ab/base` made from
an older commit, and `.` for the working tree). Runs alternate A, B, A, B in
fresh processes so clock drift hits both arms alike.
"""
import argparse, os, subprocess, sys

CODE = r'''
import sys, statistics, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2506_15556_b200 as pkg
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import LLAMA3_8B
ctxlen = int(sys.argv[2])
lm = B200LM(LLAMA3_8B, seed=0, max_seq=2048, cost_mode="measured")
rng = np.random.default_rng(0)
ctx = [int(t) for t in rng.integers(4, LLAMA3_8B.vocab, ctxlen)]
lm.decode_greedy_fused(ctx, 8)
ms = []
for i in range(4):
    lm.truncate(ctxlen)
    ms += [c for _, c in lm.decode_greedy_fused(ctx, 40)[1:]]
cand = [int(t) for t in rng.integers(4, LLAMA3_8B.vocab, 64)]
v = []
for i in range(7):
    lm.truncate(ctxlen - 8)
    v.append(lm.verify_greedy_detail(ctx, cand)["gpu_ms"])
print("RESULT", pkg.__file__, round(statistics.median(ms), 4), round(statistics.median(v), 4))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("roots", nargs="+")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--ctx", type=int, default=128)
    a = ap.parse_args()
    for r in range(a.rounds):
        for arm in a.roots:
            root, _, envs = arm.partition("@")
            env = dict(os.environ, **dict(kv.split("=", 1) for kv in envs.split(",") if kv))
            out = subprocess.run([sys.executable, "-c", CODE, os.path.abspath(root), str(a.ctx)],
                                 capture_output=True, text=True, env=env)
            line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
            print(r, arm, line[0] if line else out.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
