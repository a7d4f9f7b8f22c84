"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [f32|bf16|mid|all]

Exercises every entry point of the C-ABI on the cheap shapes: extend passes
(several chunks), a fused greedy verify with rollback, top-k verify, graph-
free and graph-replayed decode steps, logits rows. The bf16 shape uses the
8B layout (hd=128, GQA 4), so the megakernel runs its all-split and
per-tile-counter finalisation paths and the wide and decode attention units.
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path.cwd()) if (Path.cwd() / "paper_2506_15556_b200").exists() else str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2506_15556_b200 import B200LM  # noqa: E402
from paper_2506_15556_b200.shapes import TINY, small_shape  # noqa: E402


def exercise(shape, seed, use_graphs):
    rng = np.random.default_rng(seed)
    lm = B200LM(shape, seed=seed, max_seq=512, use_graphs=use_graphs)
    try:
        p = [int(t) for t in rng.integers(4, shape.vocab, 90)]
        block, handle, _ = lm.forward(p)
        am = [int(np.argmax(block.row_for(i))) for i in range(len(p))]
        cand = am[-1:] + [int(t) for t in rng.integers(4, shape.vocab, 20)]
        d = lm.verify_greedy_detail(p, cand)
        t = lm.verify_topk_detail(p, cand, 3)
        steps = lm.decode_greedy_fused(p + cand[: d["k"]], 6)
        row = np.asarray(block.row_for(len(p) - 1))
        print(shape.name, "graphs" if use_graphs else "eager", "k", d["k"], "topk-k", t["k"],
              "decode", [s[0] for s in steps], "argmax", int(row.argmax()))
    finally:
        lm.close()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("f32", "all"):
        exercise(TINY, 0, use_graphs=False)
    if which in ("bf16", "all"):
        exercise(small_shape(), 1, use_graphs=False)
    if which in ("mid", "all"):
        # GU / LM wide enough for two-piece tiles: the c_first pair finalisation
        # (verify window <= 80 rows) and the row-share scheme (the 90-row extend)
        exercise(small_shape("mid-bf16", intermediate=9728, vocab=32000), 2, use_graphs=False)
    print("sanitize_run done")


if __name__ == "__main__":
    main()
