"""Record the committed c5 pass schedule that bench.py's reference arm prices.

    python tools/make_schedule.py [--first 0] [--count 1024] [--shape llama-3-8b]

Runs c5 conversations through the reference's loop on B200LM in modeled-cost
mode (the bench's phase 1) and writes, per conversation id,
[passes, rows computed, decode passes, extend passes] to
bench_data/c5_schedule_<shape>.json (merged with what is already there).
The schedule depends on the model's argmaxes only, so it is a property of the
kernels' numerics; regenerate it after a change that alters them (bench.py
reports how many timed conversations still match).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2506_15556_b200 import B200LM, run_conversation  # noqa: E402
from paper_2506_15556_b200.build import _digest  # noqa: E402
from paper_2506_15556_b200.shapes import SHAPES  # noqa: E402
from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, synthetic_conversations  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--count", type=int, default=1024)
    ap.add_argument("--shape", default="llama-3-8b")
    a = ap.parse_args()
    shape = SHAPES[a.shape]
    lm = B200LM(shape, seed=0, cost_mode="modeled", max_seq=2048)
    spec = WorkloadSpec()
    convs = synthetic_conversations(lm.vocab, spec)
    cfg = c5_config(lm.vocab, spec)
    path = bench.schedule_path(shape.name)
    data = json.loads(path.read_text()) if path.exists() else {"conversations": {}}
    data.update({"shape": shape.name, "cost_mode": "modeled", "format": "[passes, rows, decode_passes, extend_passes]",
                 "kernels_digest": hashlib.sha256(_digest().encode()).hexdigest()[:16]})
    t0 = time.time()
    for i in range(a.first, min(len(convs), a.first + a.count)):
        conv = convs[i]
        lm.schedule = []
        run_conversation(conv.turns, cfg, lm, conversation_id=conv.id)
        data["conversations"][conv.id] = bench.summarize_schedule(lm.schedule)
        if (i - a.first) % 16 == 15:
            print(f"{i + 1 - a.first} conversations, {time.time() - t0:.0f} s", flush=True)
            path.write_text(json.dumps(data, sort_keys=True) + "\n")
    data["conversations"] = dict(sorted(data["conversations"].items()))
    path.parent.mkdir(exist_ok=True)
    path.write_text(json.dumps(data, sort_keys=True) + "\n")
    lm.close()
    print(f"wrote {path}: {len(data['conversations'])} conversations in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
