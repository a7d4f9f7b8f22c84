"""Sharded conversation simulation with JSONL event logs.

The multi-GPU form of the reference's `simulate` command (cli.py:92-106 ->
metrics.py:202-216 `run_dataset`, a sequential loop over conversations that
share one backend). Conversations are independent units, so:

* one process per GPU, each with its own `B200LM` replica; no per-pass
  collective;
* a dynamic work queue: ranks claim the next conversation index with an
  atomic `add` on the torch.distributed store (`ConversationQueue`), so
  lognormal-length conversations balance across ranks instead of a static
  i mod G split;
* every turn's events go to `<out>/events/<conversation>_<round>.jsonl`
  (the reference's `write_events_jsonl`, pipeline.py:108-130); rank 0
  gathers the per-turn metrics (a host-side object gather) and writes them in
  dataset order to `<out>/metrics.jsonl` plus `<out>/summary.json`.

In modeled-cost mode (`B200LM(cost_mode="modeled")`, the reference's
LatencyModel) a pass's cost depends only on the caller's cache handle and the
kernels are batch-invariant, so a conversation's events do not depend on
which rank ran it or what ran before it: every output file is byte-identical
for any G and any claim order — the analogue of the reference's determinism
criterion (test_acceptance.py:231-255).

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \\
        -m paper_2506_15556_b200.simulate --synthetic 64 --shape llama-3-8b --out runs/x
"""

from __future__ import annotations

import argparse
import dataclasses
import itertools
import json
import os
from pathlib import Path

from ._specstream import specstream
from .fused import run_conversation
from .report import annotate_events, summarize_percentiles

_queue_ids = itertools.count()


class ConversationQueue:
    """Work queue over indices [0, n): `claim()` returns the next unclaimed index or None.

    world == 1: a local counter. world > 1: an atomic counter on the process
    group's TCPStore (one round trip per claim, ~50 µs, against seconds of
    device work per conversation)."""

    def __init__(self, n: int, world: int = 1, store=None, tag: str | None = None):
        self.n = n
        self._local = itertools.count()
        self._store = None
        if world > 1:
            import torch.distributed as dist

            base = store if store is not None else dist.distributed_c10d._get_default_store()
            # a fresh key per queue (every rank constructs its queues in the same order)
            self._store = dist.PrefixStore(f"ps_queue/{tag if tag is not None else next(_queue_ids)}", base)

    def claim(self):
        i = self._store.add("next", 1) - 1 if self._store is not None else next(self._local)
        return i if i < self.n else None


def run_sharded(conversations, cfg, lm, out_dir, rank: int = 0, world: int = 1, baseline: bool = False,
                group=None, queue: ConversationQueue | None = None, annotate: bool = False) -> list[dict]:
    """Simulate the conversations this rank claims, write their event logs; rank 0 writes the report.

    annotate: a B200LM backend's per-call device time, rows and algorithmic bytes are added
    to every verify / generate_step event (report.annotate_events; greedy / top-k only).
    Returns the per-turn metrics (all ranks' on rank 0, this rank's elsewhere)."""
    out = Path(out_dir)
    queue = queue if queue is not None else ConversationQueue(len(conversations), world)
    recs = []
    trace = annotate and getattr(lm, "call_log", "absent") is None and getattr(lm, "shape", None) is not None
    while (i := queue.claim()) is not None:
        conv = conversations[i]
        if trace:
            lm.call_log = []
        results = run_conversation(conv.turns, cfg, lm, conversation_id=conv.id, baseline=baseline)
        calls = lm.call_log if trace else None
        if trace:
            lm.call_log = None
        for res in results:
            events = res.events
            if trace:  # this turn's share of the conversation's backend calls, in order
                n = sum(1 for e in events if e.kind in ("verify", "generate_step"))
                events, calls = annotate_events(events, calls[:n], lm.shape), calls[n:]
            m = specstream.compute_metrics(res.events)
            specstream.write_events_jsonl(events, out / "events" / f"{conv.id}_{m.round}.jsonl")
            recs.append((i, dataclasses.asdict(m)))
    if world > 1:
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, recs, group=group)
        recs = [r for part in parts for r in part]
    recs.sort(key=lambda x: (x[0], x[1]["round"]))
    rows = [r for _, r in recs]
    if rank == 0:
        out.mkdir(parents=True, exist_ok=True)
        with (out / "metrics.jsonl").open("w") as fh:
            for r in rows:
                fh.write(json.dumps(r, sort_keys=True) + "\n")
        records = [specstream.MetricsRecord(**r) for r in rows]
        # nothing here depends on G (reports must be identical for any world size)
        summary = {"turns": len(rows), "conversations": len(conversations), "baseline": baseline,
                   "mean": specstream.summarize(records), "percentiles": summarize_percentiles(records)}
        (out / "summary.json").write_text(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--dataset", help="JSONL dataset ({id, turns}) as in the reference")
    ap.add_argument("--synthetic", type=int, default=0, help="N synthetic c5 conversations instead")
    ap.add_argument("--shape", default="llama-3-8b")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cost-mode", default="modeled", choices=["modeled", "measured"])
    ap.add_argument("--baseline", action="store_true")
    ap.add_argument("--annotate", action="store_true", help="add gpu_ms / rows / algorithmic_bytes to events")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PS_SHARE_GPU") == "1":
        local = 0
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    from .backend import B200LM
    from .shapes import SHAPES
    from .vocab import SyntheticVocabulary
    from .workload import WorkloadSpec, c5_config, synthetic_conversations

    shape = SHAPES[a.shape]
    vocab = SyntheticVocabulary(shape.vocab)
    spec = WorkloadSpec(conversations=a.synthetic, seed=a.seed) if a.synthetic else WorkloadSpec()
    convs = synthetic_conversations(vocab, spec) if a.synthetic else specstream.load_dataset(a.dataset)
    cfg = c5_config(vocab, spec)
    lm = B200LM(shape, seed=a.seed, device=local, cost_mode=a.cost_mode)
    try:
        rows = run_sharded(convs, cfg, lm, a.out, rank, world, a.baseline, annotate=a.annotate)
    finally:
        lm.close()
    if rank == 0:
        print(f"{len(rows)} turns -> {a.out}")
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
