"""Sharded conversation simulation with JSONL event logs.

The multi-GPU form of the reference's `simulate` command (cli.py:92-106 ->
metrics.py:202-216 `run_dataset`; event files as pipeline.py:108-130
`write_events_jsonl`). One process per GPU; conversation i runs on rank
i mod G with that rank's own backend; every turn's events go to
`<out>/events/<conversation>_<round>.jsonl`; rank 0 gathers the per-turn
metrics (a torch.distributed object gather, host side only — no data-path
collective) and writes them in dataset order to `<out>/metrics.jsonl` plus a
`<out>/summary.json` with means and percentiles.

In modeled-cost mode (`B200LM(cost_mode="modeled")`, the reference's
LatencyModel) a pass's cost depends only on the caller's cache handle, never
on what else ran on the device, so every output file is byte-identical for
any G — the analogue of the reference's determinism criterion
(test_acceptance.py:231-255), checked by tests/test_simulate.py at G = 1, 2.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        -m paper_2506_15556_b200.simulate --synthetic 64 --shape llama-3-8b --out runs/x
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
from pathlib import Path

from .turn import run_conversation, write_events_jsonl
from .turn_metrics import compute_metrics, load_dataset, summarize, summarize_percentiles


def run_sharded(conversations, cfg, lm, out_dir, rank: int = 0, world: int = 1, baseline: bool = False,
                group=None) -> list[dict]:
    """Simulate this rank's shard, write its event logs; rank 0 writes the report.

    Returns the per-turn metrics (all ranks' on rank 0, this rank's elsewhere)."""
    out = Path(out_dir)
    recs = []
    for i, conv in enumerate(conversations):
        if i % world != rank:
            continue
        for res in run_conversation(conv.turns, cfg, lm, conversation_id=conv.id, baseline=baseline):
            m = compute_metrics(res.events)
            write_events_jsonl(res.events, out / "events" / f"{conv.id}_{m.round}.jsonl")
            recs.append((i, dataclasses.asdict(m)))
    if world > 1:
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, recs, group=group)
        recs = [r for part in parts for r in part]
    recs.sort(key=lambda x: (x[0], x[1]["round"]))
    rows = [r for _, r in recs]
    if rank == 0:
        with (out / "metrics.jsonl").open("w") as fh:
            for r in rows:
                fh.write(json.dumps(r, sort_keys=True) + "\n")
        from .turn_metrics import MetricsRecord

        records = [MetricsRecord(**r) for r in rows]
        # nothing here depends on G (reports must be identical for any world size)
        summary = {"turns": len(rows), "conversations": len(conversations), "baseline": baseline,
                   "mean": summarize(records), "percentiles": summarize_percentiles(records)}
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
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    convs = synthetic_conversations(vocab, spec) if a.synthetic else load_dataset(a.dataset)
    cfg = c5_config(vocab, spec)
    lm = B200LM(shape, seed=a.seed, device=local, cost_mode=a.cost_mode)
    try:
        rows = run_sharded(convs, cfg, lm, a.out, rank, world, a.baseline)
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
