"""Latency percentiles over per-turn metrics, and per-pass device annotations.

The reference's `summarize` reports means only (`/root/reference/pkg/src/
specstream/metrics.py:101-122`); the BASELINE metric is a p50 TTFS, so this
adds linear-interpolated percentiles over the reference's `MetricsRecord`s.

`annotate_events` adds the SURVEY §5 tracing keys to the reference's event log
(schema: pipeline.py:189-219): every `verify` and `generate_step` event gets the
device time, rows computed and algorithmic HBM bytes of the backend call that
produced it.
"""

from __future__ import annotations

import dataclasses


def percentile(values, q: float) -> float:
    """Linear-interpolated percentile (numpy's default method), q in [0, 100]."""
    xs = sorted(values)
    if not xs:
        raise ValueError("percentile of an empty set")
    pos = (len(xs) - 1) * q / 100.0
    lo = int(pos)
    hi = min(lo + 1, len(xs) - 1)
    return xs[lo] + (xs[hi] - xs[lo]) * (pos - lo)


def summarize_percentiles(records, qs=(50, 90, 99)) -> dict:
    out = {"turns": len(records)}
    for q in qs:
        out[f"p{q}_ttfs_ms"] = percentile([r.ttfs_ms for r in records], q)
        out[f"p{q}_latency_ms"] = percentile([r.audio_latency_ms for r in records], q)
        out[f"p{q}_nfetfs"] = percentile([r.nfetfs for r in records], q)
    return out


def annotate_events(events, call_log, shape) -> list:
    """The reference's turn events with `gpu_ms`, `rows_computed` and `algorithmic_bytes`
    payload keys on every verify / generate_step event.

    `call_log` is a `B200LM.call_log` collected over the turn: one (context length, rows
    computed, device ms) entry per backend call, in call order. Greedy and top-k turns
    make exactly one call per such event (a prefix hit logs 0 rows and 0 bytes); events
    are sorted stably by time, which keeps the call order. Reflection turns add judge
    passes and are not supported."""
    passes = [e for e in events if e.kind in ("verify", "generate_step")]
    if len(passes) != len(call_log):
        raise ValueError(f"{len(passes)} verify/generate_step events but {len(call_log)} backend calls "
                         "(annotate one greedy or top-k turn per call log)")
    calls = iter(call_log)
    out = []
    for e in events:
        if e.kind in ("verify", "generate_step"):
            n_ctx, rows, ms = next(calls)
            extra = {"gpu_ms": float(ms), "rows_computed": int(rows),
                     "algorithmic_bytes": int(shape.pass_bytes(rows, n_ctx)) if rows else 0}
            e = dataclasses.replace(e, payload={**e.payload, **extra})
        out.append(e)
    return out
