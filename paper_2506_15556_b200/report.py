"""Latency percentiles over per-turn metrics.

The reference's `summarize` reports means only (`/root/reference/pkg/src/
specstream/metrics.py:101-122`); the BASELINE metric is a p50 TTFS, so this
adds linear-interpolated percentiles over the reference's `MetricsRecord`s.
"""

from __future__ import annotations


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
