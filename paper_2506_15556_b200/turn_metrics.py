"""TTFS / NFETFS / audio latency from an event log, and dataset summaries.

`compute_metrics` follows the reference exactly (`/root/reference/pkg/src/
specstream/metrics.py:43-88`): TTFS = first `sentence_emitted` − final chunk
arrival; NFETFS = Σ verify.nfe + #generate_step with t in (t_final,
t_first_sentence]; audio latency = `audio_start` − final arrival. It is a
pure function of the log, so it round-trips through JSONL bit-exactly.

Beyond the reference's means-only `summarize` (`metrics.py:101-122`) this adds
the percentile summary BASELINE.json's "p50 TTFS" needs.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

NFETFS_BINS = ("1", "2-5", "6-10", "11-20", ">20")


class MalformedLogError(ValueError):
    def __init__(self, missing: list[str]) -> None:
        super().__init__(f"event log is missing required events: {', '.join(missing)}")
        self.missing = missing


@dataclass
class MetricsRecord:
    turn_id: str
    round: int
    ttfs_ms: float
    nfetfs: int
    audio_latency_ms: float
    accepted_fraction: float | None
    first_sentence_accepted: bool
    speedup: float | None = None


def compute_metrics(events) -> MetricsRecord:
    final_chunk = audio = last_verify = None
    t_sentence = None
    for e in events:
        if e.kind == "chunk_received" and e.payload.get("is_final"):
            final_chunk = e
        elif e.kind == "audio_start" and audio is None:
            audio = e
        elif e.kind == "sentence_emitted" and t_sentence is None:
            t_sentence = e.t_ms
        elif e.kind == "verify":
            last_verify = e
    missing = [name for name, v in (("final chunk_received", final_chunk), ("audio_start", audio),
                                    ("sentence_emitted", t_sentence)) if v is None]
    if missing:
        raise MalformedLogError(missing)
    t0 = final_chunk.payload["arrival_ms"]
    nfetfs = 0
    for e in events:
        if t0 < e.t_ms <= t_sentence:
            if e.kind == "verify":
                nfetfs += e.payload["nfe"]
            elif e.kind == "generate_step":
                nfetfs += 1
    return MetricsRecord(
        turn_id=events[0].turn_id, round=events[0].round, ttfs_ms=t_sentence - t0, nfetfs=nfetfs,
        audio_latency_ms=audio.t_ms - t0,
        accepted_fraction=last_verify.payload["accepted_fraction"] if last_verify else None,
        first_sentence_accepted=bool(last_verify.payload["first_sentence_accepted"]) if last_verify else False)


def attach_speedups(records, baselines) -> None:
    by_id = {b.turn_id: b for b in baselines}
    for r in records:
        if r.turn_id not in by_id:
            raise ValueError(f"no baseline record for turn {r.turn_id}")
        base = by_id[r.turn_id]
        r.speedup = base.audio_latency_ms / r.audio_latency_ms if r.audio_latency_ms > 0 else None


def summarize(records, baselines=None) -> dict:
    if not records:
        raise ValueError("cannot summarize an empty record set")
    if baselines is not None:
        if sorted(r.turn_id for r in records) != sorted(b.turn_id for b in baselines):
            raise ValueError("record and baseline turn ids do not match")
        if not baselines:
            raise ValueError("cannot summarize against an empty baseline set")
    n = len(records)
    out = {"turns": n,
           "mean_ttfs_ms": sum(r.ttfs_ms for r in records) / n,
           "mean_nfetfs": sum(r.nfetfs for r in records) / n,
           "mean_latency_ms": sum(r.audio_latency_ms for r in records) / n,
           "speedup": None}
    if baselines is not None:
        base_mean = sum(b.audio_latency_ms for b in baselines) / len(baselines)
        if out["mean_latency_ms"] > 0:
            out["speedup"] = base_mean / out["mean_latency_ms"]
    return out


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


def nfetfs_bin(value: int) -> str:
    for upper, name in ((1, "1"), (5, "2-5"), (10, "6-10"), (20, "11-20")):
        if value <= upper:
            return name
    return ">20"


def nfetfs_histogram(records, by_round: bool = False) -> dict:
    def zeros():
        return {b: 0 for b in NFETFS_BINS}
    if not by_round:
        counts = zeros()
        for r in records:
            counts[nfetfs_bin(r.nfetfs)] += 1
        return {"bins": list(NFETFS_BINS), "counts": counts}
    rounds: dict = {}
    for r in records:
        rounds.setdefault(str(r.round), zeros())[nfetfs_bin(r.nfetfs)] += 1
    return {"bins": list(NFETFS_BINS), "rounds": dict(sorted(rounds.items()))}


@dataclass
class Conversation:
    id: str
    turns: list


def load_dataset(path) -> list[Conversation]:
    convs = [Conversation(str(d["id"]), list(d["turns"]))
             for d in (json.loads(line) for line in Path(path).read_text().splitlines() if line.strip())]
    if not convs:
        raise ValueError(f"dataset {path} contains no conversations")
    return convs
