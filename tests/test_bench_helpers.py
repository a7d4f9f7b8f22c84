"""bench.py's derived metrics (CPU): the TTFS roofline fraction of SURVEY.md
§8(d) and the conversations/s conversion of per-pass times."""

import importlib.util
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parent.parent
_spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
bench = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(bench)


def ev(kind, t_ms, **payload):
    return SimpleNamespace(kind=kind, t_ms=t_ms, payload=payload)


def turn(events):
    return SimpleNamespace(events=events)


def test_ttfs_roofline_counts_computing_passes_in_the_window():
    events = [
        ev("chunk_received", 10.0, is_final=False, arrival_ms=10.0),
        ev("generate_step", 12.0, cost_ms=2.0),          # before the final chunk: outside
        ev("chunk_received", 20.0, is_final=True, arrival_ms=20.0),
        ev("verify", 24.0, cost_ms=4.0, nfe=1),
        ev("generate_step", 24.0, cost_ms=0.0),          # prefix hit: no floor
        ev("generate_step", 27.0, cost_ms=3.0),
        ev("sentence_emitted", 27.0),
        ev("generate_step", 30.0, cost_ms=3.0),          # after the sentence: outside
    ]
    out = bench.ttfs_roofline([turn(events)], pass_floor_ms=2.5)
    assert out["p50_ttfs_floor_ms"] == pytest.approx(5.0)   # verify + one decode step
    assert out["p50_ttfs_roofline_frac"] == pytest.approx(5.0 / 7.0)


def test_ttfs_roofline_skips_turns_without_a_sentence():
    events = [ev("chunk_received", 0.0, is_final=True, arrival_ms=0.0), ev("generate_step", 3.0, cost_ms=3.0)]
    assert bench.ttfs_roofline([turn(events)], pass_floor_ms=2.0) == {}


def test_conversation_rate_from_pass_times():
    rate = bench.conv_rate_from_passes({"decode_ms": 3.0, "verify_ms": 72.0},
                                       {"decode_rows": 100, "extend_rows": 144})
    # 100 * 3 ms + 144 / 72 * 72 ms = 444 ms per conversation
    assert rate == pytest.approx(1000.0 / 444.0)
