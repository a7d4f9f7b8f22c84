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


def test_cpu_schedule_pricing():
    model = {"decode_ms": 50.0, "a_ms": 100.0, "b_ms_per_row": 10.0}
    sched = [bench.summarize_schedule([(30, 1), (31, 1), (40, 72), (41, 1)])]
    assert sched[0] == [4, 75, 3, 1]
    # 3 decode passes * 50 ms + one 72-row pass at 100 ms + 72 * 10 ms
    assert bench.cpu_schedule_ms(model, sched) == pytest.approx(970.0)


def test_both_arms_print_the_same_config():
    args = bench.parse(["--steps", "5", "--warmup", "3", "--conv-per-step", "2"])
    cfg = bench.workload_config(args, world=4)
    assert cfg["timed_conversation_ids"] == [24, 64]
    assert bench.workload_config(bench.parse(["--impl", "reference", "--steps", "5", "--warmup", "3",
                                              "--conv-per-step", "2"]), world=4) == cfg


def test_pass_bytes_match_survey_floors():
    from paper_2506_15556_b200.shapes import LLAMA3_8B, QWEN_05B
    # c3 decode (W=1, C=512) 15.077 GB, c3 verify (W=72, C=128) 15.046 GB,
    # c2 verify (W=72) 1.983 GB
    assert LLAMA3_8B.pass_bytes(1, 513) / 1e9 == pytest.approx(15.077, abs=2e-3)
    assert LLAMA3_8B.pass_bytes(72, 200) / 1e9 == pytest.approx(15.046, abs=2e-3)
    assert QWEN_05B.pass_bytes(72, 200) / 1e9 == pytest.approx(1.983, abs=2e-3)
