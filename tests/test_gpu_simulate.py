"""Config c5's multi-GPU driver on the device: `simulate.run_sharded` over
B200LM backends with world sizes 1 and 2 writes byte-identical event logs and
reports (the determinism criterion of the reference, test_acceptance.py:231-255).
The two ranks share this box's one GPU (gloo for the work queue and the metric
gather; no data-path collective exists); each rank claims conversations from
the dynamic TCPStore queue, so which rank ran which conversation varies run to
run — the outputs must not."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN  # noqa: F401  (registers the markers)

pytestmark = pytest.mark.gpu

N_CONV = 6


def _setup():
    from paper_2506_15556_b200 import B200LM
    from paper_2506_15556_b200.shapes import small_shape
    from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, synthetic_conversations

    lm = B200LM(small_shape(), seed=2, max_seq=1024, cost_mode="modeled", device=0)
    spec = WorkloadSpec(conversations=N_CONV, mean_words=10.0, max_words=24, system_words=8, seed=3)
    convs = synthetic_conversations(lm.vocab, spec)
    cfg = c5_config(lm.vocab, spec, max_response_tokens=16)
    return lm, convs, cfg


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2506_15556_b200.simulate import run_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lm, convs, cfg = _setup()
    try:
        run_sharded(convs, cfg, lm, out_dir, rank, world)
    finally:
        lm.close()
        dist.destroy_process_group()


def _files(root):
    return {p.relative_to(root): p.read_bytes() for p in sorted(root.rglob("*")) if p.is_file()}


def test_sharded_simulation_on_b200_is_world_size_independent(tmp_path):
    from paper_2506_15556_b200.simulate import run_sharded

    lm, convs, cfg = _setup()
    try:
        rows = run_sharded(convs, cfg, lm, tmp_path / "g1")
    finally:
        lm.close()
    assert len(rows) == sum(len(c.turns) for c in convs)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path / "g2"))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    a, b = _files(tmp_path / "g1"), _files(tmp_path / "g2")
    assert a.keys() == b.keys() and len(a) == len(rows) + 2
    for k in a:
        assert a[k] == b[k], k


def test_annotated_events_carry_device_time_and_bytes(tmp_path):
    """SURVEY §5 tracing keys: with measured cost, every verify / generate_step event's
    gpu_ms is the cost the SimClock was charged, and algorithmic_bytes is the pass's
    SURVEY §8d byte count (0 for a prefix hit)."""
    import json

    from paper_2506_15556_b200 import B200LM
    from paper_2506_15556_b200.shapes import small_shape
    from paper_2506_15556_b200.simulate import run_sharded
    from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, synthetic_conversations

    shape = small_shape()
    lm = B200LM(shape, seed=2, max_seq=1024, cost_mode="measured")
    try:
        spec = WorkloadSpec(conversations=2, mean_words=10.0, max_words=20, system_words=8, seed=5)
        convs = synthetic_conversations(lm.vocab, spec)
        run_sharded(convs, c5_config(lm.vocab, spec, max_response_tokens=12), lm, tmp_path, annotate=True)
    finally:
        lm.close()
    n = 0
    for f in sorted((tmp_path / "events").glob("*.jsonl")):
        for line in f.read_text().splitlines():
            e = json.loads(line)
            if e["kind"] in ("verify", "generate_step"):
                n += 1
                assert abs(e["gpu_ms"] - e["cost_ms"]) < 1e-6
                assert (e["algorithmic_bytes"] > shape.weight_bytes_per_pass()) == (e["rows_computed"] > 0)
    assert n > 0
