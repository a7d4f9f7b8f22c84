"""Sharded simulation driver: world sizes 1 and 2 (gloo, CPU)
write byte-identical event logs and reports — the analogue of the reference's
determinism criterion (test_acceptance.py:231-255). The backend here is the CPU
decoder oracle (modeled costs, as the reference's LatencyModel)."""

import os
import socket

import torch.multiprocessing as mp

from oracle.decoder import CpuDecoderLM
from paper_2506_15556_b200 import LatencyModel, SyntheticVocabulary
from paper_2506_15556_b200.shapes import TINY
from paper_2506_15556_b200.simulate import ConversationQueue, run_sharded
from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, synthetic_conversations

SPEC = WorkloadSpec(conversations=5, mean_words=8.0, max_words=14, system_words=4, seed=11)


def _setup():
    vocab = SyntheticVocabulary(TINY.vocab)
    convs = synthetic_conversations(vocab, SPEC)
    cfg = c5_config(vocab, SPEC, max_response_tokens=12, chunk_words=4)
    lm = CpuDecoderLM(TINY.as_dict(), vocab, seed=0, latency=LatencyModel())
    return convs, cfg, lm


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    convs, cfg, lm = _setup()
    run_sharded(convs, cfg, lm, out_dir, rank, world)
    dist.destroy_process_group()


def _files(root):
    return {p.relative_to(root): p.read_bytes() for p in sorted(root.rglob("*")) if p.is_file()}


def test_sharded_outputs_identical_for_any_world_size(tmp_path):
    convs, cfg, lm = _setup()
    one = tmp_path / "g1"
    rows = run_sharded(convs, cfg, lm, one)
    assert len(rows) == sum(len(c.turns) for c in convs)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    two = tmp_path / "g2"
    mp.spawn(_worker, args=(2, port, str(two)), nprocs=2, join=True)
    a, b = _files(one), _files(two)
    assert a.keys() == b.keys() and len(a) == len(rows) + 2
    for k in a:
        assert a[k] == b[k], k


def _queue_worker(rank, world, port, out_dir):
    import json

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q = ConversationQueue(37, world)
    got = []
    while (i := q.claim()) is not None:
        got.append(i)
    # a second queue on the same store starts from zero again
    q2 = ConversationQueue(3, world)
    got2 = []
    while (i := q2.claim()) is not None:
        got2.append(i)
    dist.barrier()
    with open(f"{out_dir}/r{rank}.json", "w") as fh:
        json.dump([got, got2], fh)
    dist.destroy_process_group()


def test_dynamic_queue_claims_each_conversation_once(tmp_path):
    import json

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_queue_worker, args=(3, port, str(tmp_path)), nprocs=3, join=True)
    parts = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(3)]
    first = sorted(i for p in parts for i in p[0])
    second = sorted(i for p in parts for i in p[1])
    assert first == list(range(37)) and second == list(range(3))
    for p in parts:  # claims are increasing per rank
        assert p[0] == sorted(p[0])
    local = ConversationQueue(2)
    assert [local.claim(), local.claim(), local.claim()] == [0, 1, None]
