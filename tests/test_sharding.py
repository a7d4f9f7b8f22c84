"""Vocab-sharded LM-head argmax (config c4): key packing, and the MAX
all-reduce across ranks on the gloo backend (world size 2, CPU)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_15556_b200.sharding import (allreduce_keys, from_signed, local_keys, pack_keys, shard_range,
                                            to_signed, unpack_ids)


def test_shard_ranges_cover_vocab():
    for V, G in ((32000, 2), (32000, 8), (128256, 4), (151936, 8), (512, 4)):
        got = [shard_range(V, G, r) for r in range(G)]
        assert sum(c for _, c in got) == V
        assert all(b % 128 == 0 for b, _ in got)
        assert [b for b, _ in got] == sorted(b for b, _ in got)


def test_key_order_is_value_then_lowest_id():
    vals = np.array([-3.5, -0.0, 0.0, 1e-30, 2.0, 2.0, np.float32(-1e30)], dtype=np.float32)
    ids = np.array([9, 8, 7, 6, 5, 4, 3])
    k = pack_keys(vals, ids)
    assert unpack_ids(k).tolist() == ids.tolist()
    best = unpack_ids(np.array([k.max()]))[0]
    assert best == 4  # 2.0 ties between ids 5 and 4 -> lowest id
    assert np.array_equal(from_signed(to_signed(k)), k)
    assert np.argsort(to_signed(k), kind="stable").tolist() == np.argsort(k, kind="stable").tolist()


@pytest.mark.parametrize("V,G", [(1000, 2), (4096, 4)])
def test_merged_shards_equal_full_argmax(V, G):
    rng = np.random.default_rng(0)
    logits = rng.standard_normal((17, V)).astype(np.float32)
    logits[3, 10] = logits[3, 900] = 50.0  # exact tie across shards -> lowest id
    keys = []
    for r in range(G):
        b, c = shard_range(V, G, r)
        keys.append(local_keys(logits[:, b:b + c], b))
    merged = np.maximum.reduce(keys)
    assert unpack_ids(merged).tolist() == np.argmax(logits, axis=1).tolist()


def _worker(rank, world, port, V, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    logits = rng.standard_normal((9, V)).astype(np.float32)
    b, c = shard_range(V, world, rank)
    merged = allreduce_keys(local_keys(logits[:, b:b + c], b))
    out[rank] = unpack_ids(merged).tolist() == np.argmax(logits, axis=1).tolist()
    dist.destroy_process_group()


def test_gloo_allreduce_two_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, 3000, out), nprocs=2, join=True)
    assert dict(out) == {0: True, 1: True}
