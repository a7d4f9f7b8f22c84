"""Vocab-sharded LM-head argmax (config c4) — host-side mirror of the device keys.

Each of G ranks holds LM-head rows [v_begin, v_begin + count) (contiguous,
128-aligned, `shard_range`). Per row a rank computes its local (max logit,
lowest id) and packs it into one uint64,

    key = orderable(f32 logit) << 32 | (0xFFFFFFFF - id)

so that the numeric MAX over ranks is the global maximum logit and, on an
exact tie, the LOWEST id — the tie rule of `argmax_token`
(`/root/reference/pkg/src/specstream/lm.py:134-136`). On the GPU the keys are
written by the argmax epilogue and MAX-all-reduced with NCCL over NVLink
(`ps_shard_init`, csrc/runtime.cu); these helpers restate the packing for the
host (tests, gloo fallback) and do the all-reduce with torch.distributed
(signed int64: the key is offset by 2**63 so signed order equals unsigned).
"""

from __future__ import annotations

import numpy as np


def shard_range(vocab: int, shards: int, rank: int) -> tuple[int, int]:
    per = -(-((vocab + shards - 1) // shards) // 128) * 128
    begin = min(vocab, per * rank)
    return begin, min(vocab, begin + per) - begin


def orderable(values: np.ndarray) -> np.ndarray:
    u = np.asarray(values, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (u & np.uint64(0x80000000)) != 0
    return np.where(neg, (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000))


def pack_keys(values: np.ndarray, ids: np.ndarray) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint64)
    return (orderable(values) << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - ids)


def unpack_ids(keys: np.ndarray) -> np.ndarray:
    return (np.uint64(0xFFFFFFFF) - (np.asarray(keys, dtype=np.uint64) & np.uint64(0xFFFFFFFF))).astype(np.int64)


def local_keys(logits_shard: np.ndarray, v_begin: int) -> np.ndarray:
    """Keys of a [rows, count] logits block whose column 0 is vocab id v_begin."""
    local = np.argmax(logits_shard, axis=1)  # lowest id on ties
    vals = logits_shard[np.arange(len(local)), local]
    return pack_keys(vals, local + v_begin)


def to_signed(keys: np.ndarray) -> np.ndarray:
    return (np.asarray(keys, dtype=np.uint64) ^ np.uint64(1 << 63)).view(np.int64)


def from_signed(keys: np.ndarray) -> np.ndarray:
    return np.asarray(keys, dtype=np.int64).view(np.uint64) ^ np.uint64(1 << 63)


def allreduce_keys(keys: np.ndarray, group=None) -> np.ndarray:
    """MAX-all-reduce of packed keys with torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(to_signed(keys).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return from_signed(t.numpy())
