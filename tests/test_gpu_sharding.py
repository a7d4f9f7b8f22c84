"""Config c4 on one GPU: two vocab-shard instances' packed keys, merged with a
uint64 MAX (what the NCCL all-reduce computes), give exactly the argmax ids of
the unsharded instance — same weights, bit-identical logits per vocab row; and
the NCCL join itself (dlopen, communicator, all-reduce in eager passes and in
the decode graph, unpack) runs with a 1-rank communicator."""

import numpy as np
import pytest

from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import MODE_F32, small_shape
from paper_2506_15556_b200.sharding import shard_range, unpack_ids

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["bf16", "f32"])
def test_two_shards_merge_to_full_argmax(mode):
    shape = small_shape(vocab=4096) if mode == "bf16" else small_shape("s32", mode=MODE_F32, vocab=4096)
    full = B200LM(shape, seed=5, max_seq=512)
    shards = [B200LM(shape, seed=5, max_seq=512, vocab_shards=2, shard_rank=r) for r in range(2)]
    try:
        toks = [int(t) for t in np.random.default_rng(0).integers(4, shape.vocab, 80)]
        want = [int(np.argmax(full.forward(toks)[0].row_for(p))) for p in range(len(toks))]
        keys = []
        for r, lm in enumerate(shards):
            lm.forward(toks)
            keys.append(lm.shard_keys(0, len(toks)))
            b, c = shard_range(shape.vocab, 2, r)
            local = lm.forward(toks)[0]  # prefix hit: shard-local argmax ids
            ids = [int(np.argmax(local.row_for(p))) for p in range(len(toks))]
            assert all(b <= i < b + c for i in ids)
        merged = np.maximum(keys[0], keys[1])
        assert unpack_ids(merged).tolist() == want
        # decode steps on a shard keep producing keys (graph path)
        shards[0].decode_greedy_fused(toks, 6)
    finally:
        for lm in [full, *shards]:
            lm.close()


def _torch_nccl() -> str:
    """The NCCL torch ships (2.28), preferred over the system one."""
    import os

    import nvidia.nccl

    return os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")


@pytest.mark.parametrize("mode", ["bf16", "f32"])
def test_one_rank_nccl_join_equals_local_argmax(mode, monkeypatch):
    """The whole c4 join path on one GPU: a 1-rank NCCL communicator (dlopen'ed
    libnccl, ncclCommInitRank), the uint64 MAX all-reduce after every pass — in
    eager extend passes and inside the captured decode graph — and the unpack
    of the packed (max, lowest id) keys into the argmax ids. With one rank the
    all-reduce is the identity, so ids must equal an instance without it."""
    monkeypatch.setenv("PS_NCCL_LIB", _torch_nccl())
    shape = small_shape(vocab=4096) if mode == "bf16" else small_shape("s32", mode=MODE_F32, vocab=4096)
    plain = B200LM(shape, seed=5, max_seq=512)
    joined = B200LM(shape, seed=5, max_seq=512)
    try:
        joined.init_shard_comm(B200LM.nccl_unique_id(), 0, 1)
        toks = [int(t) for t in np.random.default_rng(1).integers(4, shape.vocab, 90)]
        want = plain.forward(toks)[0]
        got = joined.forward(toks)[0]
        ids = [int(np.argmax(got.row_for(p))) for p in range(len(toks))]
        assert ids == [int(np.argmax(want.row_for(p))) for p in range(len(toks))]
        assert unpack_ids(joined.shard_keys(0, len(toks))).tolist() == ids
        # decode: graph-captured steps with the all-reduce inside
        assert [t for t, _ in joined.decode_greedy_fused(toks, 24)] == \
            [t for t, _ in plain.decode_greedy_fused(toks, 24)]
        d = joined.verify_greedy_detail(toks[:40], toks[40:60])
        assert d == {**plain.verify_greedy_detail(toks[:40], toks[40:60]), "gpu_ms": d["gpu_ms"]}
    finally:
        plain.close()
        joined.close()
