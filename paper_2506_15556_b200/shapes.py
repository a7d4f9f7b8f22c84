"""Decoder shapes for the five BASELINE.json configurations, plus the seeded
weight-generation parameters both the CUDA runtime and the CPU oracle use.

The reference package (`specstream`) has no decoder at all: its backends are a
hash n-gram table and a scripted table (`/root/reference/pkg/src/specstream/lm.py:216-307`).
The configs in BASELINE.json name real model shapes with random init, so the
shapes below are ours, stated here once and passed as plain dicts to both the
C-ABI (`ps_config`, include/predgen_b200.h) and `oracle/decoder.py`.

Weights are not drawn from torch/numpy Gaussians: every element is a pure
function of (seed, tensor id, index) through a splitmix64 hash, turned into a
uniform value with std 0.02 by one IEEE fp32 multiply. The GPU initialises
16 GB in milliseconds and the numpy oracle reproduces the identical bits
(see `oracle/weights.py`, `csrc/init.cu`).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, replace

# dtype modes of the runtime
MODE_F32 = 0   # fp32 storage + fp32 SIMT math: the bit-exact parity mode
MODE_BF16 = 1  # bf16 storage, fp32 accumulate, tcgen05 GEMMs: the speed mode

# Synthetic vocabulary layout (paper_2506_15556_b200/vocab.py): EOS id 0 as in
# the reference (text.py:19), then the three sentence terminators of
# text.py:28.
EOS_ID = 0
TERMINATOR_IDS = (1, 2, 3)  # ".", "?", "!"

WEIGHT_STD = 0.02


@dataclass(frozen=True)
class DecoderShape:
    name: str
    vocab: int
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    intermediate: int
    tied_embeddings: bool
    qkv_bias: bool
    rope_theta: float
    rms_eps: float
    mode: int
    # logit bias added to the terminator / EOS ids, in units of the expected
    # logit standard deviation (WEIGHT_STD * sqrt(hidden)). Random-init
    # weights almost never pick 3 ids out of 128k; the bias (about 0.55 x the
    # expected max of V Gaussians, sqrt(2 ln V)) makes sentences end at a rate
    # comparable to natural text (synthetic vocabulary).
    term_bias_sigma: float = 2.6
    eos_bias_sigma: float = 0.0

    @property
    def q_dim(self) -> int:
        return self.heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def qkv_dim(self) -> int:
        return self.q_dim + 2 * self.kv_dim

    @property
    def logit_sigma(self) -> float:
        return WEIGHT_STD * self.hidden ** 0.5

    def body_params(self) -> int:
        per_layer = self.hidden * self.qkv_dim + self.q_dim * self.hidden
        per_layer += 3 * self.hidden * self.intermediate
        return self.layers * per_layer

    def head_params(self) -> int:
        return self.vocab * self.hidden

    @property
    def elem_bytes(self) -> int:
        return 4 if self.mode == MODE_F32 else 2

    def weight_bytes_per_pass(self) -> int:
        """Weights streamed once per forward pass (body + LM head)."""
        return (self.body_params() + self.head_params()) * self.elem_bytes

    def kv_bytes_per_token(self) -> int:
        return self.layers * 2 * self.kv_dim * self.elem_bytes

    def pass_bytes(self, rows: int, ctx: int) -> int:
        """Algorithmic HBM bytes of one pass computing `rows` new positions of a
        `ctx`-token sequence: weights once, the KV of every position
        the attention reads (cached and new), the new KV written, the embedding rows."""
        kv = self.kv_bytes_per_token()
        return self.weight_bytes_per_pass() + ctx * kv + rows * kv + rows * self.hidden * self.elem_bytes

    def as_dict(self) -> dict:
        return asdict(self)

    def with_mode(self, mode: int) -> "DecoderShape":
        return replace(self, mode=mode)


# c1: "reference's default tiny random-init decoder" — the reference has none,
# so this is ours: Qwen-style QKV bias at toy width, untied (a tied toy model
# degenerates to repeating its input token under greedy decoding).
TINY = DecoderShape("tiny", vocab=512, hidden=256, layers=4, heads=4, kv_heads=2,
                    head_dim=64, intermediate=768, tied_embeddings=False, qkv_bias=True,
                    rope_theta=1e6, rms_eps=1e-6, mode=MODE_F32, term_bias_sigma=1.9)

# c2: Qwen2.5-0.5B shape, fp32 bit-exact mode.
QWEN_05B = DecoderShape("qwen2.5-0.5b", vocab=151936, hidden=896, layers=24, heads=14,
                        kv_heads=2, head_dim=64, intermediate=4864, tied_embeddings=True,
                        qkv_bias=True, rope_theta=1e6, rms_eps=1e-6, mode=MODE_F32)

# c3 / c5: Llama-3-8B shape, bf16.
LLAMA3_8B = DecoderShape("llama-3-8b", vocab=128256, hidden=4096, layers=32, heads=32,
                         kv_heads=8, head_dim=128, intermediate=14336, tied_embeddings=False,
                         qkv_bias=False, rope_theta=5e5, rms_eps=1e-5, mode=MODE_BF16)

# c4: Mistral-7B shape, bf16 (vocab-sharded LM head across ranks).
MISTRAL_7B = DecoderShape("mistral-7b", vocab=32000, hidden=4096, layers=32, heads=32,
                          kv_heads=8, head_dim=128, intermediate=14336, tied_embeddings=False,
                          qkv_bias=False, rope_theta=1e4, rms_eps=1e-5, mode=MODE_BF16)

SHAPES = {s.name: s for s in (TINY, QWEN_05B, LLAMA3_8B, MISTRAL_7B)}


def small_shape(name: str = "small-bf16", mode: int = MODE_BF16, **kw) -> DecoderShape:
    """A cheap shape with the 8B layout (untied, no bias, hd=128, GQA 4) for tests."""
    base = dict(vocab=2048, hidden=512, layers=2, heads=4, kv_heads=1, head_dim=128,
                intermediate=1024, tied_embeddings=False, qkv_bias=False,
                rope_theta=5e5, rms_eps=1e-5, mode=mode)
    base.update(kw)
    return DecoderShape(name, **base)
