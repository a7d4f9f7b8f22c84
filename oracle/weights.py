"""ORACLE (test infrastructure only — never imported by the product path).

Counter-based weight generator, restated in numpy so that the CPU oracle holds
bit-identical weights to the ones `csrc/init.cu` writes into HBM.

The reference has no decoder (its backends are `NGramLM`, a PRNG keyed by the
context window, `/root/reference/pkg/src/specstream/lm.py:236-243`, and the
scripted table, `lm.py:262-297`), so this generator is ours; the spec below is
the one DESIGN.md states and the CUDA kernel implements:

    mix(z)   = splitmix64 finaliser
    key      = mix(seed*G + tid*C + D)
    h(i)     = mix(key + (i+1)*G)                (uint64, wrapping)
    u        = h >> 41                           in [0, 2^23)
    w        = fp32(u - 2^22) * fp32(std*sqrt(3)/2^22)   (one IEEE fp32 multiply)
    bf16(w)  = round-to-nearest-even of the fp32 bits

Tensor ids: embed 1, untied LM head 2, layer l: 64+16l + {wq 0, wk 1, wv 2,
wo 3, w_gate 4, w_up 5, w_down 6, bq 7, bk 8, bv 9}. Elements are indexed
row-major in the [out_features, in_features] layout.
"""

from __future__ import annotations

import numpy as np

G = np.uint64(0x9E3779B97F4A7C15)
C = np.uint64(0xD1B54A32D192ED03)
D = np.uint64(0x632BE59BD9B4E019)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

TID_EMBED = 1
TID_LM_HEAD = 2
WQ, WK, WV, WO, WGATE, WUP, WDOWN, BQ, BK, BV = range(10)


def layer_tid(layer: int, which: int) -> int:
    return 64 + 16 * layer + which


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, tid: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.array([np.uint64(seed) * G + np.uint64(tid) * C + D], dtype=np.uint64)
        return _mix(z)[0]


def scale_f32(std: float) -> np.float32:
    return np.float32(std * np.sqrt(3.0) / float(1 << 22))


def uniform_f32(seed: int, tid: int, count: int, std: float = 0.02,
                chunk: int = 1 << 24, first: int = 0) -> np.ndarray:
    """`count` fp32 weights of tensor `tid` from element `first` on, identical to init.cu's output."""
    key = _key(seed, tid)
    scale = scale_f32(std)
    out = np.empty(count, dtype=np.float32)
    with np.errstate(over="ignore"):
        for lo in range(0, count, chunk):
            hi = min(count, lo + chunk)
            idx = np.arange(first + lo + 1, first + hi + 1, dtype=np.uint64)
            h = _mix(key + idx * G)
            u = (h >> np.uint64(41)).astype(np.int64) - (1 << 22)
            out[lo:hi] = u.astype(np.float32) * scale
    return out


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))
    return ((bits + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp64/fp32 -> fp32 -> bf16 (RNE) -> back to float64."""
    return bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(x, dtype=np.float32))).astype(np.float64)


def tensor(seed: int, tid: int, shape: tuple[int, ...], bf16: bool, std: float = 0.02) -> np.ndarray:
    """The stored weight values as float64 (bf16-rounded when the model is bf16)."""
    n = int(np.prod(shape))
    w = uniform_f32(seed, tid, n, std)
    if bf16:
        return bf16_bits_to_f32(f32_to_bf16_bits(w)).astype(np.float64).reshape(shape)
    return w.astype(np.float64).reshape(shape)
