"""ctypes binding of the C-ABI library (include/predgen_b200.h).

There is no fallback: if `libpredgen_b200.so` is missing or fails to load,
constructing a B200 backend raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpredgen_b200.so"

PS_OK = 0
PS_ERR_INVALID = -1
PS_ERR_PREFIX = -2
PS_ERR_CUDA = -3
PS_ERR_CAPACITY = -4
PS_ERR_UNSUPPORTED = -5


class NativeLibraryError(RuntimeError):
    """The CUDA runtime library is missing or unusable (no CPU fallback exists)."""


class DeviceError(RuntimeError):
    """A CUDA / driver failure inside the runtime."""


class CapacityError(ValueError):
    """The context does not fit the KV capacity (max_seq)."""


class PsConfig(ctypes.Structure):
    _fields_ = [
        ("vocab", ctypes.c_int32), ("hidden", ctypes.c_int32), ("layers", ctypes.c_int32),
        ("heads", ctypes.c_int32), ("kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("intermediate", ctypes.c_int32),
        ("tied_embeddings", ctypes.c_int32), ("qkv_bias", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float),
        ("term_bias", ctypes.c_float), ("eos_bias", ctypes.c_float),
        ("seed", ctypes.c_uint64),
        ("max_seq", ctypes.c_int32), ("device", ctypes.c_int32),
        ("vocab_shards", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
        ("use_graphs", ctypes.c_int32), ("reserved", ctypes.c_int32 * 7),
    ]


class PsStats(ctypes.Structure):
    _fields_ = [
        ("passes", ctypes.c_int64), ("rows", ctypes.c_int64), ("decode_steps", ctypes.c_int64),
        ("prefix_hits", ctypes.c_int64), ("kv_tokens", ctypes.c_int64), ("kv_pages_used", ctypes.c_int64),
        ("rollbacks", ctypes.c_int64), ("launches", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64), ("weight_bytes", ctypes.c_double), ("gpu_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = ctypes.POINTER
_i32p = _P(ctypes.c_int32)
_f32p = _P(ctypes.c_float)
_f64p = _P(ctypes.c_double)
_h = ctypes.c_void_p

# name -> (restype, argtypes); every symbol the header declares
SIGNATURES = {
    "ps_last_error": (ctypes.c_char_p, []),
    "ps_create": (ctypes.c_int, [_P(PsConfig), _P(ctypes.c_void_p)]),
    "ps_destroy": (None, [_h]),
    "ps_forward": (ctypes.c_int, [_h, _i32p, ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _f32p]),
    "ps_logits_rows": (ctypes.c_int, [_h, ctypes.c_int32, ctypes.c_int32, _f32p]),
    "ps_verify_greedy": (ctypes.c_int, [_h, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, _i32p, _i32p, _i32p,
                                        _f32p]),
    "ps_verify_topk": (ctypes.c_int, [_h, _i32p, ctypes.c_int32, _i32p, ctypes.c_int32, ctypes.c_int32, _i32p,
                                      _i32p, _i32p, _i32p, _f32p]),
    "ps_decode_greedy": (ctypes.c_int, [_h, _i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _i32p, _i32p,
                                        _f32p]),
    "ps_truncate": (ctypes.c_int, [_h, ctypes.c_int32]),
    "ps_resident": (ctypes.c_int, [_h, _i32p, ctypes.c_int32, _i32p]),
    "ps_argmax_rows": (ctypes.c_int, [_h, ctypes.c_int32, ctypes.c_int32, _i32p]),
    "ps_set_terminators": (ctypes.c_int, [_h, _P(ctypes.c_uint8), ctypes.c_int32]),
    "ps_read_weights": (ctypes.c_int, [_h, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _f32p]),
    "ps_get_stats": (ctypes.c_int, [_h, _P(PsStats)]),
    "ps_profile_decode": (ctypes.c_int, [_h, ctypes.c_int32, _f64p, _f64p]),
    "ps_trace": (ctypes.c_int, [_h, _P(ctypes.c_uint64), ctypes.c_int64, _i32p, _i32p]),
    "ps_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "ps_shard_init": (ctypes.c_int, [_h, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]),
    "ps_shard_keys": (ctypes.c_int, [_h, ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_uint64)]),
}

_lib = None


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the runtime library; raise if it is unavailable."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeLibraryError(
            f"{p} is missing: build it with `python -m paper_2506_15556_b200.build` "
            "(there is no CPU fallback for the B200 backend)")
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error(lib) -> str:
    msg = lib.ps_last_error()
    return msg.decode() if msg else ""


def check(lib, rc: int, what: str = "") -> None:
    if rc == PS_OK:
        return
    from ._specstream import specstream  # local import: the ABI check needs no reference

    PrefixViolationError = specstream.lm.PrefixViolationError
    msg = f"{what}: {last_error(lib)}" if what else last_error(lib)
    if rc == PS_ERR_PREFIX:
        raise PrefixViolationError(msg)
    if rc == PS_ERR_INVALID:
        raise ValueError(msg)
    if rc == PS_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == PS_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(msg)


def i32_array(values):
    n = len(values)
    return (ctypes.c_int32 * max(n, 1))(*values)
