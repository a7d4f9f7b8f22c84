"""`B200LM`: the reference's `LanguageModel` surface backed by the CUDA runtime.

A subclass of `specstream.lm.LanguageModel` (`/root/reference/pkg/src/specstream/
lm.py:157-213`), so the reference's own `verify_greedy`, `verify_topk`,
`verify_reflection`, `ar_generate`, `jacobi_generate`, `greedy_decode`,
`run_turn` and `run_baseline` run on it unchanged (tests/test_gpu_dropin.py).

Semantics kept from the reference:

* `forward(context, cache)` returns rows for every position not covered by
  `cache`, row j scoring token j+1; a handle over the whole context; and the
  cost. Handle checks raise `PrefixViolationError` (`lm.py:192-199`).
* cache transparency (`SPEC.md:158`): rows are bit-identical whatever the
  cache, because the device keeps one resident sequence, reuses its longest
  common prefix, and every kernel is batch-invariant. A
  `_prefill` over a prefix the verify pass left resident costs nothing, and
  the first decode after a verify reads the correction token the verify pass
  already scored.

Cost modes: "modeled" charges the reference's `LatencyModel` exactly
(`lm.py:56-57`), so decisions and event logs are comparable bit-for-bit with
the CPU oracle; "measured" charges the CUDA-event milliseconds of the work
the device actually did (a prefix hit costs 0).

Rows are lazy: a `LazyRow` knows its argmax (computed on the device by the
LM-head phase) and materialises the fp32 logits only when something other
than `np.argmax` touches it.

Fused entry points (`verify_greedy_fused`, `verify_topk_fused`,
`decode_greedy_fused`) bind the one-call C-ABI paths; `fused.py` plugs the
verify ones into the reference's loop.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from ._specstream import specstream
from .shapes import MODE_BF16, DecoderShape
from .vocab import SyntheticVocabulary, terminator_mask

_lm = specstream.lm
CacheHandle = _lm.CacheHandle
LogitsBlock = _lm.LogitsBlock
LatencyModel = _lm.LatencyModel
JudgeResult = _lm.JudgeResult
JudgeUnsupportedError = _lm.JudgeUnsupportedError
PrefixViolationError = _lm.PrefixViolationError


def decoder_judge(lm, partial_prompt: str, partial_answer: str):
    """PredGen's self-consistency judge for a decoder backend: one fresh pass
    over the reference's formatted judge prompt (`format_judge_prompt`,
    lm.py:117-131), then the exact last row's scores of "yes" and "no"
    (`JudgeResult.consistent` iff yes > no, lm.py:107-114). Returns
    (JudgeResult, cost of the pass)."""
    ids = lm.vocab.judge_ids
    toks = ids(_lm.format_judge_prompt(partial_prompt, partial_answer))
    block, _, cost = lm.forward(toks)
    row = block.last_row
    yes, no = ids("yes")[0], ids("no")[0]
    return JudgeResult(yes_score=float(row[yes]), no_score=float(row[no])), cost


def ps_config(shape: DecoderShape, seed: int = 0, max_seq: int = 2048, device: int = 0, vocab_shards: int = 1,
              shard_rank: int = 0, use_graphs: bool = True) -> _native.PsConfig:
    """The `ps_config` (include/predgen_b200.h) of a decoder shape: the logit biases
    of the terminator / EOS ids are given in units of the logit std 0.02*sqrt(H)."""
    cfg = _native.PsConfig()
    sigma = 0.02 * math.sqrt(shape.hidden)
    for name in ("vocab", "hidden", "layers", "heads", "kv_heads", "head_dim", "intermediate", "mode"):
        setattr(cfg, name, int(getattr(shape, name)))
    cfg.tied_embeddings = int(shape.tied_embeddings)
    cfg.qkv_bias = int(shape.qkv_bias)
    cfg.rope_theta = shape.rope_theta
    cfg.rms_eps = shape.rms_eps
    cfg.term_bias = float(np.float32(shape.term_bias_sigma * sigma))
    cfg.eos_bias = float(np.float32(shape.eos_bias_sigma * sigma))
    cfg.seed = seed
    cfg.max_seq = max_seq
    cfg.device = device
    cfg.vocab_shards = vocab_shards
    cfg.shard_rank = shard_rank
    cfg.use_graphs = int(use_graphs)
    return cfg


class LazyRow:
    """One logits row: argmax known, fp32 values fetched from the device on demand."""

    __slots__ = ("_lm", "_ctx", "_pos", "_argmax", "_values")

    def __init__(self, lm: "B200LM", ctx: tuple, pos: int, argmax: int) -> None:
        self._lm = lm
        self._ctx = ctx
        self._pos = pos
        self._argmax = argmax
        self._values = None

    # np.argmax(row) dispatches here (numpy's _wrapfunc) — no transfer needed.
    def argmax(self, axis=None, out=None, **kw):
        if axis not in (None, 0, -1) or out is not None or kw:
            return np.asarray(self).argmax(axis=axis, out=out, **kw)
        return np.intp(self._argmax)

    def _materialize(self) -> np.ndarray:
        if self._values is None:
            self._values = self._lm._row_values(self._ctx, self._pos)
        return self._values

    def __array__(self, dtype=None, copy=None):
        v = self._materialize()
        return v if dtype is None else v.astype(dtype)

    def __len__(self) -> int:
        return self._lm.vocab_size

    def __getitem__(self, idx):
        return self._materialize()[idx]

    def __iter__(self):
        return iter(self._materialize())

    def __getattr__(self, name):
        return getattr(self._materialize(), name)


class _LazyRows:
    def __init__(self, lm: "B200LM", ctx: tuple, first: int, argmax: list[int]) -> None:
        self._rows = [LazyRow(lm, ctx, first + i, a) for i, a in enumerate(argmax)]

    def __len__(self) -> int:
        return len(self._rows)

    def __getitem__(self, i):
        return self._rows[i]

    def __iter__(self):
        return iter(self._rows)

    def __array__(self, dtype=None, copy=None):
        arr = np.stack([np.asarray(r) for r in self._rows])
        return arr if dtype is None else arr.astype(dtype)


class B200LM(_lm.LanguageModel):
    def __init__(self, shape: DecoderShape, vocab=None, seed: int = 0, latency: LatencyModel | None = None,
                 cost_mode: str = "modeled", device: int = 0, max_seq: int = 2048, use_graphs: bool = True,
                 vocab_shards: int = 1, shard_rank: int = 0) -> None:
        vocab = SyntheticVocabulary(shape.vocab) if vocab is None else vocab
        if len(vocab) != shape.vocab:
            raise ValueError(f"vocabulary has {len(vocab)} ids, decoder shape expects {shape.vocab}")
        if cost_mode not in ("modeled", "measured"):
            raise ValueError("cost_mode must be 'modeled' or 'measured'")
        super().__init__(vocab, latency)
        self.shape = shape
        self.cost_mode = cost_mode
        self._lib = _native.load()
        self._h = ctypes.c_void_p()
        cfg = ps_config(shape, seed, max_seq=max_seq, device=device, vocab_shards=vocab_shards,
                        shard_rank=shard_rank, use_graphs=use_graphs)
        self.seed = seed
        self.max_seq = max_seq
        self.vocab_shards = vocab_shards
        self.shard_rank = shard_rank
        _native.check(self._lib, self._lib.ps_create(ctypes.byref(cfg), ctypes.byref(self._h)), "ps_create")
        mask = terminator_mask(vocab)
        buf = (ctypes.c_uint8 * len(mask)).from_buffer_copy(mask)
        self._call("ps_set_terminators", buf, len(mask))
        self.last_verify_ms = 0.0
        self.verify_ms: list[float] = []
        self.decode_ms: list[float] = []   # device ms of every 1-row pass
        self.extend_ms: list[tuple] = []   # (rows, device ms) of every wider pass
        # (context length, rows computed, device ms) of every pass, when a caller sets it to a list
        self.schedule: list | None = None
        # the same for every call (a prefix hit logs 0 rows): report.annotate_events joins it
        # with the reference's verify / generate_step events
        self.call_log: list | None = None

    # -- plumbing -----------------------------------------------------------------
    def _call(self, name: str, *args) -> None:
        if not self._h:
            raise RuntimeError("backend is closed")
        _native.check(self._lib, getattr(self._lib, name)(self._h, *args), name)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.ps_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        st = _native.PsStats()
        self._call("ps_get_stats", ctypes.byref(st))
        return st.as_dict()

    def _rows_computed(self) -> int:
        st = _native.PsStats()
        self._call("ps_get_stats", ctypes.byref(st))
        return int(st.rows)

    def _note_verify_pass(self, n_ctx: int, rows_before: int, ms: float) -> None:
        if self.schedule is not None or self.call_log is not None:
            rows = self._rows_computed() - rows_before
            if rows and self.schedule is not None:
                self.schedule.append((n_ctx, rows, ms))
            if self.call_log is not None:
                self.call_log.append((n_ctx, rows, ms))

    def resident(self) -> list[int]:
        n = ctypes.c_int32()
        buf = (ctypes.c_int32 * self.max_seq)()
        self._call("ps_resident", buf, self.max_seq, ctypes.byref(n))
        return list(buf[: n.value])

    def read_weights(self, tid: int, offset: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        self._call("ps_read_weights", tid, offset, count, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        return out

    def _cost(self, uncached: int, ms: float) -> float:
        return self.latency.pass_cost(uncached) if self.cost_mode == "modeled" else float(ms)

    # -- vocab sharding (config c4) ------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _native.load()
        buf = ctypes.create_string_buffer(128)
        _native.check(lib, lib.ps_nccl_unique_id(buf), "ps_nccl_unique_id")
        return buf.raw

    def init_shard_comm(self, unique_id: bytes, rank: int, world: int) -> None:
        buf = ctypes.create_string_buffer(unique_id, 128)
        self._call("ps_shard_init", buf, rank, world)

    def shard_keys(self, first: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self._call("ps_shard_keys", first, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        return out

    def _row_values(self, ctx: tuple, pos: int) -> np.ndarray:
        """fp32 logits of position `pos` given ctx[:pos+1] (re-established if rolled back)."""
        if self.vocab_shards > 1:
            raise NotImplementedError("logits rows of a vocab-sharded instance cover one shard only")
        res = self.resident()
        if len(res) <= pos or tuple(res[: pos + 1]) != tuple(ctx[: pos + 1]):
            # batch invariance makes the recomputed row bit-identical
            self._sync(list(ctx[: pos + 1]), pos + 1)
        out = np.empty(self.vocab_size, dtype=np.float32)
        self._call("ps_logits_rows", pos, 1, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        return out

    def _sync(self, context: list[int], row_from: int):
        n = len(context)
        toks = _native.i32_array(context)
        am = (ctypes.c_int32 * max(n - row_from, 1))()
        computed = ctypes.c_int32()
        ms = ctypes.c_float()
        self._call("ps_forward", toks, n, row_from, am, ctypes.byref(computed), ctypes.byref(ms))
        return list(am[: n - row_from]), computed.value, ms.value

    # -- LanguageModel surface ---------------------------------------------------------
    def _cached_start(self, context, cache) -> int:
        """The reference's handle rules (lm.py:190-199); the first uncached position."""
        start = 0
        if cache is not None:
            if cache.backend_id != self._backend_id:
                raise PrefixViolationError("cache handle belongs to a different backend instance")
            if tuple(context[: len(cache.prefix)]) != tuple(cache.prefix):
                raise PrefixViolationError("context does not extend the cached prefix")
            start = len(cache.prefix)
        if start >= len(context):
            raise PrefixViolationError("forward pass requires at least one uncached position")
        return start

    def forward(self, context, cache=None):
        start = self._cached_start(context, cache)
        ctx = tuple(int(t) for t in context)
        argmax, computed, ms = self._sync(list(ctx), start)
        if computed and self.schedule is not None:
            self.schedule.append((len(ctx), computed, ms))
        if self.call_log is not None:
            self.call_log.append((len(ctx), computed, ms))
        if computed == 1:
            self.decode_ms.append(ms)
        elif computed > 1:
            self.extend_ms.append((computed, ms))
        rows = _LazyRows(self, ctx, start, argmax)
        return LogitsBlock(rows, start), CacheHandle(ctx, self._backend_id), self._cost(len(ctx) - start, ms)

    def judge_consistency(self, partial_prompt: str, partial_answer: str):
        """Self-consistency judge (verify_reflection, verify.py:116-158): a pass over the
        judge prompt on the device, yes/no scores from the exact fp32 last row."""
        if self.vocab_shards > 1:
            raise JudgeUnsupportedError("the judge needs the full LM-head row (vocab-sharded instance)")
        return decoder_judge(self, partial_prompt, partial_answer)

    # -- fused one-call paths (C-ABI; fused.py plugs the verifiers into the loop) -------
    def verify_greedy_fused(self, prompt, candidate):
        """One fused pass: (k, handle over prompt ++ candidate, cost)."""
        if not prompt:
            raise ValueError("verification requires a nonempty prompt context")
        p = _native.i32_array(prompt)
        c = _native.i32_array(candidate)
        k = ctypes.c_int32()
        term = ctypes.c_int32()
        ms = ctypes.c_float()
        rows0 = self._rows_computed() if self.schedule is not None or self.call_log is not None else 0
        self._call("ps_verify_greedy", p, len(prompt), c, len(candidate), ctypes.byref(k), ctypes.byref(term),
                   None, ctypes.byref(ms))
        self._note_verify_pass(len(prompt) + len(candidate), rows0, ms.value)
        self.last_verify_ms = ms.value
        self.verify_ms.append(ms.value)
        seq = tuple(int(t) for t in prompt) + tuple(int(t) for t in candidate)
        return k.value, CacheHandle(seq, self._backend_id), self._cost(len(seq), ms.value)

    def verify_greedy_detail(self, prompt, candidate) -> dict:
        """Fused verify returning every device output (tests / diagnostics)."""
        p = _native.i32_array(prompt)
        c = _native.i32_array(candidate)
        k, term, ms = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_float()
        am = (ctypes.c_int32 * (len(candidate) + 1))()
        self._call("ps_verify_greedy", p, len(prompt), c, len(candidate), ctypes.byref(k), ctypes.byref(term),
                   am, ctypes.byref(ms))
        return {"k": k.value, "first_term": term.value, "argmax": list(am), "gpu_ms": ms.value}

    def verify_topk_fused(self, prompt, candidate, topk: int):
        """Fused top-k verify (rank counting on the device): (k, handle over prompt ++ candidate, cost)."""
        if not prompt:
            raise ValueError("verification requires a nonempty prompt context")
        rows0 = self._rows_computed() if self.schedule is not None or self.call_log is not None else 0
        d = self.verify_topk_detail(prompt, candidate, topk)
        self._note_verify_pass(len(prompt) + len(candidate), rows0, d["gpu_ms"])
        self.last_verify_ms = d["gpu_ms"]
        self.verify_ms.append(d["gpu_ms"])
        seq = tuple(int(t) for t in prompt) + tuple(int(t) for t in candidate)
        return d["k"], CacheHandle(seq, self._backend_id), self._cost(len(seq), d["gpu_ms"])

    def verify_topk_detail(self, prompt, candidate, topk: int) -> dict:
        """Fused top-k verify returning every device output, ranks included."""
        p = _native.i32_array(prompt)
        c = _native.i32_array(candidate)
        k, term, ms = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_float()
        am = (ctypes.c_int32 * (len(candidate) + 1))()
        rk = (ctypes.c_int32 * max(1, len(candidate)))()
        self._call("ps_verify_topk", p, len(prompt), c, len(candidate), int(topk), ctypes.byref(k),
                   ctypes.byref(term), am, rk, ctypes.byref(ms))
        return {"k": k.value, "first_term": term.value, "argmax": list(am), "rank": list(rk)[: len(candidate)],
                "gpu_ms": ms.value}

    def decode_greedy_fused(self, seq, n: int):
        """Up to n greedy tokens continuing `seq`, stopping after EOS: [(token, cost_ms)].
        One C-ABI call: the first token is the resident row's argmax, the rest are
        graph-replayed 1-row steps chained on the device (no host round trip per token).
        Same tokens as the reference's `greedy_decode` (lm.py:350-382)."""
        if n <= 0:
            return []
        s = _native.i32_array(seq)
        out = (ctypes.c_int32 * n)()
        ms = (ctypes.c_float * n)()
        got = ctypes.c_int32()
        self._call("ps_decode_greedy", s, len(seq), n, 1, out, ctypes.byref(got), ms)
        steps = []
        for i in range(got.value):
            cost = self._cost(1, ms[i])
            steps.append((int(out[i]), cost))
            if i > 0 or ms[i] > 0:
                self.decode_ms.append(ms[i])
        return steps

    def truncate(self, n: int) -> None:
        """Roll the resident sequence back to n tokens (ps_truncate)."""
        self._call("ps_truncate", int(n))

    def profile_decode(self, steps: int = 4) -> dict:
        ms = (ctypes.c_double * 8)()
        by = (ctypes.c_double * 8)()
        self._call("ps_profile_decode", steps, ms, by)
        names = ["embed_norms", "qkv_gemm", "attention", "o_gemm", "gate_up_gemm", "down_gemm", "lm_head",
                 "whole_pass"]
        return {n: {"ms": ms[i], "bytes": by[i]} for i, n in enumerate(names)}

    @property
    def is_bf16(self) -> bool:
        return self.shape.mode == MODE_BF16
