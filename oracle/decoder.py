"""ORACLE (test infrastructure only — never imported by the product path).

CPU restatement of the decoder the B200 runtime executes, used as the checker
for `paper_2506_15556_b200` (tests/, `__graft_entry__.smoke()` and the
`cpu_baseline` leg of bench.py only).

The reference has no decoder arithmetic — `LanguageModel.forward` is backed by
a hash n-gram table (`/root/reference/pkg/src/specstream/lm.py:216-243`) — so
the numerics below are **parity unpinned** by any reference test; what the
reference pins is the *contract* this class follows:

* `forward(context, cache)` scores every uncached position, row j scores token
  j+1 given tokens 0..j, and returns a handle over the whole context plus the
  modeled cost `pass_cost(len(ctx) - start)` (`lm.py:182-203`);
* `PrefixViolationError` for a foreign handle, a context that does not extend
  the cached prefix, or a fully cached context (`lm.py:192-199`);
* argmax ties go to the lowest id (`lm.py:134-136`), EOS is id 0 (`text.py:19`).

Model (Llama/Qwen family): x = E[tok]; per layer x += Wo·attn(rope(Wq·n(x)+bq),
rope(Wk·n(x)+bk), Wv·n(x)+bv); x += Wd·(silu(Wg·n(x)) ⊙ Wu·n(x)); logits =
n(x)·Eout^T + bias, with n = RMSNorm (γ = 1). Accumulation is float64. In bf16
mode the GPU's formulation is followed: the GEMM operand is bf16(x) (the
un-normalised residual) and the RMSNorm scale is applied to the GEMM output,
W·(x·rstd) = rstd·(W·x); the same rounding points as the GPU are applied
(weights, bf16(x), q/k/v, attention output, SwiGLU product) so the comparison
measures accumulation-order effects only.
"""

from __future__ import annotations

import numpy as np

from . import specstream
from . import weights as W

_lm = specstream.lm
CacheHandle, LogitsBlock, PrefixViolationError = _lm.CacheHandle, _lm.LogitsBlock, _lm.PrefixViolationError

MODE_F32 = 0
MODE_BF16 = 1


class GeneratorWeights:
    """Weights from the counter-based generator (oracle/weights.py): bit-identical to
    what csrc/init.cu writes into HBM."""

    def __init__(self, seed: int, bf16: bool):
        self.seed, self.bf16 = seed, bf16

    def tensor(self, tid: int, shape) -> np.ndarray:
        return W.tensor(self.seed, tid, shape, self.bf16)

    def rows(self, tid: int, lo: int, hi: int, cols: int) -> np.ndarray:
        w = W.uniform_f32(self.seed, tid, (hi - lo) * cols, first=lo * cols)
        if self.bf16:
            w = W.bf16_bits_to_f32(W.f32_to_bf16_bits(w))
        return w.astype(np.float64).reshape(hi - lo, cols)


class DecoderOracle:
    """Weights + an incremental KV cache for one token sequence.

    `weights` supplies the stored values (default: the generator). With
    `stream=True` nothing is kept resident: every layer's matrices are fetched
    when the layer runs and dropped after it, the embedding is gathered per
    token and the LM head is applied in row blocks, so a full 8B-shape pass
    needs about one layer of float64 weights in host memory (SURVEY §8c,
    the layer-streamed oracle of tests/test_gpu_fullshape.py)."""

    HEAD_BLOCK = 8192

    def __init__(self, shape: dict, seed: int = 0, dtype=np.float64, max_layers: int | None = None,
                 share_layer_weights: bool = False, weights=None, stream: bool = False):
        self.s = dict(shape)
        self.seed = seed
        self.dtype = dtype
        s = self.s
        self.bf16 = s["mode"] == MODE_BF16
        H, V = s["hidden"], s["vocab"]
        self.H, self.V = H, V
        self.nh, self.nkv, self.hd = s["heads"], s["kv_heads"], s["head_dim"]
        self.I = s["intermediate"]
        self.L = s["layers"]
        self.eps = s["rms_eps"]
        self.src = weights if weights is not None else GeneratorWeights(seed, self.bf16)
        self.stream = stream
        self.n_layers_run = self.L if max_layers is None else min(self.L, max_layers)
        self.share = share_layer_weights
        self._head_tid = W.TID_EMBED if s["tied_embeddings"] else W.TID_LM_HEAD
        if not stream:
            self.embed = self.src.tensor(W.TID_EMBED, (V, H)).astype(dtype)
            self.head = self.embed if s["tied_embeddings"] else self.src.tensor(W.TID_LM_HEAD, (V, H)).astype(dtype)
            self.layers = []
            for l in range(self.n_layers_run):
                if share_layer_weights and l > 0:
                    self.layers.append(self.layers[0])
                    continue
                self.layers.append(self._load_layer(l))
            if share_layer_weights:
                # timing-only mode (bench cpu_baseline): every layer streams layer 0's
                # weights, so per-pass memory traffic matches the full model.
                while len(self.layers) < self.L:
                    self.layers.append(self.layers[0])
            self.n_layers_run = len(self.layers)

        self.bias = np.zeros(V, dtype=dtype)
        sigma = 0.02 * np.sqrt(H)
        self.bias[1:4] = np.float32(s.get("term_bias_sigma", 0.0) * sigma)
        self.bias[0] = np.float32(s.get("eos_bias_sigma", 0.0) * sigma)

        half = self.hd // 2
        self.inv_freq = s["rope_theta"] ** (-(np.arange(half, dtype=np.float64) * 2.0) / self.hd)
        self.reset()

    def _load_layer(self, l: int) -> dict:
        H, qd, kvd = self.H, self.nh * self.hd, self.nkv * self.hd

        def t(which, shp):
            return self.src.tensor(W.layer_tid(l, which), shp).astype(self.dtype)

        lay = {"wq": t(W.WQ, (qd, H)), "wk": t(W.WK, (kvd, H)), "wv": t(W.WV, (kvd, H)), "wo": t(W.WO, (H, qd)),
               "wg": t(W.WGATE, (self.I, H)), "wu": t(W.WUP, (self.I, H)), "wd": t(W.WDOWN, (H, self.I))}
        if self.s["qkv_bias"]:
            lay["bq"] = t(W.BQ, (qd,))
            lay["bk"] = t(W.BK, (kvd,))
            lay["bv"] = t(W.BV, (kvd,))
        return lay

    def _layer(self, l: int) -> dict:
        return self._load_layer(l) if self.stream else self.layers[l]

    def _embed(self, tokens) -> np.ndarray:
        if not self.stream:
            return self.embed[np.asarray(tokens, dtype=np.int64)].astype(self.dtype)
        return np.stack([self.src.rows(W.TID_EMBED, int(t), int(t) + 1, self.H)[0] for t in tokens]).astype(self.dtype)

    def _head(self, hn) -> np.ndarray:
        if not self.stream:
            return hn @ self.head.T
        out = np.empty((hn.shape[0], self.V), dtype=self.dtype)
        for lo in range(0, self.V, self.HEAD_BLOCK):
            hi = min(self.V, lo + self.HEAD_BLOCK)
            out[:, lo:hi] = hn @ self.src.rows(self._head_tid, lo, hi, self.H).astype(self.dtype).T
        return out

    # -- state -----------------------------------------------------------------
    def reset(self) -> None:
        self.tokens: list[int] = []
        self.k = [np.zeros((self.nkv, 0, self.hd), dtype=self.dtype) for _ in range(self.n_layers_run)]
        self.v = [np.zeros((self.nkv, 0, self.hd), dtype=self.dtype) for _ in range(self.n_layers_run)]

    def truncate(self, n: int) -> None:
        self.tokens = self.tokens[:n]
        self.k = [k[:, :n] for k in self.k]
        self.v = [v[:, :n] for v in self.v]

    # -- math --------------------------------------------------------------------
    def _r(self, x):
        return W.round_bf16(x).astype(self.dtype) if self.bf16 else x

    def _operand(self, x):
        """(GEMM operand, output scale): fp32 mode normalises first; bf16 mode
        feeds bf16(x) and scales the product by rstd (the GEMM epilogues of csrc/megakernel.cu)."""
        if self.bf16:
            rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + self.eps)
            return self._r(x), rstd
        return self._norm(x), 1.0

    def _norm(self, x):
        ms = np.mean(x * x, axis=-1, keepdims=True)
        return x / np.sqrt(ms + self.eps)

    def _rope(self, x, pos):
        # x [W, n, hd]; rotate-half pairing (i, i + hd/2)
        ang = np.outer(pos.astype(np.float64), self.inv_freq)  # [W, half]
        c = np.cos(ang)[:, None, :].astype(self.dtype)
        s = np.sin(ang)[:, None, :].astype(self.dtype)
        half = self.hd // 2
        a, b = x[..., :half], x[..., half:]
        return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)

    def extend(self, new_tokens: list[int]) -> tuple[np.ndarray, np.ndarray]:
        """Append tokens; return (final normed hidden [W,H], logits [W,V])."""
        n0 = len(self.tokens)
        Wn = len(new_tokens)
        pos = np.arange(n0, n0 + Wn)
        x = self._embed(new_tokens)
        scale = 1.0 / np.sqrt(self.hd)
        grp = self.nh // self.nkv
        for li in range(self.n_layers_run):
            lay = self._layer(li)
            xn, sc_in = self._operand(x)
            q = (xn @ lay["wq"].T) * sc_in
            k = (xn @ lay["wk"].T) * sc_in
            v = (xn @ lay["wv"].T) * sc_in
            if "bq" in lay:
                q = q + lay["bq"]
                k = k + lay["bk"]
                v = v + lay["bv"]
            q = self._r(self._rope(q.reshape(Wn, self.nh, self.hd), pos))
            k = self._r(self._rope(k.reshape(Wn, self.nkv, self.hd), pos))
            v = self._r(v.reshape(Wn, self.nkv, self.hd))
            self.k[li] = np.concatenate([self.k[li], k.transpose(1, 0, 2)], axis=1)
            self.v[li] = np.concatenate([self.v[li], v.transpose(1, 0, 2)], axis=1)
            K, V = self.k[li], self.v[li]  # [nkv, n0+Wn, hd]
            o = np.empty((Wn, self.nh, self.hd), dtype=self.dtype)
            ctx_len = n0 + Wn
            mask = np.arange(ctx_len)[None, :] <= pos[:, None]  # [Wn, ctx]
            for h in range(self.nh):
                kh = h // grp
                sc = (q[:, h, :] @ K[kh].T) * scale
                sc = np.where(mask, sc, -np.inf)
                m = sc.max(axis=1, keepdims=True)
                p = np.exp(sc - m)
                o[:, h, :] = (p @ V[kh]) / p.sum(axis=1, keepdims=True)
            o = self._r(o.reshape(Wn, -1))
            x = x + o @ lay["wo"].T
            xn, sc_in = self._operand(x)
            g = (xn @ lay["wg"].T) * sc_in
            u = (xn @ lay["wu"].T) * sc_in
            a = self._r(g / (1.0 + np.exp(-g)) * u)
            x = x + a @ lay["wd"].T
        self.tokens.extend(int(t) for t in new_tokens)
        hn, sc_in = self._operand(x)
        logits = self._head(hn) * sc_in + self.bias
        return hn, logits

    def ensure(self, context: list[int]) -> None:
        """Make the resident sequence equal `context` (LCP reuse, then extend)."""
        n = 0
        for a, b in zip(self.tokens, context):
            if a != b:
                break
            n += 1
        if n < len(self.tokens):
            self.truncate(n)


class GapRows(np.ndarray):
    """Row array that records the top-2 gap of every row whose argmax is taken.

    `np.argmax(row)` dispatches to `row.argmax()`, so the reference's own
    `argmax_token` (lm.py:134-136) reports exactly the rows it consumed.
    """

    def argmax(self, *args, **kwargs):
        base = self.view(np.ndarray)
        if base.ndim == 1 and getattr(self, "_sink", None) is not None:
            self._sink(top2_gap(base))
        return base.argmax(*args, **kwargs)

    def __array_finalize__(self, obj):
        self._sink = getattr(obj, "_sink", None)


def argmax_lowest(row: np.ndarray) -> int:
    return int(np.argmax(row))


def top2_gap(row: np.ndarray) -> float:
    part = np.partition(row, -2)[-2:]
    return float(part[1] - part[0])


class CpuDecoderLM(_lm.LanguageModel):
    """A reference `LanguageModel` (`lm.py:157-213`) over `DecoderOracle`.

    Rows for already-resident positions are kept from the pass that computed
    them (float64 accumulation makes recomputation immaterial), so `forward`
    costs only the uncached tail, like the B200 backend.
    """

    def __init__(self, shape: dict, vocab, seed: int = 0, latency=None, dtype=np.float64):
        super().__init__(vocab, latency)
        self.model = DecoderOracle(shape, seed, dtype=dtype)
        self._rows: list[np.ndarray] = []  # logits row per resident position
        self.min_gap = np.inf  # smallest top-2 gap over every row handed out
        self.passes = 0

    def _record_gap(self, gap: float) -> None:
        self.min_gap = min(self.min_gap, gap)

    def _materialize(self, context: list[int]) -> None:
        m = self.model
        m.ensure(context)
        self._rows = self._rows[: len(m.tokens)]
        if len(m.tokens) < len(context):
            _, logits = m.extend(context[len(m.tokens):])
            self._rows.extend(logits)

    def forward(self, context, cache=None):
        start = 0
        if cache is not None:
            if cache.backend_id != self._backend_id:
                raise PrefixViolationError("cache handle belongs to a different backend instance")
            if tuple(context[: len(cache.prefix)]) != cache.prefix:
                raise PrefixViolationError("context does not extend the cached prefix")
            start = len(cache.prefix)
        if start >= len(context):
            raise PrefixViolationError("forward pass requires at least one uncached position")
        ctx = tuple(int(t) for t in context)
        self._materialize(list(ctx))
        rows = np.stack(self._rows[start: len(ctx)]).view(GapRows)
        rows._sink = self._record_gap
        self.passes += 1
        return LogitsBlock(rows, start), CacheHandle(ctx, self._backend_id), self.latency.pass_cost(len(ctx) - start)

    def judge_consistency(self, partial_prompt, partial_answer):
        """PredGen self-judgment (verify.py:116-158 calls it): one fresh pass over
        the formatted judge prompt (lm.py:117-131), then the last row's scores of
        "yes" and "no" (lm.py:107-114). Judge text is mapped to ids by the
        vocabulary's `judge_ids` (host tokenisation, identical on both sides)."""
        ids = self.vocab.judge_ids
        toks = ids(_lm.format_judge_prompt(partial_prompt, partial_answer))
        block, _, cost = self.forward(toks)
        row = block.last_row
        return _lm.JudgeResult(yes_score=float(row[ids("yes")[0]]), no_score=float(row[ids("no")[0]])), cost
