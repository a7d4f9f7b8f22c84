"""ORACLE (test infrastructure only — the checker, never the thing measured).

Full-shape bf16 parity of a device backend against the layer-streamed float64
oracle (north_star: "the bf16 mode reports its argmax agreement
rate"). Used by tests/test_gpu_fullshape.py and by bench.py's agreement line.

The device pass is a real verify: a `ctx`-token prompt made resident by one
pass, then ONE `window`-row pass over the candidate, exactly the shape the
bench's verify step runs. The oracle recomputes all `ctx + window` positions
teacher-forced in float64 with the GPU's bf16 rounding points
(oracle/decoder.py), streaming one layer of weights at a time. Its weights are
read back from the device (`read_weights`) — so the comparison is of the
computation, on exactly the values the kernels used — and every tensor's
leading elements are checked bit-identical to the generator spec first.

Tie rule for the agreement: the reference's `argmax_token` (lm.py:134-136),
highest score, lowest id; rows whose oracle top-2 gap is <= tau are ambiguous
under fp32-vs-fp64 accumulation and are reported but not counted.
"""

from __future__ import annotations

import time

import numpy as np

from . import weights as W
from .decoder import DecoderOracle, top2_gap


class DeviceWeights:
    """Stored weights read back from a device backend (duck type: `read_weights`)."""

    SPOT = 1 << 14  # leading elements of every tensor checked against the generator

    def __init__(self, lm, seed: int, bf16: bool):
        self.lm, self.seed, self.bf16 = lm, seed, bf16
        self.checked: set[int] = set()

    def _spot_check(self, tid: int, count: int) -> None:
        if tid in self.checked:
            return
        n = min(count, self.SPOT)
        got = self.lm.read_weights(tid, 0, n)
        want = W.uniform_f32(self.seed, tid, n)
        if self.bf16:
            want = W.bf16_bits_to_f32(W.f32_to_bf16_bits(want))
        if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
            raise AssertionError(f"device weights of tensor {tid} differ from the generator spec")
        self.checked.add(tid)

    def tensor(self, tid: int, shape) -> np.ndarray:
        n = int(np.prod(shape))
        self._spot_check(tid, n)
        return self.lm.read_weights(tid, 0, n).astype(np.float64).reshape(shape)

    def rows(self, tid: int, lo: int, hi: int, cols: int) -> np.ndarray:
        self._spot_check(tid, hi * cols)
        return self.lm.read_weights(tid, lo * cols, (hi - lo) * cols).astype(np.float64).reshape(hi - lo, cols)


def fullshape_agreement(lm, shape, seed: int = 0, ctx: int = 128, window: int = 72, tau: float = 0.02,
                        trial_seed: int = 0) -> dict:
    """One verify-shaped pass on `lm` vs the streamed oracle; returns the agreement record.

    `lm` holds `shape` with weight seed `seed` (it is left with ctx + window tokens resident)."""
    rng = np.random.default_rng(trial_seed)
    prompt = [int(t) for t in rng.integers(4, shape.vocab, ctx)]
    cand = [int(t) for t in rng.integers(4, shape.vocab, window)]
    toks = prompt + cand
    t0 = time.perf_counter()
    lm.truncate(0)
    block0, handle, _ = lm.forward(prompt)
    block, _, _ = lm.forward(toks, handle)                       # one `window`-row pass
    first = ctx - 1                                              # rows a verify consumes
    rows = [block0.row_for(first)] + [block.row_for(p) for p in range(ctx, ctx + window)]
    dev_argmax = [int(np.argmax(r)) for r in rows]               # device argmax (lazy rows)
    got = np.stack([np.asarray(r) for r in rows])                # fp32 logits (ps_logits_rows)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = DecoderOracle(shape.as_dict(), seed=seed, weights=DeviceWeights(lm, seed, shape.mode == 1), stream=True)
    _, want_all = ref.extend(toks)
    want = want_all[first:]
    t_ref = time.perf_counter() - t0
    gaps = np.array([top2_gap(r) for r in want])
    ok = gaps > tau
    g_arg, w_arg = got.argmax(1), want.argmax(1)
    agree = int((g_arg[ok] == w_arg[ok]).sum())
    diff = np.abs(got.astype(np.float64) - want)
    # the lazy rows' device argmax equals the argmax of their materialised values
    consistent = all(d == int(g) for d, g in zip(dev_argmax, g_arg))
    return {"shape": shape.name, "rows": int(len(want)), "rows_gap_gt_tau": int(ok.sum()), "tau": tau,
            "agree": agree, "rate": agree / max(1, int(ok.sum())), "rate_all_rows": float((g_arg == w_arg).mean()),
            "max_abs_logit_diff": float(diff.max()), "mean_abs_logit_diff": float(diff.mean()),
            "logit_std": float(want.std()), "min_gap": float(gaps.min()), "device_argmax_consistent": consistent,
            "mismatch_gaps": [float(x) for x in gaps[g_arg != w_arg]],
            "ctx": ctx, "window": window, "oracle_s": t_ref, "device_s": t_dev}


def merge_records(recs: list[dict]) -> dict:
    """Pool several trials' agreement records."""
    out = dict(recs[0])
    for k in ("rows", "rows_gap_gt_tau", "agree", "oracle_s", "device_s"):
        out[k] = sum(r[k] for r in recs)
    out["rate"] = out["agree"] / max(1, out["rows_gap_gt_tau"])
    out["rate_all_rows"] = sum(r["rate_all_rows"] * r["rows"] for r in recs) / out["rows"]
    out["max_abs_logit_diff"] = max(r["max_abs_logit_diff"] for r in recs)
    out["mean_abs_logit_diff"] = sum(r["mean_abs_logit_diff"] * r["rows"] for r in recs) / out["rows"]
    out["min_gap"] = min(r["min_gap"] for r in recs)
    out["device_argmax_consistent"] = all(r["device_argmax_consistent"] for r in recs)
    out["mismatch_gaps"] = sorted(g for r in recs for g in r["mismatch_gaps"])
    out["trials"] = len(recs)
    return out
