"""Regenerate the candidate from the accepted prefix, keeping first-sentence audio warm.

Same API, pass accounting and event timing as the reference's
`specstream.generate` (`/root/reference/pkg/src/specstream/generate.py`):

* `ar_generate` (`generate.py:129-178`): response = R[:k] (cut at EOS) plus
  greedy tokens; one charged "prefill" pass when no usable cache covers
  seq[:-1] (`_prefill`, `generate.py:118-126`), then one "decode" pass per
  token; the deadline is checked before every pass (`generate.py:164`).
* `jacobi_generate` (`generate.py:181-291`), `SentenceTracker`
  (`generate.py:294-326`), `predictive_generate` (`generate.py:332-416`).

B200 fast path: a backend exposing `decode_greedy_fused(seq, n)` runs up to n
decode steps back to back on the device (CUDA-graph replays, no host round
trip per token) and returns (token, cost_ms) per step. The loop below replays
those steps through the same meter / deadline / callback sequence as the
per-pass loop, so the event log is identical; steps past a deadline (possible
only in measured-cost mode, where costs are not known in advance) are rolled
back on the device with `discard_after` and never charged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .model_api import argmax_token
from .speech import BUFFERED, CANCELED, SYNTHESIZING
from .vocab import EOS_ID, SENTENCE_TERMINATORS


@dataclass(frozen=True)
class GenerationBudget:
    deadline: float | None = None
    max_new_tokens: int = 256

    def __post_init__(self) -> None:
        if self.max_new_tokens < 0:
            raise ValueError("max_new_tokens must be nonnegative")


@dataclass(frozen=True)
class PassRecord:
    at_ms: float
    kind: str  # prefill | decode | jacobi
    new_tokens: int
    uncached: int
    cost_ms: float


@dataclass
class GenerationResult:
    response: list
    complete: bool
    nfe: int
    cost_ms: float
    passes: list = field(default_factory=list)


class _PassMeter:
    def __init__(self, clock) -> None:
        self.clock = clock
        self._local = 0.0
        self.passes: list[PassRecord] = []

    @property
    def now(self) -> float:
        return self.clock.now if self.clock is not None else self._local

    def record(self, kind: str, cost: float, uncached: int, new_tokens: int) -> float:
        if self.clock is None:
            self._local += cost
        else:
            self.clock.charge(cost)
        self.passes.append(PassRecord(self.now, kind, new_tokens, uncached, cost))
        return self.now

    def expired(self, budget) -> bool:
        return bool(budget is not None and budget.deadline is not None and self.now >= budget.deadline)

    def total(self) -> float:
        return sum(p.cost_ms for p in self.passes)


def _cut_at_eos(tokens, eos: int):
    tokens = list(tokens)
    if eos in tokens:
        return tokens[: tokens.index(eos) + 1], True
    return tokens, False


def _matching_cache(cache, seq, limit: int):
    """`cache` shortened to its common prefix with seq[:limit] (None if empty)."""
    if cache is None:
        return None
    n = 0
    for a, b in zip(cache.prefix, seq[:limit]):
        if a != b:
            break
        n += 1
    return cache.truncated(n) if n else None


def _ensure_prefill(lm, seq, cache, meter):
    target = len(seq) - 1
    cache = _matching_cache(cache, seq, target)
    have = 0 if cache is None else cache.cached_prefix_length
    if have < target:
        _, cache, cost = lm.forward(seq[:target], cache)
        meter.record("prefill", cost, target - have, 0)
    return cache


def _steps_before_deadline(now: float, deadline, cost: float, cap: int) -> int:
    """How many fixed-cost passes start before `deadline` (float-exact replay)."""
    if deadline is None:
        return cap
    n = 0
    while n < cap and now < deadline:
        now = now + cost
        n += 1
    return n


def _decode_fused(lm, seq, response, budget, meter, max_new, on_tokens) -> bool:
    """Device-side decode loop; returns True when EOS was produced."""
    eos = lm.eos_id
    remaining = max_new
    while remaining > 0 and not meter.expired(budget):
        deadline = budget.deadline if budget is not None else None
        est = lm.decode_cost_estimate()
        if lm.cost_mode == "modeled":
            n = _steps_before_deadline(meter.now, deadline, est, remaining)
        elif deadline is None:
            n = remaining
        else:
            n = min(remaining, max(1, math.ceil((deadline - meter.now) / max(est, 1e-6)) + 1))
        steps = lm.decode_greedy_fused(seq, n)
        used = 0
        for tok, cost in steps:
            if meter.expired(budget):
                break
            at = meter.record("decode", cost, 1, 1)
            seq.append(tok)
            response.append(tok)
            used += 1
            remaining -= 1
            if on_tokens is not None:
                on_tokens([tok], at)
            if tok == eos:
                lm.discard_after(len(seq))
                return True
        if used < len(steps):
            lm.discard_after(len(seq))
            break
        if not steps:
            break
    return False


def ar_generate(k, context, candidate, lm, cache=None, budget=None, clock=None,
                on_tokens=None) -> GenerationResult:
    if not 0 <= k <= len(candidate):
        raise ValueError("accepted count k out of range")
    if budget is not None and budget.deadline is not None and clock is None:
        raise ValueError("a deadline budget requires a clock")
    meter = _PassMeter(clock)
    base, done = _cut_at_eos(candidate[:k], lm.eos_id)
    max_new = 256 if budget is None else budget.max_new_tokens
    if done or max_new == 0 or meter.expired(budget):
        return GenerationResult(base, done, 0, 0.0, meter.passes)
    seq = list(context) + base
    if not seq:
        raise ValueError("generation requires a nonempty context")
    response = list(base)
    cache = _ensure_prefill(lm, seq, cache, meter)

    if getattr(lm, "decode_greedy_fused", None) is not None:
        complete = _decode_fused(lm, seq, response, budget, meter, max_new, on_tokens)
        return GenerationResult(response, complete, len(meter.passes), meter.total(), meter.passes)

    complete = False
    for _ in range(max_new):
        if meter.expired(budget):
            break
        have = 0 if cache is None else cache.cached_prefix_length
        block, cache, cost = lm.forward(seq, cache)
        at = meter.record("decode", cost, len(seq) - have, 1)
        tok = argmax_token(block.last_row)
        seq.append(tok)
        response.append(tok)
        if on_tokens is not None:
            on_tokens([tok], at)
        if tok == lm.eos_id:
            complete = True
            break
    return GenerationResult(response, complete, len(meter.passes), meter.total(), meter.passes)


def jacobi_generate(k, context, candidate, lm, cache=None, budget=None, clock=None,
                    on_tokens=None) -> GenerationResult:
    """Fixed-point refinement of the rejected window, then greedy tail (generate.py:181-291)."""
    if not 0 <= k <= len(candidate):
        raise ValueError("accepted count k out of range")
    if budget is not None and budget.deadline is not None and clock is None:
        raise ValueError("a deadline budget requires a clock")
    meter = _PassMeter(clock)
    head, done = _cut_at_eos(candidate[:k], lm.eos_id)
    if done:
        return GenerationResult(head, True, 0, 0.0, meter.passes)
    seq_base = list(context) + head
    if not seq_base:
        raise ValueError("generation requires a nonempty context")
    window = list(candidate[k:])
    b = len(seq_base)
    if not window:
        return ar_generate(k, context, candidate, lm, cache, budget, clock, on_tokens)
    if meter.expired(budget):
        return GenerationResult(head + window, False, 0, 0.0, meter.passes)

    iter_cache = _ensure_prefill(lm, seq_base, cache, meter)
    confirmed, converged, complete, rounds = 0, False, False, 0
    last = None
    while not converged:
        if meter.expired(budget):
            break
        if rounds > len(window):
            raise RuntimeError("window failed to converge; backend is not deterministic")
        have = 0 if iter_cache is None else iter_cache.cached_prefix_length
        block, last, cost = lm.forward(seq_base + window, iter_cache)
        rounds += 1
        at = meter.record("jacobi", cost, b + len(window) - have, 0)
        preds = [argmax_token(block.row_for(b - 1 + i)) for i in range(len(window))]
        agree = 0
        while agree < len(window) and window[agree] == preds[agree]:
            agree += 1
        if agree == len(window):
            fresh = window[confirmed:]
            confirmed = len(window)
            converged = True
        else:
            upto = min(len(window), agree + 1)
            window = preds
            fresh = window[confirmed:upto]
            confirmed = upto
            converged = confirmed == len(window)
        if fresh and on_tokens is not None:
            on_tokens(fresh, at)
        if lm.eos_id in fresh:
            complete = True
            break
        iter_cache = last.truncated(b - 1) if b >= 1 else None

    response = head + window
    if complete:
        response, complete = _cut_at_eos(response, lm.eos_id)
        return GenerationResult(response, complete, len(meter.passes), meter.total(), meter.passes)
    if not converged:
        return GenerationResult(response, False, len(meter.passes), meter.total(), meter.passes)
    tail = ar_generate(len(response), context, response, lm, cache=last, budget=budget,
                       clock=clock, on_tokens=on_tokens)
    return GenerationResult(tail.response, tail.complete, len(meter.passes) + tail.nfe,
                            meter.total() + tail.cost_ms, meter.passes + tail.passes)


class SentenceTracker:
    """Fires `on_sentence(index, text, at, tokens)` per completed sentence."""

    def __init__(self, vocab, on_sentence) -> None:
        self.vocab = vocab
        self.on_sentence = on_sentence
        self.tokens: list[int] = []
        self._scanned = 0
        self._start = 0
        self.count = 0

    def _emit(self, end: int, at: float) -> None:
        seg = self.tokens[self._start:end]
        self.on_sentence(self.count, self.vocab.detokenize(seg), at, seg)
        self.count += 1
        self._start = end

    def feed(self, tokens, at: float) -> None:
        self.tokens.extend(t for t in tokens if t != EOS_ID)
        while self._scanned < len(self.tokens):
            self._scanned += 1
            if self.vocab.surface(self.tokens[self._scanned - 1]) in SENTENCE_TERMINATORS:
                self._emit(self._scanned, at)

    def flush_fragment(self, at: float) -> None:
        if self._start < len(self.tokens):
            self._emit(len(self.tokens), at)


GENERATORS = {"ar": ar_generate, "jacobi": jacobi_generate}


def predictive_generate(k, context, candidate, lm, tts, clock, generator="ar", deadline=None,
                        max_response_tokens=256, current_job=None, final_round=False,
                        on_sentence=None):
    if generator not in GENERATORS:
        raise ValueError(f"unknown generator {generator!r}")
    state = {"job": current_job}

    def reconcile(text: str, at: float) -> None:
        if tts is None:
            return
        job = state["job"]
        if job is not None and job.state != CANCELED and job.text == text:
            if final_round and job.state == BUFFERED:
                tts.resume(job, at)
            elif final_round and job.state == SYNTHESIZING:
                tts.resume_when_buffered(job)
            return
        if job is not None and job.live:
            tts.cancel(job)
        state["job"] = (tts.synthesize_streaming if final_round else tts.synthesize_buffer)(text, at)

    def on_complete_sentence(idx, text, at, tokens) -> None:
        if idx == 0:
            reconcile(text, at)
        elif final_round and tts is not None:
            tts.synthesize_streaming(text, at)
        if on_sentence is not None:
            on_sentence(idx, text, at, tokens)

    tracker = SentenceTracker(lm.vocab, on_complete_sentence)
    head, head_done = _cut_at_eos(candidate[:k], lm.eos_id)
    tracker.feed(head, clock.now)
    if head_done:
        result = GenerationResult(head, True, 0, 0.0, [])
    else:
        spent = len(candidate) if generator == "jacobi" else len(head)
        budget = GenerationBudget(deadline, max(0, max_response_tokens - spent))
        result = GENERATORS[generator](k, context, candidate, lm, budget=budget, clock=clock,
                                       on_tokens=tracker.feed)
    if result.complete or final_round:
        tracker.flush_fragment(clock.now)
    if final_round and tracker.count == 0:
        job = state["job"]
        if job is not None and job.live:
            tts.cancel(job)
        state["job"] = None
    return result, state["job"]
