"""How many leading candidate tokens survive a newer prompt.

API and accounting of the reference's `specstream.verify`
(`/root/reference/pkg/src/specstream/verify.py`):

* `verify_greedy(P, R, lm, clock)` — one fresh pass over P ++ R; k = longest
  prefix of R whose token equals the argmax of the row before it (row
  `len(P)+i-1`, `verify.py:43-55`); `first_sentence_accepted` iff the first
  terminator of R lies inside R[:k] (`verify.py:58-60`); cache covers P ++
  R[:k]; nfe 1; uncached = len(P)+len(R) (`verify.py:63-97`).
* `verify_topk`, `verify_reflection`, `make_verifier` (`verify.py:100-175`).

B200 fast paths: when the backend exposes `verify_greedy_fused(P, R)` (the
`ps_verify_greedy` C-ABI call), the pass, the per-row argmax, the compare and
the first-mismatch scan all run on the device and only k comes back; with
`verify_topk_fused(P, R, k)` (`ps_verify_topk`) the candidate ranks are
counted on the device from the pass's own logits. Either outcome is
field-for-field what the generic path computes.
"""

from __future__ import annotations

from dataclasses import dataclass

from .model_api import JudgeUnsupportedError, argmax_token, topk_tokens
from .vocab import first_sentence


@dataclass
class VerifierOutcome:
    accepted_count: int
    first_sentence_accepted: bool
    cache: object
    cost_ms: float
    nfe: int
    uncached_positions: int
    judge_fallback: str | None = None


def _charge(clock, cost: float) -> None:
    if clock is not None:
        clock.charge(cost)


def _leading_matches(prompt, candidate, block, accepts) -> int:
    base = len(prompt) - 1
    for i, tok in enumerate(candidate):
        if not accepts(block.row_for(base + i), tok):
            return i
    return len(candidate)


def _first_sentence_inside(candidate, k: int, vocab) -> bool:
    span = first_sentence(candidate, vocab)
    return span is not None and span.end <= k


def _outcome(prompt, candidate, k, handle, cost, vocab) -> VerifierOutcome:
    return VerifierOutcome(
        accepted_count=k,
        first_sentence_accepted=_first_sentence_inside(candidate, k, vocab),
        cache=handle.truncated(len(prompt) + k),
        cost_ms=cost,
        nfe=1,
        uncached_positions=len(prompt) + len(candidate),
    )


def _verify_with_rule(prompt, candidate, lm, accepts, clock) -> VerifierOutcome:
    if not prompt:
        raise ValueError("verification requires a nonempty prompt context")
    block, handle, cost = lm.forward(list(prompt) + list(candidate))
    _charge(clock, cost)
    k = _leading_matches(prompt, candidate, block, accepts) if candidate else 0
    return _outcome(prompt, candidate, k, handle, cost, lm.vocab)


def verify_greedy(prompt, candidate, lm, clock=None) -> VerifierOutcome:
    fused = getattr(lm, "verify_greedy_fused", None)
    if fused is None:
        return _verify_with_rule(prompt, candidate, lm,
                                 lambda row, tok: tok == argmax_token(row), clock)
    if not prompt:
        raise ValueError("verification requires a nonempty prompt context")
    k, handle, cost = fused(list(prompt), list(candidate))
    _charge(clock, cost)
    return _outcome(prompt, candidate, k, handle, cost, lm.vocab)


def verify_topk(prompt, candidate, lm, k: int, clock=None) -> VerifierOutcome:
    if k < 1:
        raise ValueError("top-k verification requires k >= 1")
    fused = getattr(lm, "verify_topk_fused", None)
    if fused is None or getattr(lm, "vocab_shards", 1) > 1:
        return _verify_with_rule(prompt, candidate, lm,
                                 lambda row, tok: tok in topk_tokens(row, k), clock)
    if not prompt:
        raise ValueError("verification requires a nonempty prompt context")
    acc, handle, cost = fused(list(prompt), list(candidate), k)
    _charge(clock, cost)
    return _outcome(prompt, candidate, acc, handle, cost, lm.vocab)


def verify_reflection(prompt, candidate, lm, clock=None, judge_prompt_text=None) -> VerifierOutcome:
    span = first_sentence(candidate, lm.vocab)
    if span is None:
        return verify_greedy(prompt, candidate, lm, clock)
    prompt_text = lm.vocab.detokenize(prompt) if judge_prompt_text is None else judge_prompt_text
    sentence = lm.vocab.detokenize(candidate[: span.end])
    try:
        verdict, judge_cost = lm.judge_consistency(prompt_text, sentence)
    except JudgeUnsupportedError:
        out = verify_greedy(prompt, candidate, lm, clock)
        out.judge_fallback = "judge_unsupported"
        return out
    _charge(clock, judge_cost)
    if verdict.consistent:
        return VerifierOutcome(accepted_count=span.end, first_sentence_accepted=True, cache=None,
                               cost_ms=judge_cost, nfe=1, uncached_positions=0)
    out = verify_greedy(prompt, candidate, lm, clock)
    out.cost_ms += judge_cost
    out.nfe += 1
    out.judge_fallback = "judge_rejected"
    return out


def make_verifier(name: str, topk_k: int = 3):
    if name == "greedy":
        def run(prompt, candidate, lm, clock=None, judge_prompt_text=None):
            return verify_greedy(prompt, candidate, lm, clock)
    elif name == "topk":
        def run(prompt, candidate, lm, clock=None, judge_prompt_text=None):
            return verify_topk(prompt, candidate, lm, topk_k, clock)
    elif name == "reflection":
        def run(prompt, candidate, lm, clock=None, judge_prompt_text=None):
            return verify_reflection(prompt, candidate, lm, clock, judge_prompt_text)
    else:
        raise ValueError(f"unknown verifier {name!r}")
    return run
