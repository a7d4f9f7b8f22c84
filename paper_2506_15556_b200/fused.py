"""One-call device verifiers, plugged into the reference's own loop.

The reference verifies by one `lm.forward(P ++ R)` followed by a host loop
over the rows (`_verify_by_rule`, `/root/reference/pkg/src/specstream/
verify.py:63-83`). On `B200LM` that generic path already costs one device
pass (the argmax of every row comes back with it), but top-k is another
matter: `topk_tokens` sorts a Python list of all V scores per row
(`lm.py:139-145`, 237 ms per row at V = 128k), which would dwarf the pass.

`verify_greedy` / `verify_topk` below call the fused C-ABI entry points
instead — pass, per-row argmax (or candidate rank), compare, first mismatch
and first terminator on the device, KV rolled back to |P| + k — and build the
reference's own `VerifierOutcome` with the reference's own helpers, field for
field what `_verify_by_rule` returns (tests/test_gpu_dropin.py asserts equal
event logs). Backends without the fused calls get the reference's functions.

`run_turn` / `run_conversation` run the reference's `specstream.pipeline`
functions unmodified; for the duration of the call its `make_verifier` name
(pipeline.py:26, resolved at pipeline.py:292) is bound to the one here. This
is a process-global binding, like the reference's own module-level backend id
counter (lm.py:148-154): one pipeline per process.
"""

from __future__ import annotations

import contextlib

from ._specstream import specstream

_verify = specstream.verify
_pipeline = specstream.pipeline


def _outcome(prompt, candidate, k, handle, cost, vocab):
    return _verify.VerifierOutcome(
        accepted_count=k,
        first_sentence_accepted=_verify._sentence_covered(candidate, k, vocab),
        cache=handle.truncated(len(prompt) + k),
        cost_ms=cost,
        nfe=1,
        uncached_positions=len(prompt) + len(candidate),
    )


def verify_greedy(prompt, candidate, lm, clock=None):
    """`specstream.verify.verify_greedy` (verify.py:86-97) in one device call."""
    fused = getattr(lm, "verify_greedy_fused", None)
    if fused is None:
        return _verify.verify_greedy(prompt, candidate, lm, clock)
    if not prompt:
        raise ValueError("verification requires a nonempty prompt context")
    k, handle, cost = fused(list(prompt), list(candidate))
    _verify._charge(clock, cost)
    return _outcome(prompt, candidate, k, handle, cost, lm.vocab)


def verify_topk(prompt, candidate, lm, k: int, clock=None):
    """`specstream.verify.verify_topk` (verify.py:100-113) in one device call:
    rank(t) = #{j : s_j > s_t or (s_j == s_t and j < t)} counted on the device,
    accept while rank < k (the (-score, id) order of `topk_tokens`, lm.py:139-145)."""
    if k < 1:
        raise ValueError("top-k verification requires k >= 1")
    fused = getattr(lm, "verify_topk_fused", None)
    if fused is None:
        return _verify.verify_topk(prompt, candidate, lm, k, clock)
    if getattr(lm, "vocab_shards", 1) > 1:
        raise NotImplementedError("top-k verification needs whole LM-head rows; this backend holds one vocab "
                                  "shard (config c4 supports greedy verification only)")
    if not prompt:
        raise ValueError("verification requires a nonempty prompt context")
    acc, handle, cost = fused(list(prompt), list(candidate), k)
    _verify._charge(clock, cost)
    return _outcome(prompt, candidate, acc, handle, cost, lm.vocab)


def make_verifier(name: str, topk_k: int = 3):
    """`specstream.verify.make_verifier` (verify.py:161-175) with the fused
    greedy / top-k verifiers; reflection is the reference's own."""
    if name == "greedy":
        return lambda prompt, candidate, lm, clock=None, judge_prompt_text=None: verify_greedy(
            prompt, candidate, lm, clock)
    if name == "topk":
        return lambda prompt, candidate, lm, clock=None, judge_prompt_text=None: verify_topk(
            prompt, candidate, lm, topk_k, clock)
    return _verify.make_verifier(name, topk_k)


@contextlib.contextmanager
def fused_verifiers():
    """Bind the reference pipeline's `make_verifier` to the fused one for a block."""
    original = _pipeline.make_verifier
    _pipeline.make_verifier = make_verifier
    try:
        yield
    finally:
        _pipeline.make_verifier = original


def run_turn(*args, **kwargs):
    """The reference's `run_turn` (pipeline.py:270-367) with fused verifiers."""
    with fused_verifiers():
        return _pipeline.run_turn(*args, **kwargs)


def run_conversation(*args, **kwargs):
    """The reference's `run_conversation` (pipeline.py:416-434) with fused verifiers."""
    with fused_verifiers():
        return _pipeline.run_conversation(*args, **kwargs)
