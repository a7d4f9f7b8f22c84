"""The backend surface the predict-and-verify loop talks to.

Same names, argument meanings and error behaviour as the reference's
`specstream.lm` (`/root/reference/pkg/src/specstream/lm.py`), so code written
against the reference — including the reference's own `verify_greedy`,
`ar_generate` and `run_turn` — runs unchanged on `B200LM`:

* `LatencyModel.pass_cost(u) = base + per_token * u` (`lm.py:40-57`)
* `CacheHandle` is an immutable prefix value with free truncation (`lm.py:60-81`)
* `LogitsBlock.row_for / last_row` (`lm.py:84-104`)
* `argmax_token` ties to the lowest id; `topk_tokens` orders by (-score, id)
  (`lm.py:134-145`)
* `LanguageModel.forward` rules: foreign handle, non-extending context and a
  fully cached context raise `PrefixViolationError` (`lm.py:182-203`)
* `greedy_decode` is the prefill-then-decode oracle loop (`lm.py:350-382`)
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .vocab import EOS_ID, split_words

DEFAULT_MAX_NEW_TOKENS = 256


class PrefixViolationError(ValueError):
    """The supplied cache does not cover a prefix of the context."""


class JudgeUnsupportedError(RuntimeError):
    """The backend cannot score consistency judgments."""


@dataclass(frozen=True)
class LatencyModel:
    pass_base_ms: float = 30.0
    per_new_token_ms: float = 0.5

    def __post_init__(self) -> None:
        if min(self.pass_base_ms, self.per_new_token_ms) < 0:
            raise ValueError("latency parameters must be nonnegative")

    def pass_cost(self, uncached_positions: int) -> float:
        return self.pass_base_ms + self.per_new_token_ms * uncached_positions


@dataclass(frozen=True)
class CacheHandle:
    """A materialised context prefix on one backend instance.

    On the B200 backend the KV pages are owned by the backend, not the handle
    (handles have no release hook); a handle only names a prefix, which the
    backend resolves against its resident sequence.
    """

    prefix: tuple
    backend_id: int

    @property
    def cached_prefix_length(self) -> int:
        return len(self.prefix)

    def truncated(self, length: int) -> "CacheHandle":
        if length > len(self.prefix):
            raise PrefixViolationError(
                f"cannot extend cache of length {len(self.prefix)} to {length} by truncation")
        return CacheHandle(self.prefix[:length], self.backend_id)


@dataclass(frozen=True)
class LogitsBlock:
    """Score rows for positions first_position .. first_position+len(rows)-1."""

    rows: object  # np.ndarray, or a lazy row provider with __len__/__getitem__
    first_position: int

    def row_for(self, position: int) -> np.ndarray:
        i = position - self.first_position
        if i < 0 or i >= len(self.rows):
            raise IndexError(f"position {position} not covered by this block")
        return self.rows[i]

    @property
    def last_row(self) -> np.ndarray:
        return self.rows[len(self.rows) - 1]


@dataclass(frozen=True)
class JudgeResult:
    yes_score: float
    no_score: float

    @property
    def consistent(self) -> bool:
        return self.yes_score > self.no_score


CONSISTENCY_JUDGE_TEMPLATE = (
    "<|im_start|>user\n"
    "You are given an incomplete prompt and the model's speculative partial answer.\n"
    "Please judge whether the partial prompt is consistent with the model's answer.\n"
    "Partial Prompt: {partial_prompt}\n"
    "Partial Answer: {partial_answer}\n"
    "<|im_end|>\n"
    "<|im_start|>assistant\n"
)


def decoder_judge(lm, partial_prompt: str, partial_answer: str):
    """PredGen's self-consistency judge for a decoder backend: one fresh
    forward pass over the formatted judge prompt (lm.py:117-131), then the
    last row's scores of the words "yes" and "no" (`JudgeResult.consistent`
    iff yes > no, lm.py:107-114). Returns (JudgeResult, cost of the pass)."""
    ids = lm.vocab.judge_ids
    toks = ids(format_judge_prompt(partial_prompt, partial_answer))
    block, _, cost = lm.forward(toks)
    row = block.last_row
    yes, no = ids("yes")[0], ids("no")[0]
    return JudgeResult(yes_score=float(row[yes]), no_score=float(row[no])), cost


def format_judge_prompt(partial_prompt: str, partial_answer: str) -> str:
    return CONSISTENCY_JUDGE_TEMPLATE.format(partial_prompt=partial_prompt,
                                             partial_answer=partial_answer)


def argmax_token(row) -> int:
    """Highest score; ties go to the lowest id (numpy argmax semantics)."""
    return int(np.argmax(row))


def topk_tokens(row, k: int) -> set[int]:
    if k < 1:
        raise ValueError("k must be at least 1")
    row = np.asarray(row)
    k = min(k, len(row))
    # stable sort on -score keeps equal scores in id order
    order = np.argsort(-row, kind="stable")
    return set(int(i) for i in order[:k])


_instance_ids = itertools.count(1)


def fresh_backend_id() -> int:
    return next(_instance_ids)


class LanguageModel:
    """Base for backends: vocab, latency model, instance id, judge default."""

    def __init__(self, vocab, latency: LatencyModel | None = None) -> None:
        self.vocab = vocab
        self.latency = latency or LatencyModel()
        self._backend_id = fresh_backend_id()

    @property
    def vocab_size(self) -> int:
        return len(self.vocab)

    @property
    def eos_id(self) -> int:
        return EOS_ID

    def _cached_start(self, context, cache) -> int:
        """Validate `cache` against `context`; return the first uncached position."""
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
        raise NotImplementedError

    def judge_consistency(self, partial_prompt: str, partial_answer: str):
        raise JudgeUnsupportedError(f"{type(self).__name__} has no consistency judge")

    def judge_cost(self, partial_prompt: str, partial_answer: str) -> float:
        return self.latency.pass_cost(len(split_words(format_judge_prompt(partial_prompt, partial_answer))))


def greedy_decode(lm, prompt, max_new: int = DEFAULT_MAX_NEW_TOKENS, stop=None) -> list[int]:
    """Oracle loop: prefill prompt[:-1], then one 1-row pass per new token."""
    if max_new < 0:
        raise ValueError("max_new must be nonnegative")
    seq = list(prompt)
    if max_new == 0 or not seq:
        return seq
    cache = lm.forward(seq[:-1])[1] if len(seq) > 1 else None
    generated: list[int] = []
    while len(generated) < max_new:
        block, cache, _ = lm.forward(seq, cache)
        tok = argmax_token(block.last_row)
        seq.append(tok)
        generated.append(tok)
        if tok == lm.eos_id or (stop is not None and stop(generated)):
            break
    return seq
