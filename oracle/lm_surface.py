"""ORACLE (test infrastructure only — never imported by the product path).

Minimal restatement of the reference's backend value types so the oracle runs
without `/root/reference` (which does not exist on the GPU box):
`LatencyModel` (`/root/reference/pkg/src/specstream/lm.py:40-57`),
`CacheHandle` (`lm.py:60-81`), `LogitsBlock` (`lm.py:84-104`), the error
types (`lm.py:32-37`) and the instance-id counter (`lm.py:148-154`). They are
duck-type compatible with the reference's own algorithm layer, so the
reference's `verify_greedy` / `run_turn` can drive an oracle backend directly
when generating golden fixtures (tests/golden/make_golden.py).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np


class PrefixViolationError(ValueError):
    pass


class JudgeUnsupportedError(RuntimeError):
    pass


@dataclass(frozen=True)
class LatencyModel:
    pass_base_ms: float = 30.0
    per_new_token_ms: float = 0.5

    def pass_cost(self, uncached_positions: int) -> float:
        return self.pass_base_ms + self.per_new_token_ms * uncached_positions


@dataclass(frozen=True)
class CacheHandle:
    prefix: tuple
    backend_id: int

    @property
    def cached_prefix_length(self) -> int:
        return len(self.prefix)

    def truncated(self, length: int) -> "CacheHandle":
        if length > len(self.prefix):
            raise PrefixViolationError("cannot extend a cache by truncation")
        return CacheHandle(self.prefix[:length], self.backend_id)


@dataclass(frozen=True)
class LogitsBlock:
    rows: np.ndarray
    first_position: int

    def row_for(self, position: int) -> np.ndarray:
        idx = position - self.first_position
        if not 0 <= idx < len(self.rows):
            raise IndexError(f"position {position} not covered by this block")
        return self.rows[idx]

    @property
    def last_row(self) -> np.ndarray:
        return self.rows[-1]


# oracle backends draw ids from a range far from the product's counter so a
# handle can never be mistaken across the two.
_ids = itertools.count(1_000_000)


@dataclass(frozen=True)
class JudgeResult:
    """lm.py:107-114: consistent iff yes_score > no_score."""
    yes_score: float
    no_score: float

    @property
    def consistent(self) -> bool:
        return self.yes_score > self.no_score


# lm.py:117-126, verbatim template text (a data constant of the reference API)
JUDGE_TEMPLATE = (
    "<|im_start|>user\n"
    "You are given an incomplete prompt and the model's speculative partial answer.\n"
    "Please judge whether the partial prompt is consistent with the model's answer.\n"
    "Partial Prompt: {partial_prompt}\n"
    "Partial Answer: {partial_answer}\n"
    "<|im_end|>\n"
    "<|im_start|>assistant\n"
)


def fresh_backend_id() -> int:
    return next(_ids)
