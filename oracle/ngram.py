"""ORACLE (test infrastructure only — never imported by the product path).

Restatement of the reference's hash n-gram backend, `NGramLM`
(`/root/reference/pkg/src/specstream/lm.py:216-243`): the score row for a
context is `numpy.random.default_rng([seed, len(window), *window]).random(V)`
over the last `order` tokens. Third-party dependency: numpy's PCG64 /
`SeedSequence` (numpy >= 1.24, unpinned in `pkg/pyproject.toml:10-12`; 2.3.5
here). Pinned by the reference's golden sequence `test_lm.py:161-168`
(`[9, 10, 10, 10, 9, 10, 3, 6, 11, 3]`), re-asserted in tests/test_oracle.py.

It lets the CPU test suite drive the product package's algorithm layer
(verify / generate / pipeline) with the same backend the reference's own tests
use, so golden event logs from the reference compare one-to-one.
"""

from __future__ import annotations

import numpy as np

from .lm_surface import CacheHandle, JudgeUnsupportedError, LatencyModel, LogitsBlock, PrefixViolationError, fresh_backend_id


class NGramOracleLM:
    def __init__(self, vocab, seed: int = 0, order: int = 3, latency: LatencyModel | None = None,
                 judge_error: type = JudgeUnsupportedError):
        # judge_error: the caller's capability-error type (the reference's or
        # the product's), raised by judge_consistency (lm.py:205-206)
        self._judge_error = judge_error
        self.vocab = vocab
        self.latency = latency or LatencyModel()
        self._backend_id = fresh_backend_id()
        self.seed = seed
        self.order = order
        self._memo: dict[tuple, np.ndarray] = {}

    @property
    def vocab_size(self) -> int:
        return len(self.vocab)

    @property
    def eos_id(self) -> int:
        return 0

    def next_row(self, context: tuple) -> np.ndarray:
        window = tuple(context[-self.order:]) if self.order > 0 else ()
        row = self._memo.get(window)
        if row is None:
            row = np.random.default_rng([self.seed, len(window), *window]).random(self.vocab_size)
            self._memo[window] = row
        return row

    def forward(self, context, cache=None):
        start = 0
        if cache is not None:
            if cache.backend_id != self._backend_id:
                raise PrefixViolationError("cache handle belongs to a different backend instance")
            if tuple(context[: len(cache.prefix)]) != tuple(cache.prefix):
                raise PrefixViolationError("context does not extend the cached prefix")
            start = len(cache.prefix)
        if start >= len(context):
            raise PrefixViolationError("forward pass requires at least one uncached position")
        ctx = tuple(context)
        rows = np.stack([self.next_row(ctx[: j + 1]) for j in range(start, len(ctx))])
        return LogitsBlock(rows, start), CacheHandle(ctx, self._backend_id), self.latency.pass_cost(len(ctx) - start)

    def judge_consistency(self, partial_prompt, partial_answer):
        raise self._judge_error("n-gram oracle has no judge")
