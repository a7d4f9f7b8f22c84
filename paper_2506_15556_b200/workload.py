"""The c5 synthetic conversation workload (simulated by simulate.py and bench.py).

Config c5 (BASELINE.json): 1024 synthetic conversations with an MT-Bench /
Lmsys-like length distribution, 8B shape, one stream per GPU.

Prompt words ~ lognormal(ln 25, 0.6) clipped to [4, 120]; half of the
conversations have a second turn; words are uniform over the non-special ids
of the synthetic vocabulary; rate 600 chars/min; response cap 64.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._specstream import specstream

PipelineConfig = specstream.PipelineConfig
Conversation = specstream.Conversation


@dataclass(frozen=True)
class WorkloadSpec:
    conversations: int = 1024
    mean_words: float = 25.0
    sigma: float = 0.6
    min_words: int = 4
    max_words: int = 120
    two_turn_share: float = 0.5
    system_words: int = 32
    seed: int = 0


def _words(rng, vocab, n: int) -> str:
    ids = rng.integers(4, len(vocab), size=n)
    return " ".join(vocab.surface(int(i)) for i in ids)


def _length(rng, spec: WorkloadSpec) -> int:
    n = int(round(rng.lognormal(np.log(spec.mean_words), spec.sigma)))
    return int(min(spec.max_words, max(spec.min_words, n)))


def synthetic_conversations(vocab, spec: WorkloadSpec = WorkloadSpec()) -> list[Conversation]:
    """Deterministic dataset: conversation i depends only on (spec.seed, i)."""
    out = []
    for i in range(spec.conversations):
        rng = np.random.default_rng([spec.seed, i])
        turns = [_words(rng, vocab, _length(rng, spec))]
        if rng.random() < spec.two_turn_share:
            turns.append(_words(rng, vocab, _length(rng, spec)))
        out.append(Conversation(id=f"c{i:05d}", turns=turns))
    return out


def system_prompt(vocab, spec: WorkloadSpec = WorkloadSpec()) -> str:
    rng = np.random.default_rng([spec.seed, 1 << 30])
    return _words(rng, vocab, spec.system_words) if spec.system_words else ""


def c5_config(vocab, spec: WorkloadSpec = WorkloadSpec(), **overrides) -> PipelineConfig:
    base = dict(system_prompt=system_prompt(vocab, spec), chunk_words=2, max_response_tokens=64,
                rate_chars_per_min=600.0)
    base.update(overrides)
    return PipelineConfig(**base)
