"""B200-native predict-and-verify loop of PredGen (arXiv 2506.15556).

Public names mirror the reference package `specstream`
(`/root/reference/pkg/src/specstream/__init__.py:10-66`) for the hot path —
chunked prompt stream, verify, regenerate, TTFS accounting — plus `B200LM`,
the CUDA backend behind the reference's `LanguageModel` surface. The toy
backends (`NGramLM`, `ScriptedLM`) and the CLI are out of scope.
"""

from .backend import B200LM, LazyRow
from .clocks import PromptStream, SimClock, StreamChunk, WallClock, make_stream
from .generation import GenerationBudget, GenerationResult, SentenceTracker, ar_generate, jacobi_generate, predictive_generate
from .model_api import (
    CacheHandle,
    JudgeResult,
    JudgeUnsupportedError,
    LanguageModel,
    LatencyModel,
    LogitsBlock,
    PrefixViolationError,
    argmax_token,
    greedy_decode,
    topk_tokens,
)
from .shapes import LLAMA3_8B, MISTRAL_7B, QWEN_05B, SHAPES, TINY, DecoderShape
from .speech import TtsJob, TtsLatencyModel, TtsSimulator
from .turn import (
    EventLog,
    PipelineConfig,
    PipelineEvent,
    TurnResult,
    TurnState,
    read_events_jsonl,
    run_baseline,
    run_conversation,
    run_turn,
    write_events_jsonl,
)
from .turn_metrics import (
    Conversation,
    MalformedLogError,
    MetricsRecord,
    compute_metrics,
    load_dataset,
    nfetfs_histogram,
    summarize,
    summarize_percentiles,
)
from .verifier import VerifierOutcome, make_verifier, verify_greedy, verify_reflection, verify_topk
from .vocab import EOS_ID, SentenceSpan, SyntheticVocabulary, Vocabulary, VocabularyError, build_vocabulary, first_sentence

__version__ = "0.1.0"
