"""B200-native predict-and-verify backend for PredGen (arXiv 2506.15556).

`B200LM` is a `specstream.lm.LanguageModel` (the reference package's backend
surface, `/root/reference/pkg/src/specstream/lm.py:157-213`) whose arithmetic
runs in hand-written sm_100a kernels behind a C ABI (include/predgen_b200.h).
The predict-and-verify loop is the reference's own, unmodified code
(installed into baseline/_ref, see `_specstream.py`); this package adds:

* `B200LM` and the synthetic vocabulary of the random-init decoders;
* `fused`: one-call device verifiers bound into the reference's pipeline;
* `workload` / `simulate`: the sharded conversation simulation (one process
  per GPU, dynamic work queue) and the c5 synthetic workload;
* `report.summarize_percentiles`: p50/p90/p99 TTFS next to the reference's means.

For convenience the reference's hot-path names are re-exported, so code
written against `specstream` can switch its import.
"""

from ._specstream import specstream
from .backend import B200LM, LazyRow
from .fused import make_verifier, run_conversation, run_turn, verify_greedy, verify_topk
from .report import percentile, summarize_percentiles
from .shapes import LLAMA3_8B, MISTRAL_7B, QWEN_05B, SHAPES, TINY, DecoderShape
from .vocab import SyntheticVocabulary

# the reference's public API (specstream/__init__.py:10-66), unchanged
PipelineConfig = specstream.PipelineConfig
run_baseline = specstream.run_baseline
make_stream = specstream.make_stream
SimClock = specstream.SimClock
compute_metrics = specstream.compute_metrics
summarize = specstream.summarize
greedy_decode = specstream.greedy_decode
ar_generate = specstream.ar_generate
jacobi_generate = specstream.jacobi_generate
predictive_generate = specstream.predictive_generate
verify_reflection = specstream.verify_reflection
LatencyModel = specstream.LatencyModel
CacheHandle = specstream.CacheHandle
LogitsBlock = specstream.LogitsBlock
PrefixViolationError = specstream.PrefixViolationError
JudgeUnsupportedError = specstream.JudgeUnsupportedError
Conversation = specstream.Conversation
MetricsRecord = specstream.MetricsRecord
read_events_jsonl = specstream.read_events_jsonl
write_events_jsonl = specstream.write_events_jsonl

__version__ = "0.2.0"
