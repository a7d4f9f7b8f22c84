"""ORACLE — test infrastructure, not product.

CPU restatements used only as the checker by tests/, `__graft_entry__.smoke()`
and the `cpu_baseline` / `--impl reference` legs of bench.py:

* `weights`  — the counter-based weight generator (bit-identical to csrc/init.cu)
* `decoder`  — float64 numpy decoder + `CpuDecoderLM`, the `LanguageModel`
               contract of `/root/reference/pkg/src/specstream/lm.py:182-203`
* `ngram`    — the reference's `NGramLM` (lm.py:216-243), pinned by its golden
               sequence (test_lm.py:161-168)
* `lm_surface` — value types of lm.py:32-154 so the oracle runs without the
               reference installed

Decoder numerics are parity-unpinned by the reference (it has no decoder); the
algorithm layer is pinned by golden event logs the reference itself produced
(tests/golden/make_golden.py).
"""
