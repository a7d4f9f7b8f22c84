"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs only in the build container (it imports the read-only reference package
from /root/reference/pkg/src); the outputs are committed and the tests read
those files, so nothing at test time needs /root/reference.

    python tests/golden/make_golden.py [--skip-decoder]

* ngram_turns.json — the reference's `run_turn` / `run_baseline` event logs
  (pipeline.py:270-413) over its own `NGramLM` (lm.py:216-243) for varied
  prompts, chunkings, caps, verifiers and generators, plus its
  `greedy_decode` golden sequence (test_lm.py:161-168). Pins this package's
  algorithm layer one-to-one against the reference's.
* tiny_turns.json / tiny_verify.npz — config c1: the reference's algorithm
  layer driving the oracle decoder (`oracle.decoder.CpuDecoderLM`, float64)
  on the tiny fp32 shape: full event logs, per-(P, R) verify outcomes, argmax
  rows and logit slices. Trials whose consumed rows have a top-2 logit gap
  below 1e-4 are skipped (ambiguous under fp32 vs fp64 accumulation); the
  minimum gap of every kept trial is recorded.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF_SRC))

import specstream as ref  # noqa: E402  (the reference, read-only)
from specstream import lm as ref_lm  # noqa: E402
from specstream.pipeline import PipelineConfig as RefConfig  # noqa: E402

from oracle.decoder import CpuDecoderLM  # noqa: E402
from paper_2506_15556_b200.shapes import TINY  # noqa: E402
from paper_2506_15556_b200.vocab import SyntheticVocabulary  # noqa: E402

WORDS = ("alpha bravo charlie delta echo foxtrot golf hotel india juliet kilo lima "
         "mike november oscar papa quebec romeo sierra tango uniform victor whiskey "
         "xray yankee zulu . ? !").split()

GAP_MIN = 1e-4


def events_json(result) -> list[dict]:
    return [e.to_dict() for e in result.events]


def ngram_cases():
    rng = np.random.default_rng(20261017)
    cases = []
    variants = [
        dict(),
        dict(chunk_words=1, max_response_tokens=12),
        dict(chunk_words=3, max_response_tokens=40, system_prompt=""),
        dict(generator="jacobi", max_response_tokens=24),
        dict(verifier="topk", topk_k=3, max_response_tokens=24),
        dict(verifier="reflection", max_response_tokens=24),
        dict(rate_chars_per_min=3000.0, max_response_tokens=48),
        dict(lm_latency={"pass_base_ms": 12.0, "per_new_token_ms": 0.25}, max_response_tokens=30),
    ]
    for i in range(24):
        v = variants[i % len(variants)]
        n_words = int(rng.integers(3, 40))
        prompt = " ".join(WORDS[int(rng.integers(0, len(WORDS)))] for _ in range(n_words))
        second = " ".join(WORDS[int(rng.integers(0, len(WORDS)))] for _ in range(int(rng.integers(2, 12))))
        cases.append({"cfg": v, "turns": [prompt, second] if i % 3 == 0 else [prompt], "seed": 1000 + i})
    return cases


def make_ngram():
    out = {"greedy_decode": None, "cases": []}
    vocab = ref.build_vocabulary(["Capital of France ? Paris . filler words one two three"])
    out["greedy_decode"] = {
        "corpus": "Capital of France ? Paris . filler words one two three",
        "seed": 42, "prompt": "one two", "max_new": 8,
        "tokens": ref.greedy_decode(ref.NGramLM(vocab, seed=42), vocab.tokenize("one two"), max_new=8),
    }
    for case in ngram_cases():
        cfg = RefConfig.from_dict(dict(case["cfg"]))
        texts = ([cfg.system_prompt] if cfg.system_prompt else []) + case["turns"]
        vocab = ref.build_vocabulary(texts)
        rec = dict(case)
        for baseline in (False, True):
            lm = ref.NGramLM(vocab, seed=case["seed"], latency=cfg.lm_latency)
            results = ref.run_conversation(case["turns"], cfg, lm, conversation_id="g", baseline=baseline)
            rec["baseline" if baseline else "speculative"] = [
                {"final_text": r.final_text, "nfe_total": r.nfe_total, "events": events_json(r)} for r in results]
        out["cases"].append(rec)
    (HERE / "ngram_turns.json").write_text(json.dumps(out, sort_keys=True) + "\n")
    print("ngram cases:", len(out["cases"]))


def tiny_prompt(rng, vocab, n):
    ids = rng.integers(4, len(vocab), size=n)
    return " ".join(vocab.surface(int(i)) for i in ids)


def make_tiny():
    shape = TINY.as_dict()
    vocab = SyntheticVocabulary(TINY.vocab)
    # c1: 64-token query in 8 chunks, 32-token candidate cap, no system prompt
    cfg = RefConfig(system_prompt="", chunk_words=8, max_response_tokens=32)
    turns = []
    trial = 0
    while len(turns) < 6 and trial < 40:
        rng = np.random.default_rng(7000 + trial)
        text = tiny_prompt(rng, vocab, 64)
        rec = {"trial": trial, "prompt": text}
        ok = True
        for baseline in (False, True):
            lm = CpuDecoderLM(shape, vocab, seed=0, latency=ref_lm.LatencyModel())
            run = ref.run_baseline if baseline else ref.run_turn
            stream = ref.make_stream(text, cfg.rate_chars_per_min, cfg.chunk_words)
            res = run([], stream, cfg, lm)
            rec["baseline" if baseline else "speculative"] = {
                "final_text": res.final_text, "nfe_total": res.nfe_total, "events": events_json(res),
                "min_gap": float(lm.min_gap)}
            ok = ok and lm.min_gap > GAP_MIN
        if ok:
            turns.append(rec)
        trial += 1
    (HERE / "tiny_turns.json").write_text(json.dumps({"shape": shape, "config": "c1", "seed": 0,
                                                      "turns": turns}, sort_keys=True) + "\n")
    print("tiny turns kept:", len(turns), "of", trial)

    # per-pass verify goldens: random (P, R) pairs, argmax rows and logit slices
    lm = CpuDecoderLM(shape, vocab, seed=0)
    rng = np.random.default_rng(99)
    P, R, K, AM, LG, FS, GAP = [], [], [], [], [], [], []
    while len(K) < 24:
        p = [int(t) for t in rng.integers(4, len(vocab), size=int(rng.integers(1, 40)))]
        # candidates: half greedy continuations with a corrupted tail, half random
        if len(K) % 2 == 0:
            g = ref.greedy_decode(lm, p, max_new=int(rng.integers(1, 33)))[len(p):]
            cut = int(rng.integers(0, len(g) + 1))
            r = g[:cut] + [int(t) for t in rng.integers(1, len(vocab), size=len(g) - cut)]
        else:
            r = [int(t) for t in rng.integers(1, len(vocab), size=int(rng.integers(0, 33)))]
        out = ref.verify_greedy(p, r, lm)
        block, _, _ = lm.forward(p + r)
        rows = np.stack([block.row_for(len(p) - 1 + i) for i in range(len(r) + 1)])
        gaps = [float(np.partition(x, -2)[-1] - np.partition(x, -2)[-2]) for x in rows]
        if min(gaps) <= GAP_MIN:
            continue
        P.append(p); R.append(r); K.append(out.accepted_count); FS.append(out.first_sentence_accepted)
        AM.append([int(np.argmax(x)) for x in rows]); LG.append(rows[:, :64].astype(np.float64)); GAP.append(min(gaps))
    np.savez_compressed(HERE / "tiny_verify.npz",
                        prompts=np.array(json.dumps(P)), cands=np.array(json.dumps(R)), k=np.array(K),
                        first_sentence=np.array(FS), argmax=np.array(json.dumps(AM)),
                        logits64=np.array(json.dumps([x.tolist() for x in LG])), min_gap=np.array(GAP))
    print("tiny verify cases:", len(K), "k:", K)


def _turn_record(lm, cfg, turns, conv_id):
    """The reference's run_conversation on `lm` (speculative and baseline arms)."""
    rec = {}
    for baseline in (False, True):
        lm.min_gap = np.inf
        res = ref.run_conversation(turns, cfg, lm, conversation_id=conv_id, baseline=baseline)
        rec["baseline" if baseline else "speculative"] = [
            {"final_text": r.final_text, "nfe_total": r.nfe_total, "events": events_json(r)} for r in res]
        rec["min_gap_" + ("baseline" if baseline else "speculative")] = float(lm.min_gap)
    return rec


def make_c2(n_conv: int = 4):
    """Config c2: Qwen2.5-0.5B shape, fp32, 128-token query in 16 chunks, cap 64.
    Conversations 0 and 2 have a second turn (the reply goes into the history)."""
    from paper_2506_15556_b200.shapes import QWEN_05B
    shape = QWEN_05B.as_dict()
    vocab = SyntheticVocabulary(QWEN_05B.vocab)
    cfg = RefConfig(system_prompt="", chunk_words=8, max_response_tokens=64)
    convs, trial = [], 0
    lm = CpuDecoderLM(shape, vocab, seed=0, latency=ref_lm.LatencyModel())
    while len(convs) < n_conv and trial < 12:
        rng = np.random.default_rng(9000 + trial)
        turns = [tiny_prompt(rng, vocab, 128)]
        if len(convs) % 2 == 0:
            turns.append(tiny_prompt(rng, vocab, 48))
        rec = {"trial": trial, "turns": turns, **_turn_record(lm, cfg, turns, f"c2-{trial}")}
        ok = min(rec["min_gap_speculative"], rec["min_gap_baseline"]) > GAP_MIN
        print("c2 trial", trial, "turns", len(turns), "gap", rec["min_gap_speculative"], rec["min_gap_baseline"],
              "kept" if ok else "skipped", flush=True)
        if ok:
            convs.append(rec)
        trial += 1
    (HERE / "c2_turns.json").write_text(json.dumps({"shape": shape, "config": "c2", "seed": 0,
                                                   "conversations": convs}, sort_keys=True) + "\n")
    print("c2 conversations kept:", len(convs), "of", trial)


def make_tiny_topk(n_turns: int = 5):
    """Config c1 with the reference's top-k verifier (k = 3, verify.py:100-113):
    event logs of `run_turn` on the float64 oracle decoder. A top-k decision
    depends on where the candidate token ranks, not only on the top-2 gap, so a
    turn is kept only if the float32 oracle (a different accumulation) gives the
    identical event log — the decisions are not near a rank boundary."""
    shape = TINY.as_dict()
    vocab = SyntheticVocabulary(TINY.vocab)
    cfg = RefConfig(system_prompt="", chunk_words=8, max_response_tokens=32, verifier="topk", topk_k=3)
    turns, trial = [], 0
    while len(turns) < n_turns and trial < 40:
        rng = np.random.default_rng(7700 + trial)
        text = tiny_prompt(rng, vocab, 64)
        logs = []
        for dtype in (np.float64, np.float32):
            lm = CpuDecoderLM(shape, vocab, seed=0, latency=ref_lm.LatencyModel(), dtype=dtype)
            res = ref.run_turn([], ref.make_stream(text, cfg.rate_chars_per_min, cfg.chunk_words), cfg, lm)
            logs.append({"final_text": res.final_text, "nfe_total": res.nfe_total, "events": events_json(res),
                         "min_gap": float(lm.min_gap)})
        ks = [e["k"] for e in logs[0]["events"] if e["kind"] == "verify"]
        ok = logs[0]["events"] == logs[1]["events"] and logs[0]["min_gap"] > GAP_MIN
        print("topk trial", trial, "k per round", ks, "kept" if ok else "skipped", flush=True)
        if ok:
            turns.append({"trial": trial, "prompt": text, "speculative": logs[0]})
        trial += 1
    (HERE / "tiny_topk_turns.json").write_text(json.dumps({"shape": shape, "config": "c1-topk3", "seed": 0,
                                                          "turns": turns}, sort_keys=True) + "\n")
    print("topk turns kept:", len(turns), "of", trial)


def make_tiny_generator(generator: str = "jacobi", n_turns: int = 4):
    """Config c1 with the reference's Jacobi generator (generate.py:181-291) on the float64
    oracle decoder: full event logs, kept when every consumed row's top-2 gap > GAP_MIN."""
    shape = TINY.as_dict()
    vocab = SyntheticVocabulary(TINY.vocab)
    cfg = RefConfig(system_prompt="", chunk_words=8, max_response_tokens=32, generator=generator)
    turns, trial = [], 0
    while len(turns) < n_turns and trial < 30:
        rng = np.random.default_rng(7900 + trial)
        text = tiny_prompt(rng, vocab, 64)
        lm = CpuDecoderLM(shape, vocab, seed=0, latency=ref_lm.LatencyModel())
        res = ref.run_turn([], ref.make_stream(text, cfg.rate_chars_per_min, cfg.chunk_words), cfg, lm)
        rec = {"trial": trial, "prompt": text, "speculative": {"final_text": res.final_text, "nfe_total": res.nfe_total,
                                                              "events": events_json(res), "min_gap": float(lm.min_gap)}}
        kinds = sorted({e["pass_kind"] for e in rec["speculative"]["events"] if e["kind"] == "generate_step"})
        print(generator, "trial", trial, "passes", kinds, "gap", lm.min_gap, flush=True)
        if lm.min_gap > GAP_MIN:
            turns.append(rec)
        trial += 1
    (HERE / f"tiny_{generator}_turns.json").write_text(json.dumps({"shape": shape, "config": f"c1-{generator}",
                                                                  "seed": 0, "turns": turns}, sort_keys=True) + "\n")
    print(generator, "turns kept:", len(turns), "of", trial)


if __name__ == "__main__":
    if "--jacobi" in sys.argv:
        make_tiny_generator("jacobi")
        sys.exit(0)
    if "--c2" in sys.argv:
        make_c2()
        sys.exit(0)
    if "--topk" in sys.argv:
        make_tiny_topk()
        sys.exit(0)
    make_ngram()
    if "--skip-decoder" not in sys.argv:
        make_tiny()
