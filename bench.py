"""Benchmark: PredGen predict-and-verify conversation simulation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (config c5 of BASELINE.json): synthetic MT-Bench/Lmsys-length
conversations on the Llama-3-8B shape (bf16, random init), run through the
reference's own loop (`specstream.run_conversation` with the fused verifiers
bound in, paper_2506_15556_b200/fused.py) on `B200LM`. One process per GPU,
ranks claim conversations from a shared work queue (no per-pass collective).

Two phases, because the two BASELINE metrics need two clocks:

1. conversations/s (the JSON `value`): the reference's modeled cost
   (`LatencyModel`, lm.py:40-57) drives the SimClock, exactly like the
   reference's `simulate` command; every decision then depends only on the
   model's argmaxes, so the pass schedule of a conversation is deterministic.
   Step s = conversations [s*P*N, (s+1)*P*N) (P = --conv-per-step per rank).
   value = conversations / max-over-ranks device time of every pass;
   e2e = conversations / max-over-ranks CUDA-event wall time of the steps
   (host Python, H2D token copies and D2H argmax reads included).
   The per-conversation pass schedule is compared with the committed one
   (bench_data/, tools/make_schedule.py) that the reference arm prices.
2. latency (rank 0): measured cost — every pass charges its CUDA-event ms —
   over a fixed set of conversations: p50 verify-step latency, decode-step
   latency, p50/p90 simulated TTFS, each with its HBM-roofline fraction.

`bf16_agreement` (rank 0): argmax agreement of one 72-row verify pass with
the layer-streamed float64 oracle (oracle/parity.py) — the oracle as the
checker of what was timed, not part of any timed region.

`--impl reference` (and `cpu_baseline`): the reference has no decoder (its LM
is a hash table, lm.py:216-243), so its CPU path for this workload is the
oracle decoder (oracle/decoder.py, numpy fp32, all host threads) pricing the
SAME pass schedule: per-pass CPU times t(rows) = a + b*rows fitted on a
bounded sample of 8B-shape passes, summed over the timed conversations'
committed schedule (same conversation ids, same config dict as this arm).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("conversations/sec (c5 predict-and-verify simulation, modeled-cost schedule); "
          "verify-step latency; simulated p50 TTFS")
UNIT = "conversations/s"
TTFS_CONVERSATIONS = range(1000, 1012)  # measured-cost latency phase (rank 0)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--conv-per-step", type=int, default=2)
    ap.add_argument("--shape", default="llama-3-8b")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-agreement", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c2 / c4-shape per-pass latencies")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    return ap.parse_args(argv)


def schedule_path(shape_name: str) -> Path:
    return ROOT / "bench_data" / f"c5_schedule_{shape_name}.json"


def timed_ids(world: int, per: int, warmup: int, steps: int) -> tuple[int, int]:
    return warmup * per * world, (warmup + steps) * per * world


def workload_config(args, world: int) -> dict:
    """The config dict both arms print (identical by construction)."""
    lo, hi = timed_ids(world, args.conv_per_step, args.warmup, args.steps)
    return {"workload": "c5: synthetic MT-Bench/Lmsys-length conversations through the reference's run_turn, "
                        "Llama-3-8B shape, bf16, modeled-cost SimClock (LatencyModel 30 ms + 0.5 ms/token)",
            "shape": args.shape, "timed_conversation_ids": [lo, hi], "conversations_per_rank_per_step":
                args.conv_per_step, "chunk_words": 2, "max_response_tokens": 64, "rate_chars_per_min": 600.0,
            "schedule": str(schedule_path(args.shape).relative_to(ROOT)),
            "l2": "inputs larger than L2 (15 GB of weights streamed per pass)",
            "parallelism": f"{world} conversation shards, dynamic work queue, no per-pass collective"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:6]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PS_BENCH_SHARE_GPU=1: every rank on device 0 (tests the N>1 path on one GPU)
    device = 0 if os.environ.get("PS_BENCH_SHARE_GPU") == "1" else local
    return world, rank, device


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# -- CPU pricing of a pass schedule ---------------------------------------------------------

class CpuPassTimer:
    """Oracle decoder (numpy fp32, BLAS on all host threads) at `shape`, built once.

    Every layer streams layer 0's weights (share_layer_weights): the same bytes and
    FLOPs per pass as the full model, without generating 8B values on the host.
    Passes run over a `context`-token resident prefix (attention is < 1% of a CPU
    pass at this length)."""

    WIDTHS = (1, 8, 32, 72)

    def __init__(self, shape, threads: int, context: int = 128):
        import numpy as np
        from threadpoolctl import threadpool_limits
        from oracle.decoder import DecoderOracle

        # torchrun exports OMP_NUM_THREADS=1 to every rank, which OpenBLAS read at load
        # time: set the BLAS pool to the thread count this timer reports
        self._limits = threadpool_limits(limits=threads, user_api="blas")
        t0 = time.perf_counter()
        d = dict(shape.as_dict())
        d["mode"] = 0  # fp32 arithmetic: no bf16 rounding emulation in the timed port
        self.m = DecoderOracle(d, seed=0, dtype=np.float32, share_layer_weights=True)
        self.rng = np.random.default_rng(0)
        self.vocab, self.context, self.threads = shape.vocab, context, threads
        self.m.extend([int(t) for t in self.rng.integers(4, shape.vocab, context)])
        self.setup_s = time.perf_counter() - t0

    def sample(self, sample_s: float) -> dict:
        """Median pass times: t_decode = the 1-row pass, t(rows) = a + b*rows for wider
        passes (least squares over the per-width medians)."""
        import numpy as np

        m, rng, widths = self.m, self.rng, self.WIDTHS
        samples = {w: [] for w in widths}
        deadline = time.perf_counter() + sample_s
        i = 0
        while time.perf_counter() < deadline or any(len(v) < 2 for v in samples.values()):
            w = widths[i % len(widths)]
            i += 1
            m.truncate(self.context)
            t = time.perf_counter()
            m.extend([int(x) for x in rng.integers(4, self.vocab, w)])
            samples[w].append((time.perf_counter() - t) * 1e3)
            if w == 1:  # decode passes are the bulk of a schedule: sample them more densely
                for _ in range(3):
                    t = time.perf_counter()
                    m.extend([int(rng.integers(4, self.vocab))])
                    samples[1].append((time.perf_counter() - t) * 1e3)
            if i > 400:
                break
        ys = {w: statistics.median(samples[w]) for w in widths}
        wide = [w for w in widths if w > 1]
        b, a = np.polyfit(np.array(wide, dtype=np.float64), np.array([ys[w] for w in wide]), 1)
        return {"decode_ms": float(ys[1]), "a_ms": float(a), "b_ms_per_row": float(b),
                "median_ms": {str(w): float(y) for w, y in ys.items()},
                "samples": {str(w): len(v) for w, v in samples.items()}, "setup_s": self.setup_s,
                "threads": self.threads, "context": self.context}


def cpu_pass_model(shape, sample_s: float, threads: int, context: int = 128) -> dict:
    return CpuPassTimer(shape, threads, context).sample(sample_s)


def cpu_schedule_ms(model: dict, entries) -> float:
    """CPU time of schedule entries [passes, rows, decode_passes, extend_passes]:
    decode passes at t_decode, extend passes at a + b*rows."""
    return sum(model["decode_ms"] * e[2] + model["a_ms"] * e[3] + model["b_ms_per_row"] * (e[1] - e[2])
               for e in entries)


def load_schedule(shape_name: str) -> dict:
    p = schedule_path(shape_name)
    return json.loads(p.read_text()) if p.exists() else {"conversations": {}}


def summarize_schedule(entries) -> list:
    """[(ctx, rows, ...)] of one conversation -> [n_passes, rows, decode_passes, extend_passes]."""
    rows = sum(e[1] for e in entries)
    dec = sum(1 for e in entries if e[1] == 1)
    return [len(entries), rows, dec, len(entries) - dec]


def pass_latency(shape, hbm_gbs: float, ctx_len: int = 128, window: int = 72) -> dict:
    """p50 device ms of 1-row decode steps and of `window`-row verify passes over a
    `ctx_len`-token context at `shape`, each against its HBM floor (weights once)."""
    import numpy as np
    from paper_2506_15556_b200 import B200LM

    lm = B200LM(shape, seed=0, max_seq=1024, cost_mode="measured")
    try:
        rng = np.random.default_rng(0)
        ctx = [int(t) for t in rng.integers(4, shape.vocab, ctx_len)]
        lm.decode_greedy_fused(ctx, 4)
        dec = []
        for _ in range(3):
            lm.truncate(ctx_len)
            dec += [c for _, c in lm.decode_greedy_fused(ctx, 24)[1:]]
        cand = [int(t) for t in rng.integers(4, shape.vocab, window - 8)]
        ver = []
        for _ in range(5):
            lm.truncate(ctx_len - 8)
            ver.append(lm.verify_greedy_detail(ctx, cand)["gpu_ms"])
    finally:
        lm.close()
    floor = shape.weight_bytes_per_pass() / (hbm_gbs * 1e9) * 1e3
    # the verify window's matmul FLOPs against the dtype's arithmetic peak: bf16 = the measured
    # cuBLAS sustained figure; fp32 = FFMA issue rate, 148 SMs x 128 lanes x 2 x 1.965 GHz (computed)
    flops = 2.0 * window * (shape.body_params() + shape.head_params())
    peak_tf = 1388.8 if shape.mode == 1 else 148 * 128 * 2 * 1.965e9 / 1e12
    cfloor = flops / (peak_tf * 1e12) * 1e3
    d, v = statistics.median(dec), statistics.median(ver)
    return {"shape": shape.name, "dtype": "bf16" if shape.mode == 1 else "f32", "decode_step_ms": d,
            "verify_step_ms": v, "window": window, "hbm_floor_ms": floor, "decode_roofline_frac": floor / d,
            "verify_compute_floor_ms": cfloor, "verify_compute_peak_tflops": peak_tf,
            "verify_roofline_frac": max(floor, cfloor) / v}


def ttfs_roofline(results, pass_floor_ms: float) -> dict:
    """TTFS fraction = Σ floors of the passes in the TTFS window
    / measured TTFS. Every pass that computes rows streams all weights once, so
    its floor is the weight-bytes floor; prefix hits (cost 0) have none."""
    fracs, floors = [], []
    for res in results:
        ev = res.events
        t0 = next((e.payload["arrival_ms"] for e in ev if e.kind == "chunk_received" and e.payload.get("is_final")),
                  None)
        ts = next((e.t_ms for e in ev if e.kind == "sentence_emitted"), None)
        if t0 is None or ts is None or ts <= t0:
            continue
        fl = sum(pass_floor_ms for e in ev if e.kind in ("verify", "generate_step") and t0 < e.t_ms <= ts
                 and e.payload.get("cost_ms", 0.0) > 0.0)
        floors.append(fl)
        fracs.append(fl / (ts - t0))
    if not fracs:
        return {}
    return {"p50_ttfs_floor_ms": statistics.median(floors), "p50_ttfs_roofline_frac": statistics.median(fracs)}


# -- reference arm ------------------------------------------------------------------------------

def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2506_15556_b200.shapes import SHAPES
    shape = SHAPES[args.shape]
    threads = os.cpu_count() or 1
    sched = load_schedule(shape.name)["conversations"]
    lo, hi = timed_ids(world, args.conv_per_step, args.warmup, args.steps)
    ids = [f"c{i:05d}" for i in range(lo, hi)]
    have = [sched[c] for c in ids if c in sched]
    if not have:
        print(json.dumps({"impl": "reference", "unavailable": f"no committed pass schedule for {args.shape}"}))
        return
    per_step = max(2.0, args.cpu_sample_s / max(1, args.steps))
    timer = CpuPassTimer(shape, threads)  # built once: the oracle's weights are the setup cost
    models = []
    for i in range(args.warmup + args.steps):
        m = timer.sample(per_step if i >= args.warmup else 1.0)
        if i >= args.warmup:
            models.append(m)
    model = {k: statistics.median(m[k] for m in models) for k in ("decode_ms", "a_ms", "b_ms_per_row")}
    # conversations the schedule lacks are priced at the mean of those it has
    total_ms = cpu_schedule_ms(model, have) * len(ids) / len(have)
    rate = len(ids) / (total_ms / 1e3)
    sample = (f"oracle port (numpy fp32, {threads} threads, {cpu_model()}) at the {shape.name} shape: "
              f"decode pass {model['decode_ms']:.1f} ms, wider passes {model['a_ms']:.1f} ms + "
              f"{model['b_ms_per_row']:.2f} ms/row (fit on 8/32/72 rows), over a 128-token context, summed over "
              f"the committed pass schedule of conversations "
              f"{lo}..{hi - 1} ({len(have)}/{len(ids)} scheduled)")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, synthetic vocabulary and conversations)",
            "config": workload_config(args, world),
            "verify_step_ms": model["a_ms"] + 72 * model["b_ms_per_row"],
            "decode_step_ms": model["decode_ms"],
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -- our arm --------------------------------------------------------------------------------------

def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return reference_arm(args)
    world, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        # conversation shards never exchange data: gloo carries the work queue, the timing
        # barrier and a max over two scalars; NCCL stays off the data path.
        import torch.distributed as dist
        dist.init_process_group("gloo")
    from paper_2506_15556_b200 import B200LM, run_conversation, specstream, summarize_percentiles
    from paper_2506_15556_b200.shapes import SHAPES
    from paper_2506_15556_b200.simulate import ConversationQueue
    from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, synthetic_conversations

    shape = SHAPES[args.shape]
    lm = B200LM(shape, seed=0, cost_mode="modeled", device=local, max_seq=2048)
    spec = WorkloadSpec()
    convs = synthetic_conversations(lm.vocab, spec)
    cfg = c5_config(lm.vocab, spec)
    per = args.conv_per_step
    live_sched: dict = {}
    traffic = {"bytes": 0.0, "ms": 0.0, "decode_bytes": 0.0, "decode_ms": 0.0}

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def run_step(s: int):
        first = (s * per * world) % len(convs)
        q = ConversationQueue(per * world, world, tag=f"step{s}")
        n = 0
        while (j := q.claim()) is not None:
            conv = convs[(first + j) % len(convs)]
            lm.schedule = []
            run_conversation(conv.turns, cfg, lm, conversation_id=conv.id)
            live_sched[conv.id] = summarize_schedule(lm.schedule)
            for ctx_len, rows, ms in lm.schedule:
                b = shape.pass_bytes(rows, ctx_len)
                traffic["bytes"] += b
                traffic["ms"] += ms
                if rows == 1:
                    traffic["decode_bytes"] += b
                    traffic["decode_ms"] += ms
            n += 1
        lm.schedule = None
        return n

    for w in range(args.warmup):
        run_step(w)
    for k in traffic:
        traffic[k] = 0.0
    s0 = lm.stats()
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    done = 0
    timed = set()
    for k in range(args.steps):
        before = set(live_sched)
        done += run_step(args.warmup + k)
        timed |= set(live_sched) - before
    torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    s1 = lm.stats()
    device_ms = s1["gpu_ms"] - s0["gpu_ms"]
    delta = {k: s1[k] - s0[k] for k in ("launches", "h2d_bytes", "d2h_bytes", "decode_steps", "rows", "passes")}
    vals = {"elapsed": elapsed_ms, "device": device_ms, "done": float(done)}
    mine = {c: live_sched[c] for c in timed}
    if world > 1:
        t = torch.tensor([elapsed_ms, device_ms], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        n = torch.tensor([float(done)], dtype=torch.float64)
        torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.SUM)
        vals = {"elapsed": float(t[0]), "device": float(t[1]), "done": float(n[0])}
        parts = [None] * world
        torch.distributed.all_gather_object(parts, mine)
        mine = {k: v for p in parts for k, v in p.items()}
    n_conv = int(vals["done"])

    # schedule check against the committed one (what the reference arm prices)
    committed = load_schedule(shape.name)["conversations"]
    matched = sum(1 for c, v in mine.items() if committed.get(c) == v)
    sched_info = {"timed_conversations": len(mine), "match_committed": matched,
                  "passes_per_conversation": sum(v[0] for v in mine.values()) / max(1, len(mine)),
                  "rows_per_conversation": sum(v[1] for v in mine.values()) / max(1, len(mine)),
                  "decode_passes_per_conversation": sum(v[2] for v in mine.values()) / max(1, len(mine))}

    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        hbm, src = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        pass
    weight_bytes = s1["weight_bytes"]
    floor_ms = weight_bytes / (hbm * 1e9) * 1e3

    line = {
        "metric": METRIC, "value": n_conv / (vals["device"] / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": vals["elapsed"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if shape.mode == 1 else "f32",
        "data": "synthetic (random-init weights, synthetic vocabulary and conversations)",
        "config": workload_config(args, world),
        "e2e": {"value": n_conv / (vals["elapsed"] / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": delta["h2d_bytes"] / args.steps,
                "d2h_bytes_per_step": delta["d2h_bytes"] / args.steps},
        "schedule": sched_info,
        # every timed pass's algorithmic bytes (weights + cached KV read + new KV
        # written + embedding rows) over its own device time: the whole workload's HBM roofline
        "workload_hbm": {"algorithmic_bytes": traffic["bytes"], "device_ms": traffic["ms"],
                         "achieved_GBs": traffic["bytes"] / max(traffic["ms"], 1e-9) / 1e6,
                         "frac": traffic["bytes"] / max(traffic["ms"], 1e-9) / 1e6 / hbm,
                         "decode_frac": traffic["decode_bytes"] / max(traffic["decode_ms"], 1e-9) / 1e6 / hbm},
        "gpu_launches": delta["launches"], "passes": delta["passes"], "rows_computed": delta["rows"],
        "clocks": clocks,
    }

    # -- phase 2: measured-cost latency (rank 0) ------------------------------------------
    if rank == 0 and not args.no_latency:
        lm.cost_mode = "measured"
        lm.decode_ms.clear()
        results = []
        for i in TTFS_CONVERSATIONS:
            conv = convs[i % len(convs)]
            results += run_conversation(conv.turns, cfg, lm, conversation_id=conv.id)
        records = [specstream.compute_metrics(r.events) for r in results]
        verify = [e.payload["cost_ms"] for r in results for e in r.events
                  if e.kind == "verify" and e.payload["cost_ms"] > 0]
        ttfs = summarize_percentiles(records)
        line["verify_step_ms"] = {"p50": statistics.median(verify) if verify else None, "count": len(verify),
                                  "hbm_floor_ms": floor_ms,
                                  "roofline_frac": floor_ms / statistics.median(verify) if verify else None}
        line["decode_step_ms"] = {"p50": statistics.median(lm.decode_ms) if lm.decode_ms else None,
                                  "count": len(lm.decode_ms), "hbm_floor_ms": floor_ms,
                                  "roofline_frac": floor_ms / statistics.median(lm.decode_ms)
                                  if lm.decode_ms else None}
        line["ttfs_ms"] = {**{k: v for k, v in ttfs.items() if "ttfs" in k or "nfetfs" in k},
                           **ttfs_roofline(results, floor_ms), "turns": len(records),
                           "conversations": [TTFS_CONVERSATIONS.start, TTFS_CONVERSATIONS.stop - 1],
                           "cost": "measured (CUDA-event ms of every pass)"}
        lm.cost_mode = "modeled"

    # -- bf16 argmax agreement at this shape (rank 0): the oracle as the checker ----------------
    if rank == 0 and not args.no_agreement and shape.mode == 1:
        from oracle.parity import fullshape_agreement
        rec = fullshape_agreement(lm, shape, seed=0, tau=0.1)
        line["bf16_agreement"] = {k: rec[k] for k in (
            "rate", "rows_gap_gt_tau", "tau", "rows", "rate_all_rows", "max_abs_logit_diff", "mean_abs_logit_diff",
            "mismatch_gaps", "shape", "ctx", "window")}
        line["bf16_agreement"]["how"] = ("one 72-row verify pass over a 128-token prompt vs the layer-streamed "
                                         "float64 oracle with the GPU's bf16 rounding points (oracle/parity.py); "
                                         "rate over rows whose oracle top-2 gap > tau, lowest-id ties")

    # -- roofline of the dominant kernel: the decode megakernel pass --------------------------
    prof = lm.profile_decode(steps=8)
    dom = max(prof, key=lambda c: prof[c]["ms"])
    dom_gbs = prof[dom]["bytes"] / (prof[dom]["ms"] * 1e-3) / 1e9
    traffic = None
    ncu_file = ROOT / "profiles" / "ncu_summary.json"
    if ncu_file.exists():
        try:
            traffic = json.loads(ncu_file.read_text()).get(dom, {}).get("dram_bytes_per_launch_class")
        except ValueError:
            traffic = None
    line["roofline"] = {"bound": "hbm",
                        "kernel": ("mega_kernel<decode>: one persistent tcgen05 kernel per 1-row pass"
                                   if dom == "whole_pass" else dom),
                        "achieved": dom_gbs, "peak": hbm, "unit": "GB/s", "frac": dom_gbs / hbm,
                        "traffic": traffic, "peak_source": src, "bytes_per_launch": prof[dom]["bytes"],
                        "ms_per_launch": prof[dom]["ms"]}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        model = cpu_pass_model(shape, args.cpu_sample_s, os.cpu_count() or 1)
        cpu_ms = cpu_schedule_ms(model, list(mine.values()))
        line["cpu_baseline"] = {
            "value": len(mine) / (cpu_ms / 1e3), "unit": UNIT, "cores": model["threads"], "kind": "port",
            "sample": (f"oracle decoder (numpy fp32, {cpu_model()}) at {shape.name}: decode pass "
                       f"{model['decode_ms']:.1f} ms, wider passes {model['a_ms']:.1f} ms + "
                       f"{model['b_ms_per_row']:.2f} ms/row; {sum(model['samples'].values())} sampled passes of "
                       f"1/8/32/72 rows over a 128-token context, "
                       f"summed over this run's pass schedule ({len(mine)} conversations)"),
            "per_pass_ms": model["median_ms"],
        }
        dec, ver = line.get("decode_step_ms", {}).get("p50"), line.get("verify_step_ms", {}).get("p50")
        if dec and ver:  # same pass shapes on both sides: 1-row decode, 72-row verify window
            line["cpu_baseline"]["per_pass_gpu_speedup"] = {"decode_1_row": model["median_ms"]["1"] / dec,
                                                            "verify_72_rows": model["median_ms"]["72"] / ver}
    lm.close()
    if rank == 0 and world == 1 and not args.no_extra:
        # the other BASELINE configs' per-pass latencies on this GPU (not part of `value`):
        # c2 = Qwen2.5-0.5B shape in the fp32 bit-exact mode, c4 = Mistral-7B shape bf16
        line["extra_configs"] = {name: pass_latency(SHAPES[key], hbm)
                                 for name, key in (("c2", "qwen2.5-0.5b"), ("c4_one_gpu", "mistral-7b"))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
