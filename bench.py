"""Benchmark: PredGen predict-and-verify conversation simulation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (config c5 of BASELINE.json): synthetic MT-Bench/Lmsys-length
conversations on the Llama-3-8B shape (bf16, random init, measured-cost
SimClock), sharded one stream per GPU (weak scaling: every rank simulates
`--conv-per-step` conversations per step). A "step" = that batch of
conversations through the public API (`run_conversation` -> verify / decode
-> B200LM -> C-ABI -> CUDA). One JSON line on rank 0:

* value: conversations/s over the device time of every pass (inputs are
  token ids already resident in pinned host memory; host orchestration
  excluded) — max over ranks;
* e2e: conversations/s over the CUDA-event-bracketed wall time of the steps
  (host Python loop, H2D token copies and D2H argmax reads included);
* verify-step latency (p50 ms of the fused verify calls), decode-step
  latency, simulated p50 TTFS under measured cost — the BASELINE metrics;
* roofline for the dominant kernel class (gate/up tcgen05 GEMM), measured
  with CUDA events around each launch (ps_profile_decode);
* cpu_baseline: the oracle decoder (numpy fp32, all host threads) timed on a
  bounded sample of the same 8B-shape passes, converted to conversations/s
  with this run's pass mix.

`--impl reference` times the reference's CPU path for this workload: the
reference has no decoder (its LM is a hash table, lm.py:216-243), so its
stand-in is the oracle port (oracle/decoder.py), rank 0 only.
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

METRIC = "conversations/sec (c5 predict-and-verify simulation); verify-step latency; simulated p50 TTFS"
UNIT = "conversations/s"

# pass mix of one c5 conversation on the 8B shape, measured by this bench
# (bench.py --steps 8, 2026-10-17; refreshed from the live run when available)
DEFAULT_PASS_MIX = {"decode_rows": 180.0, "extend_rows": 420.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--conv-per-step", type=int, default=2)
    ap.add_argument("--shape", default="llama-3-8b")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    return ap.parse_args()


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


def cpu_port_timing(shape, sample_s: float, threads: int, context: int = 128, window: int = 72) -> dict:
    """Oracle decoder (numpy fp32, BLAS on `threads` host threads) per-pass times at `shape`.

    Every layer streams layer 0's weights (share_layer_weights): the same bytes
    and FLOPs per pass as the full model, without generating 8B values on the
    host. Returns ms for a 1-row decode pass and a `window`-row verify pass.
    """
    import numpy as np
    from oracle.decoder import DecoderOracle
    t0 = time.perf_counter()
    d = dict(shape.as_dict())
    d["mode"] = 0  # fp32 arithmetic: no bf16 rounding emulation in the timed port
    m = DecoderOracle(d, seed=0, dtype=np.float32, share_layer_weights=True)
    rng = np.random.default_rng(0)
    m.extend([int(t) for t in rng.integers(4, shape.vocab, context)])
    setup_s = time.perf_counter() - t0
    dec, ver = [], []
    deadline = time.perf_counter() + sample_s
    base = len(m.tokens)
    while time.perf_counter() < deadline or len(dec) < 2 or len(ver) < 1:
        t = time.perf_counter()
        m.extend([int(rng.integers(4, shape.vocab))])
        dec.append((time.perf_counter() - t) * 1e3)
        if len(dec) % 4 == 0:
            m.truncate(base)
            t = time.perf_counter()
            m.extend([int(x) for x in rng.integers(4, shape.vocab, window)])
            ver.append((time.perf_counter() - t) * 1e3)
            m.truncate(base)
        if len(dec) > 64:
            break
    return {"decode_ms": statistics.median(dec), "verify_ms": statistics.median(ver), "decode_samples": len(dec),
            "verify_samples": len(ver), "setup_s": setup_s, "threads": threads}


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


def conv_rate_from_passes(t: dict, mix: dict) -> float:
    per_conv_ms = mix["decode_rows"] * t["decode_ms"] + mix["extend_rows"] / 72.0 * t["verify_ms"]
    return 1000.0 / per_conv_ms


def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2506_15556_b200.shapes import SHAPES
    shape = SHAPES[args.shape]
    threads = os.cpu_count() or 1
    per_step = max(2.0, args.cpu_sample_s / max(1, args.steps + args.warmup))
    times = []
    t = None
    for i in range(args.warmup + args.steps):
        t = cpu_port_timing(shape, per_step if i >= args.warmup else 1.0, threads)
        if i >= args.warmup:
            times.append(t)
    dec = statistics.median(x["decode_ms"] for x in times)
    ver = statistics.median(x["verify_ms"] for x in times)
    rate = conv_rate_from_passes({"decode_ms": dec, "verify_ms": ver}, DEFAULT_PASS_MIX)
    sample = (f"oracle port (numpy fp32, {threads} threads) at the {shape.name} shape: median of 1-row decode and "
              f"72-row verify passes over a 128-token context; conversations/s = 1 / (decode_rows*t_dec + "
              f"extend_rows/72*t_verify) with the c5 pass mix {DEFAULT_PASS_MIX}")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / rate, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "c5: synthetic MT-Bench/Lmsys-length conversations", "shape": shape.name},
            "verify_step_ms": ver, "decode_step_ms": dec,
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    world, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        # The conversation shards never exchange data; the only collectives are
        # the timing barrier and a max over two scalars, so gloo (host) is used
        # and NCCL stays off the data path.
        import torch.distributed as dist
        dist.init_process_group("gloo")
    from paper_2506_15556_b200 import B200LM, summarize_percentiles
    from paper_2506_15556_b200.shapes import SHAPES
    from paper_2506_15556_b200.workload import WorkloadSpec, c5_config, shard, simulate, synthetic_conversations

    shape = SHAPES[args.shape]
    lm = B200LM(shape, seed=0, cost_mode="measured", device=local, max_seq=2048)
    spec = WorkloadSpec()
    convs = synthetic_conversations(lm.vocab, spec)
    cfg = c5_config(lm.vocab, spec)
    mine = shard(convs, rank, world)
    per = args.conv_per_step
    need = (args.warmup + args.steps) * per
    if need > len(mine):
        mine = (mine * (need // max(1, len(mine)) + 1))[:need]

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for w in range(args.warmup):
        simulate(mine[w * per:(w + 1) * per], cfg, lm)
    s0 = lm.stats()
    lm.verify_ms.clear()
    lm.decode_ms.clear()
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    records, results = [], []
    base = args.warmup * per
    for k in range(args.steps):
        r, res = simulate(mine[base + k * per: base + (k + 1) * per], cfg, lm)
        records += r
        results += res
    torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    s1 = lm.stats()
    device_ms = s1["gpu_ms"] - s0["gpu_ms"]
    launches = s1["launches"] - s0["launches"]
    h2d = s1["h2d_bytes"] - s0["h2d_bytes"]
    d2h = s1["d2h_bytes"] - s0["d2h_bytes"]
    decode_rows = s1["decode_steps"] - s0["decode_steps"]
    all_rows = s1["rows"] - s0["rows"]
    n_conv = args.steps * per
    ttfs = summarize_percentiles(records)
    verify_nonzero = [x for x in lm.verify_ms if x > 0]
    vals = {"elapsed": elapsed_ms, "device": device_ms}
    if world > 1:
        t = torch.tensor([elapsed_ms, device_ms], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        vals = {"elapsed": float(t[0]), "device": float(t[1])}
    # roofline of the dominant kernel class, CUDA events around every launch
    prof = lm.profile_decode(steps=8)
    dom = max(("gate_up_gemm", "down_gemm", "qkv_gemm", "o_gemm", "lm_head", "whole_pass"),
              key=lambda c: prof[c]["ms"])
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        hbm, src = float(peaks["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        hbm, src = 6650.0, "fallback"
    dom_gbs = prof[dom]["bytes"] / (prof[dom]["ms"] * 1e-3) / 1e9
    step_ms = statistics.median(lm.decode_ms) if lm.decode_ms else None
    traffic = None
    ncu_file = ROOT / "profiles" / "ncu_summary.json"
    if ncu_file.exists():
        try:
            traffic = json.loads(ncu_file.read_text()).get(dom, {}).get("dram_bytes_per_launch_class")
        except ValueError:
            traffic = None
    line = {
        "metric": METRIC, "value": world * n_conv / (vals["device"] / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": vals["elapsed"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if shape.mode == 1 else "f32",
        "data": "synthetic (random-init weights, synthetic vocabulary and conversations)",
        "config": {"workload": "c5: synthetic MT-Bench/Lmsys-length conversations, Llama-3-8B shape, bf16, "
                               "measured-cost SimClock", "shape": shape.name, "conversations_per_rank_per_step": per,
                   "chunk_words": cfg.chunk_words, "max_response_tokens": cfg.max_response_tokens,
                   "l2": "inputs larger than L2 (15 GB of weights streamed per pass)",
                   "parallelism": f"{world} independent conversation shards (no per-pass collective)"},
        "e2e": {"value": world * n_conv / (vals["elapsed"] / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps},
        "verify_step_ms": {"p50": statistics.median(verify_nonzero) if verify_nonzero else None,
                           "count": len(verify_nonzero),
                           # a verify window streams the same weights once: same HBM floor
                           "hbm_floor_ms": lm.stats()["weight_bytes"] / (hbm * 1e9) * 1e3,
                           "roofline_frac": (lm.stats()["weight_bytes"] / (hbm * 1e9) * 1e3
                                             / statistics.median(verify_nonzero)) if verify_nonzero else None},
        "decode_step_ms": {"p50": step_ms, "count": len(lm.decode_ms),
                           "hbm_floor_ms": lm.stats()["weight_bytes"] / (hbm * 1e9) * 1e3},
        "ttfs_ms": {**{k: v for k, v in ttfs.items() if "ttfs" in k or "nfetfs" in k},
                    **ttfs_roofline(results, lm.stats()["weight_bytes"] / (hbm * 1e9) * 1e3)},
        "turns": len(records),
        "roofline": {"bound": "hbm",
                     "kernel": ("mega_kernel: whole 1-row decode pass, one persistent tcgen05 kernel" if dom == "whole_pass"
                                else f"{dom} (tcgen05 weight-streaming GEMM, 1-row decode step)"),
                     "achieved": dom_gbs, "peak": hbm, "unit": "GB/s", "frac": dom_gbs / hbm, "traffic": traffic,
                     "peak_source": src, "per_class_ms": {k: v["ms"] for k, v in prof.items()},
                     "decode_step_frac": (lm.stats()["weight_bytes"] / (step_ms * 1e-3) / 1e9 / hbm)
                     if step_ms else None},
        "gpu_launches": launches, "rows_computed": all_rows, "decode_steps": decode_rows,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mix = {"decode_rows": decode_rows / n_conv, "extend_rows": (all_rows - decode_rows) / n_conv}
        t = cpu_port_timing(shape, args.cpu_sample_s, os.cpu_count() or 1)
        rate = conv_rate_from_passes(t, mix)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": t["threads"], "kind": "port",
            "sample": (f"oracle decoder (numpy fp32) at {shape.name}: {t['decode_samples']} decode + "
                       f"{t['verify_samples']} 72-row passes over a 128-token context (median "
                       f"{t['decode_ms']:.0f} / {t['verify_ms']:.0f} ms), scaled by this run's pass mix "
                       f"{ {k: round(v, 1) for k, v in mix.items()} } per conversation"),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    lm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
