"""Per-phase timeline of megakernel passes (PS_TRACE=1): decode step and a 72-row verify."""
import collections, ctypes, os, sys
from pathlib import Path
os.environ["PS_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2506_15556_b200 import B200LM
from paper_2506_15556_b200.shapes import LLAMA3_8B
shape = LLAMA3_8B
lm = B200LM(shape, seed=1, max_seq=1024, cost_mode="measured")
rng = np.random.default_rng(0)
toks = [int(t) for t in rng.integers(4, shape.vocab, int(sys.argv[1]) if len(sys.argv) > 1 else 100)]
lm.forward(toks)
for rep in range(3):
    lm.truncate(len(toks))
    steps = lm.decode_greedy_fused(toks, 3)
NS = 16
names = ["EMB"] + [k for l in range(shape.layers) for k in ("QKV", "ATT", "O", "GU", "D")] + ["LM", "FIN"]

def grab():
    np_, ct = ctypes.c_int32(), ctypes.c_int32()
    lm._call("ps_trace", None, 0, ctypes.byref(np_), ctypes.byref(ct))
    buf = np.zeros(np_.value * ct.value * NS, dtype=np.uint64)
    lm._call("ps_trace", buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), buf.size, ctypes.byref(np_),
             ctypes.byref(ct))
    tr = buf.reshape(np_.value, ct.value, NS).astype(np.float64)
    t0 = tr[0, :, 2][tr[0, :, 2] > 0].min()
    # slots this pass did not write still hold an earlier pass's stamps: drop them
    return np.where(tr >= t0, (tr - t0) / 1000.0, np.nan)

def report(tr, label):
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for p in range(1, tr.shape[0]):
        start = np.nanmax(tr[p - 1, :, 2])
        a = agg[names[p]]
        a["span"].append(np.nanmax(tr[p, :, 2]) - start)
        for slot, key in ((0, "prod_bar"), (12, "prod_done"), (13, "mma_done"), (1, "bar"), (3, "fin_issued"), (4, "acc_last"), (5, "published"), (7, "waited|a_start"), (8, "a_loaded"), (14, "a_S|fin_landed"), (15, "a_softmax|fin_computed"), (9, "a_computed"), (10, "a_counted|fin_fenced"), (11, "a_merged"), (6, "deferred")):
            col = tr[p, :, slot]
            if np.isfinite(col).any():
                a[key + "_max"].append(np.nanmax(col) - start)
                a[key + "_med"].append(np.nanmedian(col) - start)
    for k, a in agg.items():
        print(label, k, " ".join(f"{kk}={np.mean(v):.1f}" for kk, v in a.items()))

print("decode step ms", [round(c, 3) for _, c in steps])
report(grab(), "decode")
lm.truncate(len(toks) - 8)
v = lm.verify_greedy_detail(toks, [5] * 64)
print("verify gpu ms", v["gpu_ms"])
report(grab(), "verify")
# per-CTA straggler view of the decode step (slot 4 = last accumulator seen)
lm.truncate(len(toks))
lm.decode_greedy_fused(toks, 2)
tr = grab()
for p in (6, 8, 9, 10):  # layer-1 QKV, O, GU, D
    start = np.nanmax(tr[p - 1, :, 2])
    acc = tr[p, :, 4] - start
    order = np.argsort(-np.nan_to_num(acc, nan=-1))
    print(names[p], "slowest CTAs", [(int(i), round(float(acc[i]), 1)) for i in order[:10]],
          "median", round(float(np.nanmedian(acc)), 1))
