"""Per-kernel breakdown of one c2 decode step and the 72-row verify pass from an
ncu launch list of tools/c2_prof.py: python tools/c2_breakdown.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
seq = [(r["Kernel Name"].split("(")[0][:44], float(r["Metric Value"].replace(",", "")) / 1000, r["Grid Size"])
       for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
starts = [i for i, s in enumerate(seq) if s[0].startswith("void embed_norm")]
for lo, hi, label in ((starts[1], starts[2], "verify-72"), (starts[-1], len(seq), "decode")):
    d, n = defaultdict(float), defaultdict(int)
    for k, v, _ in seq[lo:hi]:
        d[k] += v
        n[k] += 1
    tot = sum(d.values())
    print(f"{label}: {tot:.1f} us of serialized kernel time")
    for k in sorted(d, key=lambda k: -d[k]):
        print(f"  {k:44s} {n[k]:4d} {d[k]:9.1f} us {d[k] / tot:6.1%}")
    print("  first layer:", [(k.replace('void ', ''), round(v, 1), g) for k, v, g in seq[lo + 1:lo + 11]])
