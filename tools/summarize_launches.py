"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(line for line in open(sys.argv[1]) if not line.startswith("==")))
by = defaultdict(list)
order = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0][:60]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    v = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
    by[name].append(v)
    order.append((r["ID"], name, v, r.get("Grid Size", ""), r.get("Block Size", "")))
tot = sum(sum(v) for v in by.values())
print(f"{'kernel':60s} {'n':>6s} {'sum_us':>10s} {'avg_us':>8s} {'share':>6s}")
for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} {len(v):6d} {sum(v):10.1f} {sum(v)/len(v):8.2f} {sum(v)/tot:6.1%}")
print("total_us", round(tot, 1))
if len(sys.argv) > 2:
    for o in order[-int(sys.argv[2]):]:
        print(o)
