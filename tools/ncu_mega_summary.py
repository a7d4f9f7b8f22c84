"""Summarise the ncu launch list of `tools/profile_step.py` for the megakernel.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file L.csv python tools/profile_step.py
    python tools/ncu_mega_summary.py L.csv profiles/ncu_summary.json

profile_step.py launches the megakernel as: prefill (128 rows), verify
(72 rows), then 1-row decode steps. ncu serialises launches and runs each
with a cold L2, so absolute times are upper bounds; the DRAM bytes per launch
are what bench.py reports as `roofline.traffic` for the dominant kernel
(key "whole_pass" = one decode step of the megakernel).
"""
import csv
import json
import statistics
import sys
from collections import defaultdict


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.DictReader(line for line in open(src) if not line.startswith("==")))
    launches = defaultdict(dict)  # ID -> metric -> value
    names = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            v = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
        elif unit.lower() in ("kbyte", "kb"):
            v *= 1e3
        elif unit.lower() in ("mbyte", "mb"):
            v *= 1e6
        elif unit.lower() in ("gbyte", "gb"):
            v *= 1e9
        launches[int(r["ID"])][r["Metric Name"]] = v
        names[int(r["ID"])] = r["Kernel Name"]
    mega = [i for i in sorted(launches) if "mega_kernel" in names[i]]
    other_us = sum(launches[i].get("gpu__time_duration.sum", 0.0) for i in launches if i not in mega)

    def summ(ids):
        us = [launches[i]["gpu__time_duration.sum"] for i in ids]
        rd = [launches[i].get("dram__bytes_read.sum", 0.0) for i in ids]
        wr = [launches[i].get("dram__bytes_write.sum", 0.0) for i in ids]
        tot = [a + b for a, b in zip(rd, wr)]
        return {"n": len(ids), "avg_us": round(statistics.mean(us), 2),
                "dram_read_bytes_per_launch": round(statistics.mean(rd)),
                "dram_write_bytes_per_launch": round(statistics.mean(wr)),
                "dram_bytes_per_launch_class": round(statistics.mean(tot)),
                "dram_GBps": round(statistics.mean(tot) / (statistics.mean(us) * 1e-6) / 1e9, 1)}

    out = {
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none python tools/profile_step.py (llama-3-8b shape, bf16; ncu "
                  "serialises launches and flushes caches between them, so times are cold-L2 upper bounds)",
        "prefill_128_rows": summ(mega[:1]),
        "verify_72_rows": summ(mega[1:2]),
        "whole_pass": summ(mega[2:]),
        "other_kernels_us_total": round(other_us, 1),
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
