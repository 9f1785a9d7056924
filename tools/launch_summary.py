"""Summarise an ncu --csv launch list: per-kernel count, mean duration, DRAM GB/s."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows:
        k = r["Kernel Name"].split("(")[0][:44]
        m = r["Metric Name"]
        v = float(r["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            agg[k][0] += 1
            agg[k][1] += v
        elif "dram" in m:
            agg[k][2] += v
    print("==", path)
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} n={n:4d} avg_us={t / n / 1e3:9.1f} total_ms={t / 1e6:8.2f} "
              f"GB/s={b / t if t else 0:8.1f}")
