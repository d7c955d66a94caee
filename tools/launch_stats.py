"""Per-kernel statistics of an ncu launch list (gpurun_out/launches.csv)."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.defaultdict(list)
order = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    key = (r["Kernel Name"].split("(")[0][-48:], r["Grid Size"])
    agg[key].append(float(r["Metric Value"]))
    order.append(key)
tot = sum(sum(v) for v in agg.values())
for (k, g), v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:48s} {g:>14s} n={len(v):4d} total={sum(v) / 1e3:8.1f}us mean={sum(v) / len(v) / 1e3:7.2f}us "
          f"share={sum(v) / tot:5.3f}")
