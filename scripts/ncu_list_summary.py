"""Summarise an ncu --csv launch list (gpu__time_duration.sum): time per kernel
name (and per grid for the GEMM), share of the total."""
import collections
import csv
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    name = r["Kernel Name"].split("(")[0][:60]
    key = f"{name} grid={r.get('Grid Size', '')}"
    tot[key] += ms
    cnt[key] += 1
allms = sum(tot.values())
print(f"total {allms:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"  {v:8.3f} ms {100 * v / allms:5.1f}%  x{cnt[k]:4d}  {k}")
