"""Parse an `ncu --metrics gpu__time_duration.sum --csv` launch list: mean
duration per kernel name (last N launches of each)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") == "gpu__time_duration.sum":
            d[rec["Kernel Name"][:70]].append(float(rec["Metric Value"].replace(",", "")))
for k, v in d.items():
    tail = v[-10:]
    print(f"{k:72s} n={len(v):4d} mean(last {len(tail)}) = {sum(tail) / len(tail) / 1e3:8.2f} us")
