"""Average per-kernel metrics of an ncu --csv launch list (last 20 launches each)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        agg[(d["Kernel Name"][:48], d["Metric Name"])].append(float(d["Metric Value"].replace(",", "")))
for k, v in sorted(agg.items()):
    print(f"{k[0]:50s} {k[1]:55s} n={len(v):3d} avg={sum(v[-20:]) / len(v[-20:]):.1f}")
