"""Top stall reasons of an `ncu --page source --csv` export (SASS or source view):
python tools/ncu_stalls.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
for d in data:
    for c in stall_cols:
        try:
            tot[c] += float(d[c] or 0)
        except ValueError:
            pass
s = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{k[6:]}={v / s:.1%}" for k, v in tot.most_common(10)))
key = "Warp Stall Sampling (All Samples)"
data.sort(key=lambda d: -float(d.get(key) or 0))
for d in data[:top]:
    reasons = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{float(d[key] or 0):7.0f}  {d.get('Address', '')[:8]:8s} {d['Source'][:90]:90s} "
          + " ".join(f"{r}={v:.0f}" for v, r in reasons if v))
