"""Print the kernels of the last full reconstruct call from an ncu launch-list CSV."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
rows = rows[1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[ki][:44], float(r[vi].replace(",", ""))) for r in rows]
first = sys.argv[2] if len(sys.argv) > 2 else "tile_kernel"
idx = [i for i, (k, v) in enumerate(seq) if first in k]
last = seq[idx[-2]:idx[-1]]
tot = 0
for k, v in last:
    print(f"{k:44s} {v / 1000:8.2f} us")
    tot += v
print("sum us", tot / 1000)
