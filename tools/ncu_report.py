"""Summarise `ncu --set full` captures as a markdown table (one row per launch).

usage: python tools/ncu_report.py REP [REP ...]
Reads --page raw --csv of each capture: duration, DRAM bytes, throughput,
registers, shared memory, occupancy, L1/L2 hit rates."""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us", 1.0),
    ("dram__bytes_read.sum", "DRAM rd MB", None),
    ("dram__bytes_write.sum", "DRAM wr MB", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__shared_mem_per_block_dynamic", "dyn smem", 1.0),
    ("launch__grid_size", "grid", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1.0),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
]
_MB = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = {}
        for key, label, scale in COLS:
            if key not in h:
                continue
            i = h.index(key)
            v = float(row[i].replace(",", "")) if row[i] not in ("", "n/a") else float("nan")
            if scale is None:
                v *= _MB.get(units[i], 1.0)
            elif key == "gpu__time_duration.sum" and units[i] == "ms":
                v *= 1e3
            elif key == "gpu__time_duration.sum" and units[i] == "ns":
                v *= 1e-3
            d[label] = v
        yield row[h.index("Kernel Name")], d


if __name__ == "__main__":
    labels = [c[1] for c in COLS]
    print("| capture | kernel | " + " | ".join(labels) + " |")
    print("|---|---|" + "---|" * len(labels))
    for rep in sys.argv[1:]:
        for name, d in rows(rep):
            vals = " | ".join(f"{d.get(l, float('nan')):.1f}" for l in labels)
            print(f"| {rep.split('/')[-1]} | `{name[:60]}` | {vals} |")
