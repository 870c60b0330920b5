"""Prints an ncu --csv launch list (one line per launch, selected metrics)."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [n for n, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    if len(r) == len(h):
        d.setdefault((int(r[ii]), r[ki][:48]), {})[r[mi]] = r[vi]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
short = {"gpu__time_duration.sum": "ns", "smsp__inst_executed.sum": "inst",
         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
         "lts__t_bytes.sum": "L2B", "dram__bytes_read.sum": "dramR"}
for (i, k), m in sorted(d.items())[-last:]:
    print(i, k, " ".join(f"{short.get(a, a)}={b}" for a, b in m.items()))
