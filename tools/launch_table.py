"""Per-launch table of an ncu --metrics gpu__time_duration.sum CSV (last `n` launches).
    python tools/launch_table.py file.csv [n]"""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
data = [(int(r[ii]), r[ki][:80], float(r[vi].replace(",", ""))) for r in rows[1:]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
tot = 0.0
for d in data[-n:]:
    tot += d[2]
    print(f"{d[0]:4d} {d[2] / 1e3:9.1f} us  {d[1]}")
print(f"total {tot / 1e3:.1f} us over {min(n, len(data))} launches")
