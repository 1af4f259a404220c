"""Per-source-line stall samples of one kernel in an .ncu-rep (needs -lineinfo).
    python tools/ncu_lines.py gpurun_out/x.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
agg = []
for r in rows:
    if len(r) == len(hdr) and r[2] == "-":
        try:
            agg.append((int(r[si]), int(r[ii]), r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
print(f"total samples {tot}, warp instructions {sum(a[1] for a in agg)}")
for a in sorted(agg, reverse=True)[:top]:
    print(f"{a[0]:7d} {100 * a[0] / tot:5.1f}%  inst {a[1]:10d}  L{a[2]:>4s}  {a[3]}")
