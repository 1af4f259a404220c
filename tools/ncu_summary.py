"""Summarise ncu output for profiles/: a launch list (csv from
`ncu --metrics gpu__time_duration.sum --csv`) and/or a full capture (.ncu-rep).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/x.ncu-rep --out profiles/r1_x.md
"""

import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "gpc__cycles_elapsed.max.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((int(d["ID"]), d["Kernel Name"], float(d["Metric Value"]), d["Metric Unit"]))
    return out


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for i, name in enumerate(h):
            if name in KEYS or name == "Kernel Name":
                d[name] = (v[i], u[i])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        L = launches(a.launches)
        lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
                  "| id | kernel | time | unit |", "|---|---|---|---|"]
        for i, n, t, u in L:
            lines.append(f"| {i} | `{n[:90]}` | {t:.0f} | {u} |")
        lines.append("")
    for rep in a.rep:
        for d in raw(rep):
            lines += [f"## Full capture: `{d.get('Kernel Name', ('?',))[0][:100]}` ({rep.split('/')[-1]})", "",
                      "| metric | value | unit |", "|---|---|---|"]
            for k in KEYS:
                if k in d:
                    lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            lines.append("")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
