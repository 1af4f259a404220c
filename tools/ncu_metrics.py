"""Key metrics + top stall reasons of the first kernel in an .ncu-rep.
    python tools/ncu_metrics.py gpurun_out/x.ncu-rep"""
import csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"]:
    print(f"{k:70s} {d.get(k)}")
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
for v, k in sorted(st, reverse=True)[:10]:
    print(f"{v:12.0f} {k}")
