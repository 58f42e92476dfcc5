"""Key metrics + stall reasons of an ncu report (first kernel).
usage: python tools/ncu_digest.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__sass_inst_executed_op_local_ld.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    print(f"{k:60s} {d.get(k)}")
st = []
for k, v in d.items():
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v), k.split("stalled_")[1].split("_per")[0]))
        except ValueError:
            pass
print("stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
