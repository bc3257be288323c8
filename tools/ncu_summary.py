"""Key metrics of every kernel in one ncu --set full report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u = r[0], r[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "local_load", "lts__t_bytes.sum"]
for v in r[2:]:
    for k in keys:
        for i, n in enumerate(h):
            if n == k or (k == "local_load" and "local" in n and n.endswith(".sum") and "inst" in n):
                print(f"{n:70s} {v[i]:>20s} {u[i]}")
    stalls = [(float(v[i]), n) for i, n in enumerate(h)
              if "average_warps_issue_stalled" in n and n.endswith("per_issue_active.ratio") and v[i] not in ("", "n/a")]
    for val, n in sorted(stalls, reverse=True)[:8]:
        print(f"  stall {n.split('stalled_')[1].split('_per')[0]:28s} {val:.3f}")
    print()
