"""Summarise an ncu report (raw page) for the roofline / pipe metrics we track."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"]
out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"]).decode()
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("kernel:", d.get("Kernel Name", "")[:110])
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k]:>16s} {u[h.index(k)]}")
    stalls = [(k, float(d[k].replace(",", ""))) for k in h
              if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio") and d[k]]
    stalls.sort(key=lambda t: -t[1])
    print("  top stall reasons (cycles per issued instruction):",
          ", ".join(f"{k.split('stalled_')[1].replace('_per_issue_active.ratio', '')}={v:.2f}" for k, v in stalls[:6]))
