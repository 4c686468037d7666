"""Summarise every kernel of .ncu-rep files (the metrics profiles/ quotes):
python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]

for path in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"## {path.split('/')[-1].replace('.ncu-rep', '')}")
    for row in rows[2:]:
        print(f"      {'Kernel Name':62s} {row[h.index('Kernel Name')][:110]}")
        for k in KEYS:
            if k in h:
                print(f"      {k:62s} {row[h.index(k)]} {units[h.index(k)]}")
        st = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
        tot = sum(float(row[h.index(k)] or 0) for k in st) or 1.0
        top = sorted(((float(row[h.index(k)] or 0) / tot, k[33:]) for k in st), reverse=True)[:6]
        print("      stall share: " + ", ".join(f"{n}={v:.2f}" for v, n in top))
        print()
