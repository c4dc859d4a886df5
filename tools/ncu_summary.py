"""Condense an ncu raw page (CSV, `ncu -i rep --page raw --csv`) to the
per-kernel columns kept under profiles/ (r01_ncu_full_stack_v*.csv).
Usage: python tools/ncu_summary.py raw.csv > profiles/<name>.csv"""
import csv
import sys

COLS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
idx = [h.index(c) for c in COLS if c in h]
w = csv.writer(sys.stdout)
for r in rows:
    w.writerow([r[i] for i in idx])
