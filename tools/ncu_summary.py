#!/usr/bin/env python
"""Key counters of one ncu --set full report (the roofline's `traffic`, the
bound, warp efficiency) plus the top source lines by stall samples.
usage: ncu_summary.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = sys.argv[2] if len(sys.argv) > 2 else "20"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]} {rows[1][h.index(w)]}")
stalls = [(float(v[i]), x) for i, x in enumerate(h)
          if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued") and v[i].replace(".", "").isdigit()]
tot = sum(s for s, _ in stalls) or 1.0
print("stall samples (share):", ", ".join(f"{x.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * s / tot:.1f}%"
                                          for s, x in sorted(stalls, reverse=True)[:8]))
print()
print(subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, top],
                     capture_output=True, text=True).stdout)
