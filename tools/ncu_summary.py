#!/usr/bin/env python
"""Summarise an ncu --set full report: headline metrics, stall reasons, hottest SASS."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "smsp__warps_eligible.avg.per_cycle_active"]
for name, unit, val in zip(h, u, v):
    if name in want:
        print(f"{name:70s} {unit:8s} {val}")
stalls = [(name, float(val.replace(",", ""))) for name, val in zip(h, v)
          if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued")]
tot = sum(x for _, x in stalls) or 1
print("--- stall samples (share)")
for name, x in sorted(stalls, key=lambda t: -t[1])[:12]:
    print(f"  {name.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {x:9.0f} {100 * x / tot:5.1f}%")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
print(f"--- hottest {top} SASS instructions (index, samples, instr)")
idx = sorted(range(len(data)), key=lambda k: -int(data[k][i_s]))[:top]
for k in sorted(idx):
    print(f"  {k:5d} {data[k][i_s]:>6s}  {data[k][i_src].strip()[:90]}")
