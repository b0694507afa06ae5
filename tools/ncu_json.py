#!/usr/bin/env python
"""ncu --set full report of one fused-kernel launch -> profiles/ncu_<variant>_<cfg>.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic).
usage: tools/ncu_json.py <report.ncu-rep> <cfg> [variant]"""
import csv
import io
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
variant = sys.argv[3] if len(sys.argv) > 3 else "fused"
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True, check=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
m = dict(zip(h, v))
unit = dict(zip(h, u))


def num(name):
    x = float(m[name].replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
             "s": 1.0}.get(unit.get(name, ""), 1.0)
    return x * scale


out = {
    "kernel": m.get("Kernel Name", ""),
    "config": cfg,
    "source": f"ncu --set full --clock-control none, one launch ({rep.split('/')[-1]}); cold L2 (ncu replay)",
    "gpu_time_s": num("gpu__time_duration.sum"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
}
out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
for k, name in (("fma_pipe_active_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                ("fma_pipe_inst_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                ("registers_per_thread", "launch__registers_per_thread"),
                ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")):
    out[k] = num(name)
path = f"profiles/ncu_{variant}_{cfg}.json"
json.dump(out, open(path, "w"), indent=1)
print(path, json.dumps(out))
