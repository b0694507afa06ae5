#!/usr/bin/env python
"""Stall samples per CUDA source line of an ncu report (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = None, None
rows = []
# ncu does not escape quotes inside the source text (asm("...")): split on '","'
for line in out.splitlines():
    r = line.strip()[1:-1].split('","') if line.strip() else []
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    d["Line No"], d["Source"] = r[0], r[1]
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
        ex = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    stalls = collections.Counter()
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[k[6:]] += int(v)
            except ValueError:
                pass
    rows.append((s, ex, fname, d["Line No"], d["Source"].strip()[:70], stalls))
tot = sum(r[0] for r in rows) or 1
print(f"total samples {tot}")
for s, ex, f, ln, src, st in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100 * s / tot:5.1f}% exec {ex:>11d} {f}:{ln:<5s} {src:70s} {[(k, v) for k, v in st.most_common(3)]}")
