#!/usr/bin/env python
"""Bucket ncu SASS stall samples into contiguous regions (for locating hot phases)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
hdr = rows[1]; data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
stall_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[i_s]) for r in data)
for b0 in range(0, len(data), bucket):
    chunk = data[b0:b0 + bucket]
    s = sum(int(r[i_s]) for r in chunk)
    if s < tot * 0.01: continue
    ops = collections.Counter(r[i_src].split()[0] if not r[i_src].strip().startswith('@') else r[i_src].split()[1] for r in chunk)
    st = collections.Counter()
    for r in chunk:
        for j in stall_cols:
            try: st[hdr[j]] += int(r[j])
            except: pass
    ex = sum(int(r[i_ex]) for r in chunk)
    print(f"[{b0:5d},{b0+len(chunk):5d}) {100*s/tot:5.1f}%  exec {ex:>10d}  ops {dict(ops.most_common(4))}  stalls {[(k.replace('stall_',''),v) for k,v in st.most_common(3)]}")
