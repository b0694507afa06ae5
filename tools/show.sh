#!/bin/bash
# print bench summaries (+ ncu summary/regions if a report is given)
cd "$(dirname "$0")/.."
for f in gpurun_out/bench_*.json; do
python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).readline()); r=d['roofline']
    print(sys.argv[1].split('bench_')[1][:-5], round(d['value'],1), 'Mpx/s frac', round(r['frac'],3), 'kernel_ms', round(r['kernel_ms'],3), 'e2e', round(d.get('e2e',{}).get('value',0) or 0,1))
except Exception as e: print(sys.argv[1], 'unreadable', e)
PY
done
if [ -n "$1" ]; then python tools/ncu_summary.py "$1" 0 2>/dev/null | sed -n 3,22p; python tools/ncu_regions.py "$1" 150; fi
