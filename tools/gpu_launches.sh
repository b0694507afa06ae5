#!/bin/bash
# ncu launch list (per-kernel device time) of one bench step per config
mkdir -p gpurun_out/launches
for c in ${CONFIGS:-c2}; do
  python bench.py --profile-once --config $c > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches/$c.csv \
      python bench.py --profile-once --config $c > /dev/null 2>&1
  echo "$c rc=$?"
  python - "$c" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/launches/{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
for r in rows[1:]:
    print("  ", r[ki][:70], r[vi], r[ui])
PY
done
