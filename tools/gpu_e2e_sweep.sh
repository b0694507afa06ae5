#!/bin/bash
# host-pipeline sweep for the e2e path: strip count x edge-strip weight (c2), chunk count (c4)
for k in 2 3 4 5; do for e in 15 20 30; do
  FBF_HOST_CHUNKS=$k FBF_HOST_EDGE=$e python bench.py --config ${CFG:-c2} --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('K=$k edge=$e', round(d['value']), 'e2e', round(d['e2e']['value']))"
done; done
python bench.py --config ${CFG:-c2} --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('default', round(d['value']), 'e2e', round(d['e2e']['value']))"
