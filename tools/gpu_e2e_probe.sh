#!/bin/bash
# batch pipeline chunk count (c5, 256 images): e2e through the host entry
for k in 8 12 16; do
  FBF_HOST_BATCH_CHUNKS=$k python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chunks=$k', round(d['value']), round(d['e2e']['value']))"
done
