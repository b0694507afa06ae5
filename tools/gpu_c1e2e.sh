for r in 1 2; do
for g in - 7 8 4 1; do
  if [ "$g" = - ]; then unset FBF_GROUPS; else export FBF_GROUPS=$g; fi
  python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$r groups=$g', round(d['value']), round(d['e2e']['value']), round(d['roofline']['kernel_ms']*1000,1),'us')"
done; done
unset FBF_GROUPS
FBF_GRAPH_DEBUG=1 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep "fbf host" | sort | uniq -c
python tools/host_overhead.py
