#!/bin/bash
for m in 100000 30000 8000 0; do
  HZ_S9_PAIR_MIN_NODES=$m python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('min_nodes', $m, 'RHS/s', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'MHz', d['clocks']['sm_mhz'], 'launches', d['gpu_launches'])"
done
