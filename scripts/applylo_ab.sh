#!/bin/bash
for rep in 1 2; do for v in 1 0; do
  HZ_APPLY_LO2=$v python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('HZ_APPLY_LO2=$v rep $rep RHS/s', round(d['value'],2), 'apply', d['kernels']['apply_fine_c128']['avg_us'], 'MHz', d['clocks']['sm_mhz'])"
done; done
