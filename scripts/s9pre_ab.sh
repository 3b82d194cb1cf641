#!/bin/bash
# fused level-1 pre-visit kernel on/off, interleaved repetitions (config-2 bench)
for rep in 1 2; do for v in 1 0; do
  HZ_S9_PRE=$v python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('HZ_S9_PRE=$v rep $rep RHS/s', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'MHz', d['clocks']['sm_mhz'])"
done; done
for r in 2 8 16; do
  HZ_S9_PRE=1 HZ_S9PRE_ROWS=$r python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('HZ_S9_PRE=1 coarse rows $r RHS/s', round(d['value'],2), 'pre', d['kernels']['fused_pre_stencil_c64_L1']['avg_us'], 'MHz', d['clocks']['sm_mhz'])"
done
