#!/bin/bash
# rows per CTA of the two-sweep Galerkin-level kernel (config-2 bench, RHS/s and the kernels' avg us)
for r in 0 6 12 16 24 32; do
  HZ_S9P_ROWS=$r python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('rows', $r, 'RHS/s', round(d['value'],2), 'pair', k['jacobi2_stencil_c64_L1']['avg_us'], 'zero-pair', k['jacobi2_zero_stencil_c64_L1']['avg_us'], 'MHz', d['clocks']['sm_mhz'])"
done
