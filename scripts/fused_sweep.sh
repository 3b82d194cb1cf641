set -x
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -x -q > gpurun_out/fused_tests.log 2>&1; echo "exit $?" >> gpurun_out/fused_tests.log
for v in "HZ_FUSED_NT=128" "HZ_FUSED_NT=64" "HZ_FUSED_NT=128 HZ_FUSED_PRE_ROWS=32 HZ_FUSED_POST_ROWS=64" "HZ_FUSED_NT=64 HZ_FUSED_PRE_ROWS=32 HZ_FUSED_POST_ROWS=64"; do
  env $v timeout 300 python bench.py --steps 2 --warmup 3 > gpurun_out/bf.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/bf.json')); k=d['kernels']
print('$v', round(d['value'],2), {n: (k[n]['avg_us'], k[n]['frac']) for n in k if 'fused' in n})" >> gpurun_out/fused_sweep.txt
done
