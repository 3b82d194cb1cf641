#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/w_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/w_tests.log
for f in 1 0; do echo "HZ_FUSED_WIDE=$f $(HZ_FUSED_WIDE=$f timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"; done
echo "WIDE NT64 $(HZ_FUSED_WIDE=1 HZ_FUSED_NT=64 timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"
python scripts/profile_solve.py 8 c64 60 > gpurun_out/prof8.txt 2>&1
