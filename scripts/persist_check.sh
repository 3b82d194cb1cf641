#!/bin/bash
# persistent coarse-cycle kernels: bitwise tests, then timing (4 groups, 1 group)
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_fused.py -q -x -k persistent > gpurun_out/persist_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/persist_tests.log
for f in 1 0; do echo "HZ_COARSE_PERSIST=$f $(HZ_COARSE_PERSIST=$f timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"; done
