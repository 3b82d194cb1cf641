#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_blocking.py -q -x > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_tests.log
for f in 1 0; do echo "HZ_CYCLE_GRAPHS=$f $(HZ_CYCLE_GRAPHS=$f timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"; done
