#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x -k galerkin > gpurun_out/lf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/lf_tests.log
for f in 1 0; do echo "HZ_LEVEL_FUSE=$f $(HZ_LEVEL_FUSE=$f timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"; done
echo "rr=0 $(HZ_RESID_RESTRICT_MAX_NODES=0 timeout 300 python scripts/sweep_groups.py 32 2>&1 | tr '\n' ' ')"
python scripts/profile_solve.py 8 c64 60 > gpurun_out/prof8.txt 2>&1
