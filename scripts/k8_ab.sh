#!/bin/bash
# A/B of the k = 8 bulk-copy fused kernels against the cp.async streaming
# kernels (HZ_FUSED_K8=0) and compile-time variants (variants/libhz_*.so):
# per-kernel event profile of one 8-column bench block solved alone.
# Usage (GPU box): bash scripts/k8_ab.sh [variant ...] > gpurun_out/k8_ab.txt
for k8 in 1 0; do
  echo "== HZ_FUSED_K8=$k8"
  HZ_FUSED_K8=$k8 python scripts/profile_solve.py 8 c64 60 2>&1 | head -8
done
for v in "$@"; do
  echo "== variant $v"
  HZ_LIB_PATH=variants/libhz_$v.so python scripts/profile_solve.py 8 c64 60 2>&1 | head -8
done
