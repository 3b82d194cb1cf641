#!/bin/bash
# row-owner plane-step kernel: rows per warp (register prefetch depth 4 / 3 chunks) on configs 3 / 4 (7-point)
for rw in 1 2; do
  echo "# HZ_BT_RW=$rw"
  HZ_BT_RW=$rw HZ_PROFILE=1 python scripts/run_configs.py 3 2>&1 | grep -E "config|coarse_bt"
  HZ_BT_RW=$rw HZ_PROFILE=1 HZ_CFG4_STENCIL=7 python scripts/run_configs.py 4 2>&1 | grep -E "config|coarse_bt"
done
