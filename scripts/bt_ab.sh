#!/bin/bash
# A/B of the plane solver's sweep axis and two-sided elimination on configs 3 / 4 (7-point)
for perm in 0 1; do for tw in 0 1; do
  echo "# HZ_BT_PERMUTE=$perm HZ_BT_TWISTED=$tw"
  HZ_BT_PERMUTE=$perm HZ_BT_TWISTED=$tw HZ_PROFILE=1 python scripts/run_configs.py 3 2>&1 | grep -E "config|coarse_bt"
  HZ_BT_PERMUTE=$perm HZ_BT_TWISTED=$tw HZ_PROFILE=1 HZ_CFG4_STENCIL=7 python scripts/run_configs.py 4 2>&1 | grep -E "config|coarse_bt"
done; done
