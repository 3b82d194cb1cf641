#!/bin/bash
# production-mode (graph replay) ms per cycle for the plane-solver variants, configs 3 and 4 (7-point)
for v in "HZ_BT_TWISTED=0 HZ_BT_PERMUTE=0" "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=0" "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=2" \
         "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=2 HZ_BT_PF=1" "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=2 HZ_BT_PF=1 HZ_BT_RW=1" \
         "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=2 HZ_BT_RW=1" "HZ_BT_TWISTED=1 HZ_BT_PERMUTE=0 HZ_BT_PF=1"; do
  echo "# $v"
  env $v python scripts/cycle_time.py 3 7 60 4
  env $v python scripts/cycle_time.py 4 7 40 3
done
