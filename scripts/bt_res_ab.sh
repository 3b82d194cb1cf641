#!/bin/bash
# production-mode ms per cycle with the bench settings of configs 3 / 4 (W-cycles): row-owner plane-step kernel (HZ_BT_RES=0)
# vs the resident-r kernel (HZ_BT_RES=NW:RW:LC), two interleaved rounds
export HZ_CFG3_CYCLE=W HZ_CFG3_SHIFT=0.25 HZ_CFG3_JACOBI_WEIGHT=0.9 HZ_CFG3_RESTART=5
export HZ_CFG4_CYCLE=W HZ_CFG4_SHIFT=0.3 HZ_CFG4_JACOBI_WEIGHT=0.9 HZ_CFG4_RESTART=5
for rep in 1 2; do
for v in 0 16:2:128 16:2:256 16:1:128 16:1:256 8:2:128 8:2:256 8:4:128 24:1:256 32:1:128; do
  echo "# HZ_BT_RES=$v"
  HZ_BT_RES=$v python scripts/cycle_time.py 3 7 40 3
  HZ_BT_RES=$v python scripts/cycle_time.py 4 27 30 2
done
done
