#!/bin/bash
for v in "HZ_BT_PF=0" "HZ_BT_PF=1" "HZ_BT_PF=0 HZ_BT_RW=1" "HZ_BT_PF=1 HZ_BT_RW=1"; do
  echo "# $v"
  env $v python scripts/cycle_time.py 3 7 60 4
  env $v python scripts/cycle_time.py 4 7 40 3
done
