#!/bin/bash
for v in "HZ_BT_NW=8" "HZ_BT_NW=4" "HZ_BT_NW=4 HZ_BT_PF=0" "HZ_BT_NW=8 HZ_BT_PF=0"; do
  echo "# $v"
  env $v python scripts/cycle_time.py 4 7 40 3
  env $v python scripts/cycle_time.py 3 7 60 4
done
