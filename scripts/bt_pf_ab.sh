#!/bin/bash
for rep in 1 2 3; do for v in "HZ_BT_PF=0" "HZ_BT_PF=1"; do
  echo -n "# $v rep $rep: "; env $v HZ_BT_NW=8 python scripts/cycle_time.py 4 7 40 3
done; done
