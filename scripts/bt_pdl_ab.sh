#!/bin/bash
# production-mode (graph replay) ms per cycle: L2 prefetch of the chain's next factor block (HZ_BT_L2PF)
# and programmatic dependent launches of the plane steps (HZ_BT_PDL), configs 3 and 4, two interleaved rounds
for rep in 1 2; do
for v in "HZ_BT_L2PF=0 HZ_BT_PDL=0" "HZ_BT_L2PF=1 HZ_BT_PDL=0" "HZ_BT_L2PF=0 HZ_BT_PDL=1" "HZ_BT_L2PF=1 HZ_BT_PDL=1" "HZ_BT_L2PF=2 HZ_BT_PDL=1"; do
  echo "# $v"
  env $v python scripts/cycle_time.py 3 7 60 4
  env $v python scripts/cycle_time.py 4 7 40 3
done
done
