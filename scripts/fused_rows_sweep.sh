#!/bin/bash
# fused fine-level chunk rows at the default 32-node strips (k = 8): ms/cycle
cd "$(dirname "$0")/.."
for pr in "16 32" "8 16" "8 32" "16 16" "32 64" "4 8"; do
  set -- $pr
  echo "pre=$1 post=$2 $(HZ_FUSED_PRE_ROWS=$1 HZ_FUSED_POST_ROWS=$2 timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"
done
