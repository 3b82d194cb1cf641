#!/bin/bash
# fused fine-level visit knobs at the bench blocking (4 groups of 8): ms/cycle
cd "$(dirname "$0")/.."
run() { echo "$1 $(env $1 timeout 300 python scripts/sweep_groups.py 32 2>/dev/null)"; }
run "HZ_FUSED_VCYCLE=1"
run "HZ_FUSED_VCYCLE=0"
run "HZ_FUSED_PRE_ROWS=8 HZ_FUSED_POST_ROWS=16"
run "HZ_FUSED_PRE_ROWS=4 HZ_FUSED_POST_ROWS=8"
run "HZ_FUSED_NT=128"
run "HZ_FUSED_NT=128 HZ_FUSED_PRE_ROWS=8 HZ_FUSED_POST_ROWS=16"
run "HZ_FUSED_VCYCLE=0 HZ_K8=0"
