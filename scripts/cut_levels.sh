#!/bin/bash
# timing-only: cost of the cycle's coarse levels in the 4-group mix (HZ_DEBUG_CUT_LEVEL: a
# timing-only switch since removed from the library; results in profiles/r01_cut_levels_timing.txt)
cd "$(dirname "$0")/.."
run() { echo "$1 $(env $1 timeout 300 python scripts/sweep_groups.py ${2:-32} 2>&1 | tail -1)"; }
run "HZ_DEBUG_CUT_LEVEL=0"
run "HZ_DEBUG_CUT_LEVEL=2"
run "HZ_DEBUG_CUT_LEVEL=1"
run "HZ_DEBUG_CUT_LEVEL=0" 8
run "HZ_DEBUG_CUT_LEVEL=2" 8
run "HZ_DEBUG_CUT_LEVEL=1" 8
