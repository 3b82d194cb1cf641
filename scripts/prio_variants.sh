#!/bin/bash
# coarse-cycle stream priority at the bench blocking (4 groups of 8): ms/cycle
cd "$(dirname "$0")/.."
run() { echo "$1 $(env $1 timeout 300 python scripts/sweep_groups.py ${2:-32} 2>&1 | tail -1)"; }
run "HZ_PRIO=0"
run "HZ_PRIO=1"
run "HZ_PRIO_FROM=1"
run "HZ_PRIO=0" 8
run "HZ_PRIO=1" 8
