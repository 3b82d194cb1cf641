#!/bin/bash
# config 4 (257x257x129, k = 8, c64 preconditioner): hierarchy depth x shift x
# Jacobi weight x cycle, to cut the 65x65x33 coarse solve of the 3-level setup
cd "$(dirname "$0")/.."
r() { echo "# $1"; env HZ_CFG4_MAX_CYCLES=500 HZ_WARM=0 $1 timeout 300 python scripts/run_configs.py 4 2>&1 | grep '^{'; }
for nl in 4 5; do
  for sh in 0.5 0.9 1.3; do
    r "HZ_CFG4_NLEVELS=$nl HZ_CFG4_SHIFT=$sh"
  done
  r "HZ_CFG4_NLEVELS=$nl HZ_CFG4_SHIFT=0.9 HZ_CFG4_JACOBI_WEIGHT=0.6"
  r "HZ_CFG4_NLEVELS=$nl HZ_CFG4_SHIFT=0.9 HZ_CFG4_CYCLE=W"
done
r "HZ_CFG4_NLEVELS=3"
