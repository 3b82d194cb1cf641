#!/bin/bash
# config 4 (257x257x129, k = 8, c64): hierarchy depth / shift
cd "$(dirname "$0")/.."
r() { echo "# $1"; env $1 timeout 600 python scripts/run_configs.py 4 2>&1 | grep '^{'; }
r "HZ_CFG4_NLEVELS=4"
r "HZ_CFG4_NLEVELS=4 HZ_CFG4_SHIFT=0.7"
r "HZ_CFG4_NLEVELS=4 HZ_CFG4_SHIFT=1.0"
r "HZ_CFG4_NLEVELS=4 HZ_CFG4_SHIFT=0.7 HZ_CFG4_JACOBI_WEIGHT=0.6"
r "HZ_CFG4_NLEVELS=3 HZ_CFG4_SHIFT=0.7"
