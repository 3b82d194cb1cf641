#!/bin/bash
# config 4 (257x257x129, k = 8, c64): the compact 27-point fine operator at 3 / 4 levels
cd "$(dirname "$0")/.."
r() { echo "# $1"; env HZ_CFG4_MAX_CYCLES=500 HZ_WARM=0 $1 timeout 300 python scripts/run_configs.py 4 2>&1 | grep -E '^\{|Error'; }
r "HZ_CFG4_STENCIL=27 HZ_CFG4_NLEVELS=3"
r "HZ_CFG4_STENCIL=27 HZ_CFG4_NLEVELS=4 HZ_CFG4_SHIFT=0.9"
r "HZ_CFG4_STENCIL=27 HZ_CFG4_NLEVELS=4 HZ_CFG4_SHIFT=1.3"
r "HZ_CFG4_STENCIL=7 HZ_CFG4_NLEVELS=3"
