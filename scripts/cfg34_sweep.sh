#!/bin/bash
# configs 1, 3, 4 with the current kernels: baseline settings and blocked / c64 variants
cd "$(dirname "$0")/.."
r() { echo "# $1"; env $1 timeout 600 python scripts/run_configs.py $2 2>&1 | grep '^{'; }
r "X=0" 1
r "X=0" 3
r "HZ_CFG3_PRECOND_PRECISION=c64" 3
r "HZ_CFG3_PRECOND_PRECISION=c64 HZ_CFG3_KRYLOV_BLOCK=8" 3
r "HZ_CFG3_PRECOND_PRECISION=c64 HZ_CFG3_KRYLOV_BLOCK=8 HZ_CFG3_RESTART=5" 3
r "X=0" 4
r "HZ_CFG4_RESTART=5" 4
