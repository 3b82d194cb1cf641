#!/bin/bash
# Kernel variant A/B on the bench solve: VAR=<env name> VALS="a b ...":
# per-kernel profile (60 cycles) + bitwise check of a 20-cycle solution.
VAR=${VAR:-HZ_STENCIL_VARIANT}; VALS=${VALS:-"0 1"}; GREP=${GREP:-"stencil|fine"}
first=""
for v in $VALS; do
  echo "== $VAR=$v"
  env $VAR=$v python scripts/profile_solve.py 32 c64 60 2>&1 | grep -E "ms/cycle|$GREP|kernel total"
  env $VAR=$v python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, bench, paper_1607_00968_b200 as hz
cfg = bench.build_workload(0, 1, 32); cfg.max_cycles = 20
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
X, r = S.solve_block(torch.from_numpy(cfg.rhs_block()).cuda())
np.save('gpurun_out/kv_$v.npy', X.cpu().numpy())"
  [ -z "$first" ] && first=$v
done
for v in $VALS; do python -c "
import numpy as np
print('$VAR=$v bitwise equal to $first:', np.array_equal(np.load('gpurun_out/kv_$first.npy'), np.load('gpurun_out/kv_$v.npy')))"; done
rm -f gpurun_out/kv_*.npy
