#!/bin/bash
# Galerkin stencil kernel variants (HZ_STENCIL_VARIANT): per-kernel profile of
# the bench solve (60 cycles) and a bitwise check of the solution.
for v in 0 1 2 3; do
  echo "== variant $v"
  HZ_STENCIL_VARIANT=$v python scripts/profile_solve.py 32 c64 60 2>&1 | grep -E "ms/cycle|stencil|kernel total"
  HZ_STENCIL_VARIANT=$v python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, bench, paper_1607_00968_b200 as hz
cfg = bench.build_workload(0, 1, 32); cfg.max_cycles = 20
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
X, r = S.solve_block(torch.from_numpy(cfg.rhs_block()).cuda())
np.save('gpurun_out/stv_$v.npy', X.cpu().numpy())"
done
python -c "
import numpy as np
a = np.load('gpurun_out/stv_0.npy')
for v in (1, 2, 3): print('variant', v, 'bitwise equal to 0:', np.array_equal(a, np.load(f'gpurun_out/stv_{v}.npy')))"
rm -f gpurun_out/stv_*.npy
