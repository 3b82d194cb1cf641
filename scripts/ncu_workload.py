"""The bench workload (config 2, 32 sources as 4 concurrent blocks of 8,
FGMRES(5) + c64 V(2,2)) cut to a few cycles, for ncu: setup and one warm-up
solve run outside the profiled range (cudaProfilerStart/Stop brackets the
measured solve; run ncu with --profile-from-start off).

  python scripts/ncu_workload.py [cycles] [rhs_block]
"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
import bench

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = bench.build_workload(0, 1, 32)
if len(sys.argv) > 2:
    cfg.krylov_block = int(sys.argv[2])
cfg.max_cycles = cycles
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
S.solve_block(B)
torch.cuda.synchronize()
torch.cuda.profiler.start()
X, rep = S.solve_block(B)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("cycles", rep.cycles)
