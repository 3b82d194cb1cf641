"""Short config-2 bench-workload solve (a few cycles) for ncu captures."""
import sys, os
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench
cfg = bench.build_workload(0, 1, 32)
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg, max_cycles=int(sys.argv[1]) if len(sys.argv) > 1 else 4))
B = torch.from_numpy(cfg.rhs_block()).cuda()
X, rep = S.solve_block(B)
torch.cuda.synchronize()
print("cycles", rep.cycles)
