"""Config 4's per-GPU shard (257x257x129, k = 8, c64 preconditioner) cut to a
few FGMRES cycles, for ncu (cudaProfilerStart/Stop brackets the measured solve;
run ncu with --profile-from-start off).

  python scripts/ncu_cfg4.py [stencil=27] [cycles=3] [bench]
"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs

stencil = int(sys.argv[1]) if len(sys.argv) > 1 else 27
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if len(sys.argv) > 3 and sys.argv[3] == "bench":  # the settings of bench.py --workload cfg4 (W-cycle)
    import bench
    bench.WORKLOAD = bench.WORKLOADS["cfg4"]
    cfg = bench.build_workload(0, 1, 8)
    cfg.stencil, cfg.max_cycles = stencil, cycles
else:
    cfg = configs.config4(nlevels=3)
    cfg.source_nodes = cfg.source_nodes[:8]
    cfg.precond_precision, cfg.stencil, cfg.max_cycles = "c64", stencil, cycles
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
S.solve_block(B)
torch.cuda.synchronize()
torch.cuda.profiler.start()
X, rep = S.solve_block(B)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("cycles", rep.cycles)
