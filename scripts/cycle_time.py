"""ms per FGMRES cycle of a config's solve in production mode (CUDA-graph
replayed preconditioner cycles, no per-kernel profiling): the number variant
A/Bs of the latency-bound coarse chain should be judged on (per-kernel event
profiles run the chain as plain stream launches and are host-launch bound).

  python scripts/cycle_time.py <config 3|4> [stencil] [cycles] [reps]
"""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
sys.path.insert(0, "scripts")
import run_configs

c = int(sys.argv[1])
cfg = run_configs.make(c)
if len(sys.argv) > 2:
    cfg.stencil = int(sys.argv[2])
cfg.max_cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 40
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
cfg.tol = 1e-30
P = hz.HelmholtzProblem.from_config(cfg)
S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
best = 1e9
for r in range(reps + 1):
    torch.cuda.synchronize(); t = time.time()
    try:
        X, rep = S.solve_block(B)
        cycles = rep.cycles
    except hz.ConvergenceError:
        cycles = cfg.max_cycles
    torch.cuda.synchronize(); dt = time.time() - t
    if r > 0:
        best = min(best, 1e3 * dt / cycles)
print(f"config {c} stencil {cfg.stencil} cycles {cycles}: {best:.3f} ms per cycle (best of {reps})")
