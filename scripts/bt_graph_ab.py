"""Config 3 with the complex128 preconditioner (cycles are not graph-replayed): the plane-solver chain launched
directly (HZ_BT_GRAPH=0) vs replayed from its own CUDA graph (default).  python scripts/bt_graph_ab.py [kind]"""
import sys, time, os
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
cfg = run_configs.make(3)
cfg.precond_precision = "c128"
cfg.cycle = sys.argv[1] if len(sys.argv) > 1 else "V"
cfg.max_cycles, cfg.tol = 40, 1e-30
P = hz.HelmholtzProblem.from_config(cfg)
S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
best = 1e9
for r in range(4):
    torch.cuda.synchronize(); t = time.time()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); dt = time.time() - t
    if r: best = min(best, 1e3 * dt / rep.cycles)
print(f"HZ_BT_GRAPH={os.environ.get('HZ_BT_GRAPH', '1')} config 3 c128 {cfg.cycle}-cycle preconditioner: {best:.3f} ms per cycle")
