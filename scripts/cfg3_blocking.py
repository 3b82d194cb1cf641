import sys, time, json
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
cfg = run_configs.make(3)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
for kb in (8, 0, 4):
    cfg.cycle, cfg.shift, cfg.jacobi_weight, cfg.restart, cfg.krylov_block = "W", 0.25, 0.9, 5, kb
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    S = hz.HelmholtzSolver(P, o)
    S.solve_block(B)
    best = 1e9
    for r in range(3):
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); best = min(best, time.time() - t)
    print(json.dumps(dict(krylov_block=kb, cycles=rep.cycles, conv=bool(rep.all_converged()), s=round(best, 4), rhs_per_s=round(cfg.k / best, 2))), flush=True)
    del S
