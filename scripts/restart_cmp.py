"""Restart length x levels for the bench workload (config 2, FGMRES + V, c64)."""
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench
for nl in (4, 5):
    for restart in (3, 4, 5, 6, 8):
        cfg = bench.build_workload(0, 1, 32)
        cfg.nlevels, cfg.restart = nl, restart
        P = hz.HelmholtzProblem.from_config(cfg)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
        B = torch.from_numpy(cfg.rhs_block()).cuda()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); t = time.time()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(nlevels=nl, restart=restart, cycles=rep.cycles, conv=rep.all_converged(), s=round(dt, 3),
                              ms_per_cycle=round(1e3 * dt / rep.cycles, 3), rhs_per_s=round(32 / dt, 2))), flush=True)
        del S, P
