"""Config 2: levels x shift x small Jacobi weights, one 8-column block (c64 cycle, FGMRES(5), V), cycles and time."""
import sys, time, json, itertools
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz
import bench
cfg = bench.build_workload(0, 1, 8)
cfg.krylov_block = 0
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
grid = [(6, 0.9, 0.6)] + list(itertools.product((6, 5, 4), (0.5, 0.6, 0.7, 0.8), (0.4, 0.5)))
for nl, shift, wj in grid:
    cfg.nlevels, cfg.shift, cfg.jacobi_weight = nl, shift, wj
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 700
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(nl=nl, shift=shift, wj=wj, cycles=rep.cycles, conv=bool(rep.all_converged()),
                              worst=float(rep.rel_residual.max()), s=round(dt, 3))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(nl=nl, shift=shift, wj=wj, error=str(e)[:120])), flush=True)
