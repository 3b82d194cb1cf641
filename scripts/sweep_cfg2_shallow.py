"""Config 2 with shallow hierarchies (exact solve of a larger coarsest grid) and small shifts: cycle counts of one
8-column block (c64 cycle, FGMRES(5)), V and W.  python scripts/sweep_cfg2_shallow.py <nlevels> [shifts] [kinds]"""
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz
import bench
nl = int(sys.argv[1])
shifts = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.2, 0.3, 0.5, 0.7]
kinds = sys.argv[3].split(",") if len(sys.argv) > 3 else ["V", "W"]
cfg = bench.build_workload(0, 1, 8)
cfg.krylov_block = 0
cfg.nlevels = nl
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
for shift in shifts:
    for kind in kinds:
        for wj in (0.6, 0.8):
            cfg.shift, cfg.cycle, cfg.jacobi_weight = shift, kind, wj
            o = hz.HelmholtzSolveOptions.from_config(cfg)
            o.max_cycles = 600
            try:
                t = time.time(); S = hz.HelmholtzSolver(P, o); torch.cuda.synchronize(); ts = time.time() - t
                S.solve_block(B)
                torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
                print(json.dumps(dict(nl=nl, shift=shift, kind=kind, wj=wj, setup=round(ts, 1), cycles=rep.cycles,
                                      conv=bool(rep.all_converged()), worst=float(rep.rel_residual.max()),
                                      s=round(dt, 3), ms_per_cycle=round(1e3 * dt / rep.cycles, 3))), flush=True)
                del S
            except Exception as e:
                print(json.dumps(dict(nl=nl, shift=shift, kind=kind, wj=wj, error=str(e)[:160])), flush=True)
