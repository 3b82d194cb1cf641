"""Configs 3 / 4 with their literal level counts (4 / 4-5) at the small Jacobi weights that make config 5's 4-level
hierarchy converge (c64 cycle), timed on the second solve.  python scripts/sweep_cfg34_literal_levels.py <3|4> [stencil]"""
import sys, time, json
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
c = int(sys.argv[1])
cfg = run_configs.make(c)
if len(sys.argv) > 2:
    cfg.stencil = int(sys.argv[2])
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
if c == 3:
    grid = [(4, "V", sh, wj, r) for sh in (0.8, 1.0, 1.2) for wj in (0.5, 0.6) for r in (5,)] + [(4, "V", 1.0, 0.5, 10), (4, "W", 1.0, 0.5, 5)]
else:
    grid = [(4, "V", 1.0, 0.5, 5), (4, "V", 1.2, 0.5, 5), (5, "V", 1.0, 0.5, 5), (5, "V", 1.5, 0.5, 5), (4, "W", 1.0, 0.5, 5)]
for nl, kind, shift, wj, restart in grid:
    cfg.nlevels, cfg.cycle, cfg.shift, cfg.jacobi_weight, cfg.restart = nl, kind, shift, wj, restart
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 800
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(cfg=c, nl=nl, kind=kind, shift=shift, wj=wj, restart=restart, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), worst=float(rep.rel_residual.max()), s=round(dt, 3),
                              rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(cfg=c, nl=nl, kind=kind, shift=shift, error=str(e)[:120])), flush=True)
