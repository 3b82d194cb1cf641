"""Shift x Jacobi-weight sweep at low shifts for configs 3 and 4 (3 levels, c64 cycle), timed on the second solve.
  python scripts/sweep_cfg34_shift.py <3|4> [stencil]"""
import sys, time, json, itertools
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
c = int(sys.argv[1])
cfg = run_configs.make(c)
if len(sys.argv) > 2:
    cfg.stencil = int(sys.argv[2])
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
if c == 3:
    grid = list(itertools.product((0.1, 0.15, 0.2, 0.25, 0.3), (0.8, 0.9, 1.0), (5,)))
else:
    grid = list(itertools.product((0.2, 0.3, 0.4, 0.5), (0.8, 0.9), (10,))) + [(0.3, 0.9, 5), (0.2, 0.9, 5)]
for shift, wj, restart in grid:
    cfg.shift, cfg.jacobi_weight, cfg.restart = shift, wj, restart
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 500
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(cfg=c, stencil=cfg.stencil, shift=shift, wj=wj, restart=restart, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), s=round(dt, 3), rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(cfg=c, shift=shift, wj=wj, restart=restart, error=str(e)[:120])), flush=True)
