"""W-cycle sweep for configs 3 / 4 (3 levels, c64 cycle), timed on the second solve.  python scripts/sweep_cfg34_w.py <3|4> [stencil]"""
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
    grid = [("W", sh, wj, 5, (2, 2)) for sh in (0.2, 0.3, 0.35, 0.4, 0.5) for wj in (0.8, 0.9)]
    grid += [("W", 0.3, 0.9, 5, pp) for pp in ((2, 1), (1, 2), (3, 3))] + [("W", 0.3, 0.9, r, (2, 2)) for r in (3, 10)]
else:
    grid = [("W", 0.3, 0.9, 10, (2, 2)), ("W", 0.4, 0.9, 10, (2, 2)), ("W", 0.3, 0.9, 5, (2, 2)), ("V", 0.3, 0.9, 10, (2, 2))]
    if len(sys.argv) > 3:  # second round
        grid = [("W", 0.25, 0.9, 5, (2, 2)), ("W", 0.2, 0.9, 5, (2, 2)), ("W", 0.3, 0.9, 3, (2, 2)), ("W", 0.3, 0.9, 7, (2, 2)),
                ("W", 0.3, 0.8, 5, (2, 2)), ("W", 0.3, 0.9, 5, (1, 1)), ("W", 0.3, 0.9, 5, (3, 3)), ("W", 0.3, 0.9, 5, (2, 1))]
for kind, shift, wj, restart, (pre, post) in grid:
    cfg.cycle, cfg.shift, cfg.jacobi_weight, cfg.restart, cfg.pre, cfg.post = kind, shift, wj, restart, pre, post
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 500
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(cfg=c, kind=kind, shift=shift, wj=wj, restart=restart, pre=pre, post=post, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), s=round(dt, 3), rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(cfg=c, kind=kind, shift=shift, error=str(e)[:120])), flush=True)
