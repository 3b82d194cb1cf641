"""Cycle-kind sweep for config 3 (3 levels, c64 cycle, 2 blocks of 8): V / W / K x shift x pre/post, timed on the second solve."""
import sys, time, json, itertools
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
cfg = run_configs.make(3)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
grid = [(kind, sh, 0.9, 5, pp) for kind in ("W", "K") for sh in (0.15, 0.25) for pp in ((2, 2), (1, 1))]
grid += [("V", 0.25, 0.9, 5, (2, 2)), ("V", 0.25, 0.9, 5, (3, 3)), ("V", 0.25, 0.9, 5, (2, 3))]
for kind, shift, wj, restart, (pre, post) in grid:
    cfg.cycle, cfg.shift, cfg.jacobi_weight, cfg.restart, cfg.pre, cfg.post = kind, shift, wj, restart, pre, post
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 500
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(kind=kind, shift=shift, wj=wj, restart=restart, pre=pre, post=post, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), s=round(dt, 3), rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(kind=kind, shift=shift, error=str(e)[:120])), flush=True)
