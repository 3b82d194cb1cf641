"""Round-2 solver-setting sweep for config 3 (129x129x65, k=16, 3 levels, c64 cycle, 2 blocks of 8):
shift x Jacobi weight x restart x sweeps, timed on the second solve."""
import sys, time, json, itertools
sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
cfg = run_configs.make(3)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
grid = list(itertools.product((0.3, 0.4, 0.5, 0.6), (0.7, 0.8, 0.9), (5, 10), ((2, 2),)))
grid += [(0.5, 0.8, 5, pp) for pp in ((1, 1), (2, 1), (1, 2), (3, 3))]
grid += [(0.5, 0.8, r, (2, 2)) for r in (3, 7)]
for shift, wj, restart, (pre, post) in grid:
    cfg.shift, cfg.jacobi_weight, cfg.restart, cfg.pre, cfg.post = shift, wj, restart, pre, post
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 500
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(shift=shift, wj=wj, restart=restart, pre=pre, post=post, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), s=round(dt, 3), rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(shift=shift, wj=wj, restart=restart, pre=pre, post=post, error=str(e)[:120])), flush=True)
