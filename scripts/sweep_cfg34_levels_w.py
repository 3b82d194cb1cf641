"""4-level W-cycle hierarchies for configs 3 / 4 at the low shifts (c64 cycle), timed on the second solve.
  python scripts/sweep_cfg34_levels_w.py <3|4> [stencil]"""
import sys, time, json
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
c = int(sys.argv[1])
cfg = run_configs.make(c)
if len(sys.argv) > 2:
    cfg.stencil = int(sys.argv[2])
cfg.nlevels = 4
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
for kind, shift, wj, restart in [("W", 0.3, 0.9, 5), ("W", 0.4, 0.9, 5), ("W", 0.5, 0.9, 5), ("W", 0.7, 0.8, 5), ("K", 0.3, 0.9, 5), ("W", 0.4, 0.7, 5)]:
    cfg.cycle, cfg.shift, cfg.jacobi_weight, cfg.restart = kind, shift, wj, restart
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.max_cycles = 300
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(cfg=c, nl=4, kind=kind, shift=shift, wj=wj, restart=restart, cycles=rep.cycles,
                              conv=bool(rep.all_converged()), worst=float(rep.rel_residual.max()), s=round(dt, 3),
                              rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(cfg=c, kind=kind, shift=shift, error=str(e)[:120])), flush=True)
