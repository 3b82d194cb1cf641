"""Cycle-shape sweep for the bench workload (config 2, k=32, c64 preconditioner):
levels x restart x shift x cycle kind x pre/post sweeps x w_J, one JSON line
each (second solve timed). HZ_COMBOS="nl:restart:shift:kind:pre:post:wj,..."."""
import sys, time, json, os
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench

DEFAULT = ("5:3:1.0:V:2:2:0.8,5:3:1.0:W:2:2:0.8,4:3:1.0:W:2:2:0.8,5:5:1.0:W:2:2:0.8,"
           "5:3:1.0:V:3:3:0.8,5:3:1.0:V:1:1:0.8,5:3:1.0:V:2:2:0.9,5:3:1.0:V:2:2:0.7,"
           "5:3:0.9:W:2:2:0.8,5:3:1.0:K:2:2:0.8")
k = int(os.environ.get("HZ_K", "32"))
for c in os.environ.get("HZ_COMBOS", DEFAULT).split(","):
    nl, restart, shift, kind, pre, post, wj = c.split(":")
    cfg = bench.build_workload(0, 1, k)
    cfg.nlevels, cfg.restart, cfg.shift = int(nl), int(restart), float(shift)
    cfg.cycle, cfg.pre, cfg.post, cfg.jacobi_weight = kind, int(pre), int(post), float(wj)
    cfg.max_cycles = int(os.environ.get("HZ_MAXC", "1200"))
    try:
        P = hz.HelmholtzProblem.from_config(cfg)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
        B = torch.from_numpy(cfg.rhs_block()).cuda()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); t = time.time()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(combo=c, cycles=rep.cycles, conv=rep.all_converged(),
                              worst=max(rep.rel_residual), s=round(dt, 3),
                              ms_per_cycle=round(1e3 * dt / rep.cycles, 3),
                              rhs_per_s=round(k / dt, 2) if rep.all_converged() else 0)), flush=True)
        del S, P, X, B
    except Exception as e:
        print(json.dumps(dict(combo=c, error=str(e))), flush=True)
    torch.cuda.empty_cache()
