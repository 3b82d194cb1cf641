"""Solver settings for the bench workload (config 2, k=32, FGMRES + V, c64):
levels x restart x shift, one JSON line each (second solve timed)."""
import sys, time, json, os
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench

combos = [tuple(float(x) if "." in x else int(x) for x in c.split(":"))
          for c in os.environ.get("HZ_COMBOS", "5:3:1.0,5:2:1.0,6:3:1.0,6:2:1.0,5:3:0.8,5:3:1.2").split(",")]
for nl, restart, shift in combos:
    cfg = bench.build_workload(0, 1, 32)
    cfg.nlevels, cfg.restart, cfg.shift = nl, restart, shift
    cfg.max_cycles = 1500
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    B = torch.from_numpy(cfg.rhs_block()).cuda()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); t = time.time()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); dt = time.time() - t
    print(json.dumps(dict(nlevels=nl, restart=restart, shift=shift, cycles=rep.cycles, conv=rep.all_converged(),
                          s=round(dt, 3), ms_per_cycle=round(1e3 * dt / rep.cycles, 3),
                          rhs_per_s=round(32 / dt, 2))), flush=True)
    del S, P
