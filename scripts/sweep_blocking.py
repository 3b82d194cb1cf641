"""RHS blocking of the bench workload (config 2, 32 sources): the 32 sources
split into nb blocks of 32/nb (strided, like rank sharding), one solver per
block on the same problem, solved concurrently (hz_solve_blocks_multi_device).
Block Krylov flops per RHS scale with the block width, cycles per RHS with the
blocking; this measures the trade. One JSON line per nb:restart combo
(second solve timed)."""
import sys, time, json, os
sys.path.insert(0, ".")
import numpy as np
import torch, paper_1607_00968_b200 as hz, bench

combos = [tuple(int(x) for x in c.split(":"))
          for c in os.environ.get("HZ_COMBOS", "1:3,2:3,2:4,4:3,4:5").split(",")]
for nb, restart in combos:
    cfg = bench.build_workload(0, 1, 32)
    cfg.restart = restart
    cfg.max_cycles = 1500
    B = torch.from_numpy(cfg.rhs_block()).cuda()
    P = hz.HelmholtzProblem.from_config(cfg)
    opts = hz.HelmholtzSolveOptions.from_config(cfg)
    solvers = [hz.HelmholtzSolver(P, opts) for _ in range(nb)]
    Bs = [B[:, i::nb].contiguous() for i in range(nb)]
    for it in range(2):
        torch.cuda.synchronize(); t = time.time()
        Xs, reps = hz.solve_blocks_multi(solvers, Bs)
        torch.cuda.synchronize(); dt = time.time() - t
    cyc = [r.cycles for r in reps]
    conv = all(r.all_converged() for r in reps)
    worst = max(float(np.max(r.rel_residual)) for r in reps)
    print(json.dumps(dict(blocks=nb, k_per_block=32 // nb, restart=restart, cycles=cyc, conv=conv, worst=worst,
                          s=round(dt, 3), rhs_per_s=round(32 / dt, 2))), flush=True)
    del solvers, P, Xs
    torch.cuda.empty_cache()
