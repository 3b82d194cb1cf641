"""Concurrency scaling of blocked solves: the bench workload's solver with
rhs_block = 8 and k = 8 .. 64 sources (1 .. 8 concurrent groups); ms per
cycle tells whether the concurrent groups saturate the GPU."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
import torch, paper_1607_00968_b200 as hz, bench

for k in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,24,32,48,64").split(",")]:
    cfg = bench.build_workload(0, 1, k)
    cfg.max_cycles = 100
    B = torch.from_numpy(cfg.rhs_block()).cuda()
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    for it in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        X, rep = S.solve_block(B)
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps(dict(k=k, groups=-(-k // 8), cycles=int(rep.cycles), ms=round(ms, 2),
                          ms_per_cycle=round(ms / rep.cycles, 4),
                          ms_per_cycle_per_group=round(ms / rep.cycles / -(-k // 8), 4))), flush=True)
    del S, X
    torch.cuda.empty_cache()
