"""Blocked solves of the bench workload (config 2, 32 sources) through
HelmholtzSolveOptions.rhs_block: combos rb:restart:shift:wj:levels:order,
order 's' = strided source -> group assignment (group i = sources i, i+G, ...),
'c' = contiguous. One JSON line per combo (device-resident B, second solve
timed with CUDA events)."""
import sys, json, os
sys.path.insert(0, ".")
import numpy as np
import torch, paper_1607_00968_b200 as hz, bench

combos = os.environ.get("HZ_COMBOS", "8:5:0.9:0.6:5:s,8:5:0.9:0.6:5:c").split(",")
for c in combos:
    rb, restart, shift, wj, nl, order = c.split(":")
    rb, restart, nl, shift, wj = int(rb), int(restart), int(nl), float(shift), float(wj)
    bench.WORKLOAD["nlevels"] = nl
    cfg = bench.build_workload(0, 1, 32)
    cfg.restart, cfg.shift, cfg.jacobi_weight, cfg.krylov_block = restart, shift, wj, rb
    cfg.max_cycles = 1500
    if order == "s" and rb > 0:
        G = (32 + rb - 1) // rb
        cfg.source_nodes = np.concatenate([cfg.source_nodes[i::G] for i in range(G)])
    B = torch.from_numpy(cfg.rhs_block()).cuda()
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    for it in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        X, rep = S.solve_block(B)
        e1.record(); torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    print(json.dumps(dict(combo=c, cycles=int(rep.cycles), mean_col_cycles=rep.mean_col_cycles(),
                          conv=rep.all_converged(), worst=float(np.max(rep.rel_residual)),
                          s=round(dt, 4), rhs_per_s=round(32 / dt, 2))), flush=True)
    del S, X
    torch.cuda.empty_cache()
