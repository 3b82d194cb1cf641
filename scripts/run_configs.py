"""Run BASELINE configs 1-5 (one GPU) through the public API: setup time,
cycles, RHS/s, residuals, per-kernel roofline summary."""
import sys, time, json, os
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs

which = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4, 5]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for c in which:
    if c == 1:
        cfg = configs.config1(nlevels=3)                   # converging 3-level variant
        cfg.restart = 10
    elif c == 2:
        import bench
        cfg = bench.build_workload(0, 1, 32)
    elif c == 3:
        cfg = configs.config3(nlevels=4)
    elif c == 4:
        cfg = configs.config4(nlevels=5)
        cfg.source_nodes = cfg.source_nodes[:8]            # k = 8 per GPU (RHS sharded 8 per GPU)
    elif c == 5:
        cfg = configs.config5(nlevels=6)
    if c >= 3:
        cfg.shift = float(os.environ.get("HZ_SHIFT3D", "0.5"))
        cfg.restart = int(os.environ.get("HZ_RESTART3D", "10"))
    t = time.time()
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, max_cycles=int(os.environ.get("HZ_MAXC", "600"))))
    torch.cuda.synchronize()
    setup = time.time() - t
    B = torch.from_numpy(cfg.rhs_block()).cuda()
    torch.cuda.synchronize(); t = time.time()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); dt = time.time() - t
    with hz.kernel_profile() as prof:
        pass
    out = dict(config=c, name=cfg.name, n=cfg.n, k=cfg.k, nlevels=cfg.nlevels, shift=cfg.shift, restart=cfg.restart,
               prec=cfg.precond_precision, setup_s=round(setup, 2), solve_s=round(dt, 3), cycles=rep.cycles,
               converged=rep.all_converged(), worst_res=float(rep.rel_residual.max()),
               rhs_per_s=round(cfg.k / dt, 3), ms_per_cycle=round(1e3 * dt / max(rep.cycles, 1), 3))
    print(json.dumps(out), flush=True)
    del S, P, X, B
    torch.cuda.empty_cache()
