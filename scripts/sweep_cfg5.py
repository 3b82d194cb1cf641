"""Config 5 (513x513x257, k=8, c64 preconditioner) solver variants on one
GPU: levels / shift / cycle kind, bounded cycles. One JSON line each."""
import sys, time, json, os
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs

VARIANTS = [  # (levels, shift, kind, restart)
    (4, 1.5, "W", 5), (4, 1.0, "V", 5), (4, 1.0, "W", 5), (5, 1.5, "W", 5), (5, 1.0, "W", 5),
]
if os.environ.get("HZ_VARIANTS"):
    VARIANTS = [tuple(t(x) for t, x in zip((int, float, str, int, float), v.split(":")))
                for v in os.environ["HZ_VARIANTS"].split(",")]
maxc = int(os.environ.get("HZ_MAXC", "300"))
cfg = configs.config5(nlevels=4)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
for var in VARIANTS:
    (L, shift, kind, restart), wj = var[:4], (var[4] if len(var) > 4 else 0.8)
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.method, o.nlevels, o.shift_factor, o.cycle = "MgFgmres", L, shift, hz.CycleSpec(kind, 2, 2, wj)
    o.fgmres_restart, o.max_cycles = restart, maxc
    t = time.time()
    S = hz.HelmholtzSolver(P, o)
    torch.cuda.synchronize(); setup = time.time() - t
    t = time.time()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); dt = time.time() - t
    h = rep.history
    print(json.dumps(dict(levels=L, shift=shift, kind=kind, restart=restart, wj=wj, setup_s=round(setup, 1),
                          cycles=rep.cycles, converged=rep.all_converged(),
                          worst_res=float(rep.rel_residual.max()), solve_s=round(dt, 2),
                          ms_per_cycle=round(1e3 * dt / max(rep.cycles, 1), 2),
                          hist=[float(h[i]) for i in range(0, len(h), 50)])), flush=True)
    del S, X
    torch.cuda.empty_cache()
