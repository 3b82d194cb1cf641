"""Convergence sweep for 3D config 3 (129x129x65, k=16) on the GPU."""
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs
cfg = configs.config3(nlevels=4)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
variants = [(4, 1.0, "V", "MgFgmres", 10), (4, 1.5, "V", "MgFgmres", 10), (4, 1.0, "W", "MgFgmres", 10),
            (4, 1.0, "K", "MgFgmres", 10), (4, 2.0, "V", "MgFgmres", 10), (3, 0.5, "V", "MgFgmres", 10)]
for nl, shift, kind, method, restart in variants:
    o = hz.HelmholtzSolveOptions(method=method, tol=1e-6, max_cycles=600, nlevels=nl, shift_factor=shift,
                                 cycle=hz.CycleSpec(kind), fgmres_restart=restart, precond_precision="c128")
    try:
        t = time.time(); S = hz.HelmholtzSolver(P, o); torch.cuda.synchronize(); ts = time.time() - t
        t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(nl=nl, shift=shift, kind=kind, restart=restart, setup=round(ts, 2), cycles=rep.cycles,
                              conv=rep.all_converged(), worst=float(rep.rel_residual.max()), s=round(dt, 2),
                              rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(nl=nl, shift=shift, kind=kind, error=str(e)[:150])), flush=True)
