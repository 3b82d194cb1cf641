"""Convergence / speed sweep of solver variants on BASELINE config 2 (GPU)."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs

k = int(sys.argv[1]) if len(sys.argv) > 1 else 32
variants = [
    dict(nl=4, shift=1.0, kind="V", method="MgFgmres", restart=10),
    dict(nl=4, shift=1.0, kind="V", method="MgFgmres", restart=5),
    dict(nl=4, shift=0.8, kind="V", method="MgFgmres", restart=10),
    dict(nl=5, shift=1.0, kind="V", method="MgFgmres", restart=10),
    dict(nl=5, shift=0.8, kind="V", method="MgFgmres", restart=10),
    dict(nl=4, shift=1.0, kind="W", method="MgFgmres", restart=10),
    dict(nl=5, shift=1.0, kind="W", method="MgFgmres", restart=10),
]
cfg = configs.config2(nlevels=4, k=k)
P = hz.HelmholtzProblem.from_config(cfg)
Bd = torch.from_numpy(cfg.rhs_block()).cuda()
for v in variants:
    prec = "c64"
    o = hz.HelmholtzSolveOptions(method=v["method"], tol=1e-6, max_cycles=800, nlevels=v["nl"],
                                 shift_factor=v["shift"], cycle=hz.CycleSpec(v["kind"]),
                                 fgmres_restart=v["restart"], precond_precision=prec)
    try:
        t = time.time(); S = hz.HelmholtzSolver(P, o); ts = time.time() - t
        torch.cuda.synchronize(); t = time.time()
        X, rep = S.solve_block(Bd)
        torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(v, prec=prec, setup_s=round(ts, 2), solve_s=round(dt, 3), cycles=rep.cycles,
                              conv=rep.all_converged(), worst=float(rep.rel_residual.max()),
                              ms_per_cycle=round(1e3 * dt / max(rep.cycles, 1), 3),
                              rhs_per_s=round(k / dt, 2) if rep.all_converged() else 0)), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(v, prec=prec, error=str(e)[:200])), flush=True)
