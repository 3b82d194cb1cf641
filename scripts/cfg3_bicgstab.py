"""Config 3: the reference's default method (W-cycle block BiCGSTAB, complex128 preconditioner -- BiCGSTAB needs a fixed
preconditioner, so not the complex64 cycle) against the bench's FGMRES(5) + c64 W-cycle, 3 levels, 2 blocks of 8."""
import sys, time, json
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch, paper_1607_00968_b200 as hz
import run_configs
cfg = run_configs.make(3)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
for method, prec, shift, wj in (("MgFgmres", "c64", 0.25, 0.9), ("MgBicgstab", "c128", 0.25, 0.9), ("MgBicgstab", "c128", 0.2, 0.8),
                                ("MgFgmres", "c128", 0.25, 0.9)):
    o = hz.HelmholtzSolveOptions(method=method, tol=1e-6, max_cycles=400, nlevels=3, shift_factor=shift,
                                 cycle=hz.CycleSpec("W", 2, 2, wj), fgmres_restart=5, precond_precision=prec, rhs_block=8)
    try:
        S = hz.HelmholtzSolver(P, o)
        S.solve_block(B)
        torch.cuda.synchronize(); t = time.time(); X, rep = S.solve_block(B); torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(method=method, prec=prec, shift=shift, wj=wj, cycles=rep.cycles, conv=bool(rep.all_converged()),
                              s=round(dt, 3), rhs_per_s=round(cfg.k / dt, 2))), flush=True)
        del S
    except Exception as e:
        print(json.dumps(dict(method=method, prec=prec, error=str(e)[:150])), flush=True)
