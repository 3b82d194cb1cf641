"""PIP acceptance threshold sweep on config 2 (cycles, speed, solution vs CGS2)."""
import os, sys, time, json
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1607_00968_b200 as hz
import bench
k = 32
cfg = bench.build_workload(0, 1, k)
P = hz.HelmholtzProblem.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
Xref = None
for ortho, eta in (("cgs2", "0"), ("pip", "0.5"), ("pip", "1e-2"), ("pip", "1e-4"), ("pip", "1e-6")):
    os.environ["HZ_ORTHO"] = ortho
    os.environ["HZ_PIP_ETA2"] = eta
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); t = time.time()
    X, rep = S.solve_block(B)
    torch.cuda.synchronize(); dt = time.time() - t
    Xn = X.cpu().numpy()
    if Xref is None:
        Xref = Xn
    diff = max(np.linalg.norm(Xn[:, j] - Xref[:, j]) / np.linalg.norm(Xref[:, j]) for j in range(k))
    print(json.dumps(dict(ortho=ortho, eta2=eta, cycles=rep.cycles, conv=rep.all_converged(),
                          worst=float(rep.rel_residual.max()), s=round(dt, 3), ms_per_cycle=round(1e3*dt/rep.cycles, 3),
                          rhs_per_s=round(k/dt, 2), grams=rep.block_gram_products, sol_diff_vs_cgs2=diff)), flush=True)
    del S
