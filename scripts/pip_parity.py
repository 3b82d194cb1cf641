import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs
from oracle import ref
cfg = configs.config1(nlevels=3, nx=65, k=8)
B = cfg.rhs_block()
R = ref.RefProblem.from_config(cfg); H = ref.RefHierarchy(R, 3, cfg.shift)
Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-6, max_cycles=400)
print("ref cycles", rr.cycles, "res", rr.rel_residual.max(), "hist tail", rr.history[-3:])
for ortho, eta in (("cgs2", "0"), ("pip", "0.5"), ("pip", "1e-2"), ("pip", "1e-4")):
    os.environ["HZ_ORTHO"] = ortho; os.environ["HZ_PIP_ETA2"] = eta
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    X, rep = S.solve_block(B)
    d = max(np.linalg.norm(X[:, j] - Xr[:, j]) / np.linalg.norm(Xr[:, j]) for j in range(8))
    hd = np.max(np.abs(np.asarray(rep.history[:len(rr.history)]) - rr.history[:len(rep.history)]) / rr.history[:len(rep.history)])
    print(ortho, eta, "cycles", rep.cycles, "res", rep.rel_residual.max(), "sol diff", d, "max rel hist diff", hd, "grams", rep.block_gram_products)
