"""Uninitialised-read check without compute-sanitizer: fill the free device memory with a poison pattern, release it,
then build a solver and run cycles; any workspace read before it is written shows up as NaNs or as results that change
with the poison.  python scripts/poison_check.py [stencil] [HZ_STREAM3D]"""
import sys, os
sys.path.insert(0, ".")
stencil = int(sys.argv[1]) if len(sys.argv) > 1 else 7
os.environ["HZ_STREAM3D"] = sys.argv[2] if len(sys.argv) > 2 else "2"
import numpy as np, torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs

def poison(val):
    free, _ = torch.cuda.mem_get_info()
    n = int(free * 0.9) // 4
    t = torch.full((n,), val, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    del t
    torch.cuda.empty_cache()

for n, nl in (((97, 33, 65), 3), ((49, 37, 21), 2), ((65, 65, 33), 3)):
    cfg = configs.small_problem(3, n, seed=7, layer=3); cfg.stencil = stencil
    b = configs.random_block(cfg.num_nodes, 8, seed=11)
    res = {}
    for prec in ("c64", "c128"):
        for val in (0.0, float("nan"), 1e30, -7.25):
            poison(val)
            P = hz.HelmholtzProblem.from_config(cfg)
            S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method='MgFgmres', nlevels=nl, shift_factor=0.5,
                                                               cycle=hz.CycleSpec("V"), precond_precision=prec))
            x1 = S.cycle(b); x2 = S.cycle(b); x3 = S.cycle(b)
            X, rep = S.solve_block(b[:, :8])
            res[(prec, val)] = (x1, X)
            print(f"grid {n} {prec} poison {val}: finite {bool(np.all(np.isfinite(x1)))} x1==x2 {np.array_equal(x1, x2)} x1==x3 {np.array_equal(x1, x3)} "
                  f"same as poison 0: cycle {np.array_equal(x1, res[(prec, 0.0)][0])} solve {np.array_equal(X, res[(prec, 0.0)][1])}", flush=True)
            del S, P
