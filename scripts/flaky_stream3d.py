"""Repeats the determinism check of tests/test_gpu_stream3d.py (two cycles from the same input must agree bitwise) in
one process per grid with HZ_STREAM3D=2 and reports where two results differ."""
import sys, os
sys.path.insert(0, ".")
os.environ.setdefault("HZ_STREAM3D", "2")
import numpy as np
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for n, nl in (((97, 33, 65), 3), ((65, 65, 33), 3)):
    cfg = configs.small_problem(3, n, seed=7, layer=3)
    P = hz.HelmholtzProblem.from_config(cfg)
    b = configs.random_block(cfg.num_nodes, 8, seed=11)
    bad = 0
    for prec in ("c64",):
        for it in range(reps):
            S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method='MgFgmres', nlevels=nl, shift_factor=0.5,
                                                               cycle=hz.CycleSpec("V"), precond_precision=prec))
            xs = [S.cycle(b) for _ in range(4)]
            for j in range(1, 4):
                if not np.array_equal(xs[0], xs[j]):
                    bad += 1
                    d = np.argwhere(xs[0] != xs[j])
                    nodes = np.unique(d[:, 0])
                    zz, rem = nodes // (n[0] * n[1]), nodes % (n[0] * n[1])
                    print(f"grid {n} rep {it} call {j}: {len(d)} entries differ, {len(nodes)} nodes, z range {zz.min()}..{zz.max()}, "
                          f"y range {(rem // n[0]).min()}..{(rem // n[0]).max()}, x range {(rem % n[0]).min()}..{(rem % n[0]).max()}, "
                          f"max rel {np.abs(xs[0] - xs[j]).max() / np.abs(xs[0]).max():.2e}", flush=True)
            del S
    print(f"grid {n}: {bad} differing calls in {reps} x 3", flush=True)
