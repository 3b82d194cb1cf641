"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
itself (oracle/_ref/libseistomo_ref.so = the unmodified seistomo sources
compiled by oracle/Makefile) on small seeded inputs.

    python tests/golden/make_golden.py

The fixtures pin the numpy restatement in oracle/port.py
(tests/test_oracle_port.py) and are the reference's answers the CPU test
tier checks against without needing /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1607_00968_b200 import configs  # noqa: E402


def problem_arrays(cfg):
    return dict(ndim=cfg.ndim, n=np.asarray(cfg.n), h=np.asarray(cfg.h), m=cfg.m, omega=cfg.omega,
                gamma_base=cfg.gamma_base, ramp=cfg.ramp)


def main():
    ref.set_num_threads(1)
    out = {}
    # operator applies
    for tag, ndim, n, k in (("apply2d", 2, (33, 17, 1), 4), ("apply3d", 3, (17, 17, 9), 3)):
        cfg = configs.small_problem(ndim, n, seed=5)
        R = ref.RefProblem.from_config(cfg)
        u = configs.random_block(cfg.num_nodes, k, seed=13)
        out[tag] = dict(problem_arrays(cfg), u=u, v=R.apply_block(u), mass=R.mass(), ppw=R.ppw())
    # hierarchies + cycles + coarse solves
    for tag, ndim, n, nl in (("hier2d", 2, (65, 33, 1), 3), ("hier3d", 3, (17, 17, 9), 2)):
        cfg = configs.small_problem(ndim, n, seed=6)
        R = ref.RefProblem.from_config(cfg)
        H = ref.RefHierarchy(R, nl, 0.5)
        d = dict(problem_arrays(cfg), nlevels=nl, shift=0.5)
        for l in range(nl):
            rp, ci, v = H.level_csr(l)
            d[f"rp{l}"], d[f"ci{l}"], d[f"v{l}"] = rp, ci, v
            d[f"dims{l}"] = np.asarray(H.level_dims(l)[0])
        b = configs.random_block(cfg.num_nodes, 2, seed=17)
        d["b"] = b
        d["xV"] = H.cycle(b, kind="V")
        d["xW"] = H.cycle(b, kind="W")
        if nl > 2:
            d["xK"] = H.cycle(b, kind="K")
        dims = H.level_dims(nl - 1)[0]
        bc = configs.random_block(dims[0] * dims[1] * dims[2], 2, seed=19)
        d["bc"], d["xc"] = bc, H.coarse_solve(bc)
        out[tag] = d
    # Krylov solves (same blocking), FGMRES(10)+V and the HelmholtzSolver default
    cfg = configs.small_problem(2, (65, 65, 1), seed=4)
    B = np.zeros((cfg.num_nodes, 3), np.complex128)
    for j, idx in enumerate([10 + 65 * 2, 32 + 65 * 2, 54 + 65 * 2]):
        B[idx, j] = 1.0
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, 0.5)
    X, rep = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-6, max_cycles=200)
    out["fgmres"] = dict(problem_arrays(cfg), B=B, X=X, cycles=rep.cycles, col_cycles=rep.col_cycles,
                         rel_residual=rep.rel_residual, history=rep.history, nlevels=3, shift=0.5)
    RS = ref.RefSolver(R, method="MgBicgstab")
    X, rep = RS.solve_block(B)
    out["bicgstab"] = dict(problem_arrays(cfg), B=B, X=X, cycles=rep.cycles, col_cycles=rep.col_cycles,
                           rel_residual=rep.rel_residual, history=rep.history, nlevels=3, shift=0.2)
    # dense kernels
    rng = np.random.default_rng(23)
    W = rng.standard_normal((200, 5)) + 1j * rng.standard_normal((200, 5))
    Q, Rq, rd = ref.thin_qr(W)
    A = rng.standard_normal((12, 8)) + 1j * rng.standard_normal((12, 8))
    Bl = rng.standard_normal((12, 4)) + 1j * rng.standard_normal((12, 4))
    Y, res = ref.least_squares(A, Bl)
    Xg = rng.standard_normal((50, 3)) + 1j * rng.standard_normal((50, 3))
    Yg = rng.standard_normal((50, 4)) + 1j * rng.standard_normal((50, 4))
    out["dense"] = dict(W=W, Q=Q, R=Rq, rd=rd, A=A, Bl=Bl, Y=Y, res=res, Xg=Xg, Yg=Yg, G=ref.gram(Xg, Yg))
    # attenuation ramp + sensitivity
    out["ramp"] = dict(r2=ref.attenuation_ramp(2, (33, 17), (4, 0), (4, 5)),
                       r3=ref.attenuation_ramp(3, (9, 11, 7), (2, 3, 0), (1, 2, 3)))
    cfg = configs.small_problem(2, (33, 17, 1), seed=5)
    R = ref.RefProblem.from_config(cfg)
    u = configs.random_block(cfg.num_nodes, 1, seed=1)[:, 0]
    lam = configs.random_block(cfg.num_nodes, 1, seed=2)[:, 0]
    out["sens"] = dict(problem_arrays(cfg), u=u, lam=lam, g=R.sensitivity_output(u, lam))
    for tag, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{tag}.npz"), **d)
        print("wrote", tag)


if __name__ == "__main__":
    main()
