"""GPU tier: blocked solves (HelmholtzSolveOptions.rhs_block = b). The k
columns are solved as ceil(k/b) independent block Krylov solves of <= b
contiguous columns, run concurrently (one stream + host thread per group,
hierarchy views sharing the operators). Each group must equal solve_block on
its own columns bitwise (concurrency and the shared hierarchy change nothing),
and the compiled reference's block_fgmres / block_bicgstab on the same
column group (the reference's solve_block, src/helmholtz_solver.cpp:61-79)
within the solver tolerance (solution parity holds at the same
blocking)."""
import dataclasses

import numpy as np
import pytest
import torch

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _cfg(k=10, **kw):
    cfg = configs.config1(nlevels=3, nx=65, k=k)
    return dataclasses.replace(cfg, **kw)


def _groups(k, b):
    return [slice(c, min(k, c + b)) for c in range(0, k, b)]


@pytest.mark.parametrize("precision,method,kind", [("c128", "fgmres", "V"), ("c64", "fgmres", "V"),
                                                   ("c128", "bicgstab", "W")])
def test_blocked_solve_equals_per_group_solve_block(precision, method, kind):
    cfg = _cfg(precond_precision=precision, method=method, cycle=kind)
    P = hz.HelmholtzProblem.from_config(cfg)
    B = cfg.rhs_block()
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=4))
    X, rep = S.solve_block(B)
    assert X.shape == B.shape
    if method == "fgmres":
        assert rep.all_converged()
    single = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    cyc = 0
    for g in _groups(B.shape[1], 4):  # groups of 4, 4, 2 columns
        Xg, rg = single.solve_block(np.ascontiguousarray(B[:, g]))
        assert np.array_equal(X[:, g], Xg)
        assert np.array_equal(rep.col_cycles[g], rg.col_cycles)
        assert np.array_equal(rep.rel_residual[g], rg.rel_residual)
        cyc = max(cyc, rg.cycles)
    assert rep.cycles == cyc
    # repeatable, and the device-block entry point gives the same columns
    X2, _ = S.solve_block(B)
    assert np.array_equal(X, X2)
    Xd, _ = S.solve_block(torch.from_numpy(B).cuda())
    assert np.array_equal(Xd.cpu().numpy(), X)


def test_blocked_solve_matches_reference_per_group(ref):
    cfg = _cfg(precond_precision="c64")
    P = hz.HelmholtzProblem.from_config(cfg)
    B = cfg.rhs_block()
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=4))
    X, rep = S.solve_block(B)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, cfg.nlevels, cfg.shift)
    for g in _groups(B.shape[1], 4):
        Xr, rr = ref.krylov_solve(R, H, np.ascontiguousarray(B[:, g]), method="fgmres", kind="V",
                                  restart=cfg.restart, tol=cfg.tol, max_cycles=cfg.max_cycles)
        assert rr.all_converged()
        assert abs(int(np.max(rep.col_cycles[g])) - rr.cycles) <= 0.05 * rr.cycles + 2
        for j, c in enumerate(range(g.start, g.stop)):
            assert rel_err(X[:, c], Xr[:, j]) <= 1e-5
    assert np.all(rep.rel_residual <= cfg.tol)


def test_rhs_block_at_least_k_is_one_block():
    cfg = _cfg(k=4)
    P = hz.HelmholtzProblem.from_config(cfg)
    B = cfg.rhs_block()
    Xa, ra = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=4)).solve_block(B)
    Xb, rb = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=0)).solve_block(B)
    assert np.array_equal(Xa, Xb) and ra.cycles == rb.cycles


def test_blocked_solve_3d_one_column_groups():
    cfg = configs.small_problem(3, (17, 17, 17))
    cfg = dataclasses.replace(cfg, nlevels=2, source_nodes=cfg.source_nodes[:3] if len(cfg.source_nodes) >= 3
                              else np.array([100, 2000, 4000], dtype=np.int64))
    P = hz.HelmholtzProblem.from_config(cfg)
    B = cfg.rhs_block()
    X, rep = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=1)).solve_block(B)
    S1 = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    for j in range(B.shape[1]):
        xj, rj = S1.solve_block(np.ascontiguousarray(B[:, j:j + 1]))
        assert np.array_equal(X[:, j:j + 1], xj)
        assert rep.col_cycles[j] == rj.col_cycles[0]


# ---- the Arnoldi block algebra on its own (K = 8 register-direct DMMA
# kernels, block_k8.cuh; other widths through the staged kernels)
@pytest.mark.parametrize("n,k,nb", [(525825, 8, 1), (525825, 8, 2), (100003, 8, 6), (4097, 8, 12),
                                    (13, 8, 3), (70001, 8, 13), (9001, 16, 3), (5003, 4, 2),
                                    (262913, 16, 1), (100003, 16, 6), (4099, 16, 12), (11, 16, 2),
                                    (20001, 16, 14), (3001, 32, 3)])
def test_block_gram_and_update_match_numpy(n, k, nb):
    rng = np.random.default_rng(n + k + nb)
    Xh = [rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)) for _ in range(nb)]
    Yh = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    Cs = rng.standard_normal((nb, k, k)) + 1j * rng.standard_normal((nb, k, k))
    Xd = [torch.from_numpy(x).cuda() for x in Xh]
    Yd = torch.from_numpy(Yh).cuda()
    G = hz.block_gram(Xd, Yd)
    for i in range(nb):
        ref_g = Xh[i].conj().T @ Yh
        assert rel_err(G[i], ref_g) <= 1e-13
    hz.block_add_scaled(Yd, Xd, Cs)
    ref_y = Yh + sum(Xh[i] @ Cs[i] for i in range(nb))
    assert rel_err(Yd.cpu().numpy(), ref_y) <= 1e-14


ZLO_SOLVE = (
    "import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
    "cfg = configs.config2(nlevels=4, k=int(sys.argv[2]), nx=257, nz=129); cfg.restart = 4\n"
    "cfg.shift, cfg.jacobi_weight, cfg.precond_precision, cfg.max_cycles = 0.9, 0.6, 'c64', 400\n"
    "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))\n"
    "X, rep = S.solve_block(cfg.rhs_block())\n"
    "assert rep.all_converged(), rep.rel_residual\n"
    "np.save(sys.argv[1], X)\n")


@pytest.mark.parametrize("k", [8, 16, 4])
def test_complex64_z_blocks_match_complex128_z_blocks(k):
    """FGMRES keeps the preconditioned blocks Z_j of a complex64 cycle in
    complex64 (HZ_ZLO, default on): the values are the c128 ones before their
    exact widening, so the K = 8 / 16 paths (same DMMA update kernels) are bitwise
    equal to the c128-Z run; other widths differ by the restart update's
    rounding only."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for flag in ("1", "0"):
            path = os.path.join(d, f"x{flag}.npy")
            r = subprocess.run([sys.executable, "-c", ZLO_SOLVE, path, str(k)], cwd=root,
                               env=dict(os.environ, HZ_ZLO=flag), capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    if k in (8, 16):
        assert np.array_equal(outs[0], outs[1])
    else:
        assert rel_err(outs[0], outs[1]) <= 1e-8


GA_SOLVE = (
    "import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
    "if sys.argv[2] == '2d':\n"
    "    cfg = configs.config2(nlevels=4, k=16, nx=257, nz=129); cfg.shift, cfg.jacobi_weight = 0.9, 0.6\n"
    "else:\n"
    "    cfg = configs.config3(nlevels=3, n=(33, 33, 17), sgrid=4)\n"
    "cfg.restart, cfg.precond_precision, cfg.max_cycles, cfg.krylov_block = 5, 'c64', 80, 8\n"
    "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))\n"
    "X, rep = S.solve_block(cfg.rhs_block())\n"
    "assert np.all(np.isfinite(X)) and rep.cycles > 0\n"
    "np.save(sys.argv[1], X)\n")


@pytest.mark.parametrize("dim", ["2d", "3d"])
def test_fused_apply_gram_matches_unfused(dim):
    """W = A Z fused with the Arnoldi Gram (gram8_apply_kernel, HZ_GRAM_APPLY=1,
    off by default, for 8-column blocks with c64 Z): the same W and the same
    partial Grams as apply_lo + gram8, so the blocked solves (2 groups of 8)
    are bitwise equal."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for flag in ("1", "0"):
            path = os.path.join(d, f"x{flag}.npy")
            r = subprocess.run([sys.executable, "-c", GA_SOLVE, path, dim], cwd=root,
                               env=dict(os.environ, HZ_GRAM_APPLY=flag), capture_output=True, text=True,
                               timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dim", ["2d", "3d"])
def test_two_column_apply_of_complex64_blocks_matches_one_column(dim):
    """W = A Z on complex64 Z blocks with two columns per thread
    (apply_lo2_kernel, default) against one column per thread
    (HZ_APPLY_LO2=0): the same per-column operations, bitwise equal solves."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for flag in ("1", "0"):
            path = os.path.join(d, f"x{flag}.npy")
            r = subprocess.run([sys.executable, "-c", GA_SOLVE, path, dim], cwd=root,
                               env=dict(os.environ, HZ_APPLY_LO2=flag), capture_output=True, text=True,
                               timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("k", [8, 4])
def test_cycle_graph_replay_matches_direct_launches(k):
    """The c64 preconditioner replayed from captured CUDA graphs
    (HZ_CYCLE_GRAPHS, default on) runs the same kernels on the same buffers
    as the direct launches: the solves are bitwise equal."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for flag in ("1", "0"):
            path = os.path.join(d, f"x{flag}.npy")
            r = subprocess.run([sys.executable, "-c", ZLO_SOLVE, path, str(k)], cwd=root,
                               env=dict(os.environ, HZ_CYCLE_GRAPHS=flag), capture_output=True, text=True,
                               timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
