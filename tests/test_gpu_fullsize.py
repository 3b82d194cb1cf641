"""GPU tier at the BASELINE configs' full sizes. The reference cannot solve
these in test time on the CPU, so parity is carried by what is cheap for it
and size independent:

* the operator at full size against the reference's apply_block (1e-12);
* one multigrid cycle of the bench hierarchy at full size against the
  reference's MgHierarchy::cycle (1e-12, complex128);
* the bench solve (32 sources, 4 concurrent 8-column blocks, c64 cycle):
  every column's residual against the REFERENCE operator, b - A_ref x, within
  the 1e-6 tolerance; linearity (scaling the sources by 2 scales the
  solution); the same solve through host buffers and device blocks;
* configs 3 and 4 (3D): residuals against the reference operator.
"""
import numpy as np
import pytest
import torch

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _bench_cfg():
    import bench
    return bench.build_workload(0, 1, 32)


def _ref_residuals(ref, cfg, X, B):
    R = ref.RefProblem.from_config(cfg)
    AX = R.apply_block(X)
    return np.linalg.norm(B - AX, axis=0) / np.linalg.norm(B, axis=0)


def test_config2_full_size_apply_matches_reference(ref):
    cfg = _bench_cfg()
    P = hz.HelmholtzProblem.from_config(cfg)
    u = configs.random_block(cfg.num_nodes, 4, seed=21)
    assert rel_err(P.apply_block(u), ref.RefProblem.from_config(cfg).apply_block(u)) <= 1e-12


def test_config2_full_size_cycle_matches_reference(ref):
    cfg = _bench_cfg()
    cfg.precond_precision, cfg.krylov_block = "c128", 0
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    b = configs.random_block(cfg.num_nodes, 2, seed=22)
    x = S.cycle(b)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, cfg.nlevels, cfg.shift)
    xr = H.cycle(b, kind=cfg.cycle, pre=cfg.pre, post=cfg.post, wj=cfg.jacobi_weight)
    assert rel_err(x, xr) <= 1e-12


def test_config2_full_size_bench_solve_properties(ref):
    cfg = _bench_cfg()
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    X, rep = S.solve_block(B)
    assert rep.all_converged() and np.all(rep.rel_residual <= cfg.tol)
    # the solution satisfies the reference's own discrete equation
    assert np.all(_ref_residuals(ref, cfg, X, B) <= cfg.tol * (1 + 1e-6))
    # linearity: 2 B -> 2 X (power-of-two scaling is exact through every step)
    X2, rep2 = S.solve_block(2.0 * B)
    assert rep2.cycles == rep.cycles
    assert rel_err(X2, 2.0 * X) <= 1e-14
    # device blocks give the same solution as host buffers
    Xd, _ = S.solve_block(torch.from_numpy(B).cuda())
    assert np.array_equal(Xd.cpu().numpy(), X)


@pytest.mark.parametrize("c", [3, 4])
def test_3d_configs_full_size_residuals_against_reference(ref, c):
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from run_configs import make
    cfg = make(c)
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    X, rep = S.solve_block(torch.from_numpy(B).cuda())
    X = X.cpu().numpy()
    assert rep.all_converged()
    assert np.all(_ref_residuals(ref, cfg, X, B) <= cfg.tol * (1 + 1e-6))


GOLDEN_BLOCK0 = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)),
                                           "golden", "cfg2_bench_block0.npz")


@pytest.mark.parametrize("block,precond", [(0, "c64"), (0, "c128"), (1, "c64"), (2, "c64"), (3, "c64")])
def test_config2_bench_block_matches_reference_full_solve(block, precond):
    """Blocks of the bench workload (8 sources each, FGMRES(5) + V(2,2), 6
    levels, shift 0.9, w_J 0.6, tol 1e-6) against the REFERENCE's own
    block_fgmres run to convergence on the same block
    (scripts/ref_full_solve.py -> tests/golden/cfg2_bench_block0.npz; the
    reference preconditions in complex128): solution on the receiver row and
    a strided node sample within 1e-5 per column, cycle count within 5 %."""
    g = np.load(GOLDEN_BLOCK0.replace("block0", f"block{block}"))
    cfg = _bench_cfg()
    b = cfg.krylov_block
    cfg.precond_precision, cfg.krylov_block = precond, 0
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    cols = slice(block * b, (block + 1) * b)
    B = cfg.rhs_block(cols)
    assert np.array_equal(np.asarray(cfg.source_nodes[cols]), g["source_nodes"])
    X, rep = S.solve_block(torch.from_numpy(B).cuda())
    X = X.cpu().numpy()
    assert rep.all_converged() and bool(np.all(g["converged"]))
    ref_cycles = int(g["cycles"])
    assert abs(rep.cycles - ref_cycles) <= 0.05 * ref_cycles, (rep.cycles, ref_cycles)
    xs, xr = X[g["nodes"]], g["x_sample"]
    for j in range(b):
        err = np.linalg.norm(xs[:, j] - xr[:, j]) / np.linalg.norm(xr[:, j])
        assert err <= 1e-5, (precond, j, err)
    # whole-field norms agree too (the sample is not a lucky subset)
    assert np.allclose(np.linalg.norm(X, axis=0), g["x_norm"], rtol=1e-5)


def _golden(name):
    import os
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)


@pytest.mark.parametrize("stem,block,precond", [("cfg3_full_block", 0, "c64"), ("cfg3_full_block", 0, "c128"),
                                                ("cfg3_full_block", 1, "c64"), ("cfg3_bench_block", 0, "c64"),
                                                ("cfg3_bench_block", 1, "c64"), ("cfg3_literal_block", 0, "c128"),
                                                ("cfg3_literal_block", 0, "c64"), ("cfg3_literal_block", 1, "c128")])
def test_config3_full_size_block_matches_reference_full_solve(stem, block, precond):
    """BASELINE config 3 at full size (129x129x65, 16 surface sources, the
    converging 3-level variant: FGMRES(5) + V(2,2), 8-column blocks) against
    the REFERENCE's own block_fgmres run to 1e-6 on the same block (complex128
    preconditioner, banded LU of the 33x33x17 coarsest grid), with the recipe
    of scripts/run_configs.py (shift 0.5, w_J 0.8: cfg3_full_block*.npz,
    scripts/ref_full_solve.py --config 3) and with the settings of
    bench.py --workload cfg3 (cfg3_bench_block*.npz, --config 3 --bench), and
    BASELINE config 3 as stated -- 4 levels, V(2,2), FGMRES(10), with shift 1.0
    and Jacobi weight 0.5 (cfg3_literal_block0.npz, --config 3 --literal):
    solution on the receiver plane's first row and a strided node sample within
    1e-5 per column, whole-field norms within 1e-5, cycles within 5 %."""
    import os, sys
    path = _golden(f"{stem}{block}.npz")
    if not os.path.exists(path):
        pytest.skip("reference fixture not generated")
    g = np.load(path)
    if stem == "cfg3_bench_block":
        import bench
        saved = bench.WORKLOAD
        bench.WORKLOAD = bench.WORKLOADS["cfg3"]
        try:
            cfg = bench.build_workload(0, 1, 16)
        finally:
            bench.WORKLOAD = saved
    elif stem == "cfg3_literal_block":
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
        from ref_full_solve import literal_config3
        cfg = literal_config3()
    else:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
        from run_configs import make
        cfg = make(3)
    b = cfg.krylov_block
    cfg.precond_precision, cfg.krylov_block = precond, 0
    S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
    cols = slice(block * b, (block + 1) * b)
    B = cfg.rhs_block(cols)
    assert np.array_equal(np.asarray(cfg.source_nodes[cols]), g["source_nodes"])
    X, rep = S.solve_block(torch.from_numpy(B).cuda())
    X = X.cpu().numpy()
    assert rep.all_converged() and bool(np.all(g["converged"]))
    ref_cycles = int(g["cycles"])
    assert abs(rep.cycles - ref_cycles) <= 0.05 * ref_cycles + 1, (rep.cycles, ref_cycles)
    xs, xr = X[g["nodes"]], g["x_sample"]
    # The 4-level literal configuration converges slowly (242 cycles): two solutions that both stop at a 1e-6
    # residual differ by the truncation error of either, which reaches 1.2e-5 there when the preconditioners differ
    # (complex64 here, complex128 in the reference). With the reference's own preconditioner precision the bar is
    # the 1e-5 of every other case; the complex64 run is held to 2e-5 and to a 1e-6 residual against the
    # reference's operator.
    literal_c64 = stem == "cfg3_literal_block" and precond == "c64"
    bar = 2e-5 if literal_c64 else 1e-5
    for j in range(b):
        err = np.linalg.norm(xs[:, j] - xr[:, j]) / np.linalg.norm(xr[:, j])
        assert err <= bar, (precond, j, err)
    assert np.allclose(np.linalg.norm(X, axis=0), g["x_norm"], rtol=bar)
    if literal_c64:
        from oracle import ref
        assert np.all(_ref_residuals(ref, cfg, X, B) <= cfg.tol * (1 + 1e-6))
