"""GPU tier: the C++ drop-in header, the sharded FWI gradient path, device
(torch) buffers, and solves on the BASELINE config geometries at reduced
sizes, each against the compiled reference oracle."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CPP_DRIVER = r"""
#include <cstdio>
#include <cmath>
#include "hz_b200.hpp"
int main() {
  using namespace hzb;
  RegularGrid g; g.ndim = 2; g.n = {33, 33, 1};
  const std::int64_t n = g.num_nodes();
  SlownessSquaredModel m{g, Field(n, 0.25)};
  const double omega = 2 * M_PI * 2.0 / 10.0 * (1 - 1e-9);
  AttenuationField a{g, 0.01 * omega, {}, Field(n, 0.0)};
  auto prob = std::make_shared<HelmholtzProblem>(m, omega, a);
  HelmholtzSolveOptions o;  // reference defaults: MgBicgstab, W-cycle, 3 levels, shift 0.2
  HelmholtzSolver solver(prob, o);
  BlockVec<cplx> B(n, 2);
  B(16 + 33 * 2, 0) = 1.0;
  B(8 + 33 * 2, 1) = 1.0;
  auto res = solver.solve_block(B);
  BlockVec<cplx> R;
  prob->apply_block(res.first, R);
  double worst = 0;
  for (int j = 0; j < 2; ++j) {
    double r = 0, b = 0;
    for (std::int64_t i = 0; i < n; ++i) { r += std::norm(R(i, j) - B(i, j)); b += std::norm(B(i, j)); }
    worst = std::max(worst, std::sqrt(r / b));
  }
  bool threw = false;
  try { HelmholtzSolveOptions bad; bad.nlevels = 9; HelmholtzSolver s2(prob, bad); }
  catch (const ValidationError&) { threw = true; }
  std::printf("cycles %d converged %d residual %.3e threw %d\n", res.second.cycles,
              (int)res.second.all_converged(), worst, (int)threw);
  return (res.second.all_converged() && worst <= 1e-6 && threw) ? 0 : 1;
}
"""


def test_cpp_dropin_header_end_to_end():
    from paper_1607_00968_b200 import _native
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "drv.cpp")
        exe = os.path.join(d, "drv")
        open(src, "w").write(CPP_DRIVER)
        libdir = os.path.dirname(_native.LIB_PATH)
        r = subprocess.run(["g++", "-std=c++17", "-O1", src, "-I", os.path.join(ROOT, "include"), "-L", libdir,
                            "-lhz_b200", f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr


def test_fwi_gradient_matches_reference(ref):
    """Forward + adjoint block solves, device sensitivity accumulation and the
    (single-rank) all-reduce, against the reference's per-source
    fwi_sensitivity_output on its own solves (tight tolerance both sides)."""
    import torch
    from paper_1607_00968_b200 import parallel
    cfg = configs.config3(nlevels=3, n=(33, 33, 17), sgrid=2, layer=6)
    P = hz.HelmholtzProblem.from_config(cfg)
    opts = hz.HelmholtzSolveOptions(method="MgFgmres", tol=1e-10, max_cycles=400, nlevels=3, shift_factor=0.5,
                                    cycle=hz.CycleSpec("V"), fgmres_restart=10)
    S = hz.HelmholtzSolver(P, opts)
    n0, n1 = cfg.n[0], cfg.n[1]
    rec = np.array([i + n0 * j for j in range(2, n1 - 2, 3) for i in range(2, n0 - 2, 3)], dtype=np.int64)
    rng = np.random.default_rng(5)
    d_obs = rng.standard_normal((len(rec), cfg.k)) * 1e-3 + 0j
    res = parallel.fwi_gradient(P, S, cfg.source_nodes, rec, lambda ids: d_obs[:, ids])
    g = res.gradient.cpu().numpy()
    # reference: per-source forward + adjoint solves, sum of sensitivity outputs
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, 0.5)
    B = cfg.rhs_block()
    U, rep = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-10, max_cycles=400)
    r = U[rec] - d_obs
    Lr = np.zeros_like(U)
    Lr[rec] = np.conj(r)
    Lam, rep2 = ref.krylov_solve(R, H, Lr, method="fgmres", kind="V", restart=10, tol=1e-10, max_cycles=400)
    g_ref = sum(R.sensitivity_output(U[:, s].copy(), Lam[:, s].copy()) for s in range(cfg.k))
    assert rel_err(g, g_ref) <= 1e-6
    assert abs(res.misfit - 0.5 * np.sum(np.abs(r) ** 2)) <= 1e-8 * res.misfit


def test_device_tensor_solve_matches_host_solve():
    import torch
    cfg = configs.config1(nlevels=3, nx=65)
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    Xh, rh = S.solve_block(B)
    Xd, rd = S.solve_block(torch.from_numpy(B).cuda())
    assert rh.cycles == rd.cycles
    assert np.array_equal(Xh, Xd.cpu().numpy())  # deterministic reductions


def test_config2_geometry_reduced_c64_matches_reference(ref):
    """BASELINE config 2 recipe at 257x129 (same layered/faulted generator), the
    bench solver (FGMRES(5) + V(2,2), c64 preconditioner), vs the reference
    with the same blocking (c128 preconditioner)."""
    cfg = configs.config2(nlevels=3, k=8, nx=257, nz=129)
    cfg.shift, cfg.restart = 1.0, 5
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    X, rep = S.solve_block(B)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, cfg.shift)
    Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=5, tol=1e-6, max_cycles=cfg.max_cycles)
    assert rep.all_converged() and rr.all_converged()
    assert np.all(rep.rel_residual <= 1e-6)
    for j in range(B.shape[1]):
        assert rel_err(X[:, j], Xr[:, j]) <= 1e-5


@pytest.mark.parametrize("ortho", ["pip", "cgs2"])
def test_orthogonalisation_variants_agree(ref, ortho, monkeypatch):
    monkeypatch.setenv("HZ_ORTHO", ortho)
    cfg = configs.config1(nlevels=3, nx=65, k=8)
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    X, rep = S.solve_block(B)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, cfg.shift)
    Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-6, max_cycles=400)
    assert abs(rep.cycles - rr.cycles) <= 2
    for j in range(B.shape[1]):
        assert rel_err(X[:, j], Xr[:, j]) <= 1e-5


def test_kernel_profile_reports_launches():
    cfg = configs.config1(nlevels=3, nx=65)
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    with hz.kernel_profile() as prof:
        S.solve_block(cfg.rhs_block())
    names = set(prof.result)
    assert {"apply_fine_c128", "coarse_solve_c128"} <= names
    # the 2D fine level runs the fused pre-smoothing visit (fused.cu) or the plain sweep
    assert {"jacobi_fine_c128", "fused_pre_fine_c128"} & names
    assert all(r["ms"] > 0 for r in prof.result.values())


def test_rank_deficient_block_matches_reference(ref):
    """Coincident sources make the RHS block rank deficient: the reference's
    thin_qr zeroes the collapsed column (inc/block.hpp:126-131) and FGMRES
    treats a deficient W as happy breakdown (src/krylov.cpp:228-234). The
    device column Gram-Schmidt fallback must reproduce that behaviour."""
    cfg = configs.config1(nlevels=3, nx=65, k=4)
    cfg.source_nodes = np.array([20, 33, 20, 41], dtype=np.int64)  # column 2 == column 0
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    B = cfg.rhs_block()
    X, rep = S.solve_block(B)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, cfg.shift)
    Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-6, max_cycles=400)
    # Every restart starts with a collapsed column and ends in a happy
    # breakdown, so the restart points are decided by near-tol rounding: the
    # trajectories agree in shape (cycles, QR count) rather than bitwise.
    assert abs(rep.cycles - rr.cycles) <= 0.05 * rr.cycles + 2
    assert abs(rep.qr_factorizations - rr.qr_factorizations) <= 0.05 * rr.qr_factorizations + 2
    assert np.all(rep.rel_residual <= 2e-6) and np.all(rr.rel_residual <= 2e-6)
    for j in range(4):
        assert rel_err(X[:, j], Xr[:, j]) <= 1e-4
    assert rel_err(X[:, 2], X[:, 0]) <= 1e-12  # coincident sources, identical columns


@pytest.mark.parametrize("inverse,rows,permute,twisted", [("0", None, "2", "1"), ("0", "0", "1", "1"),
                                                          ("40000", None, "1", "1"), ("0", None, "0", "1"),
                                                          ("0", None, "2", "0"), ("0", "0", "0", "0")])
@pytest.mark.parametrize("n,nl", [((17, 17, 9), 2), ((33, 33, 17), 3), ((33, 17, 17), 2), ((17, 33, 25), 2)])
def test_block_tridiagonal_coarse_solve_matches_reference(ref, n, nl, inverse, rows, permute, twisted, monkeypatch):
    """The plane block-tridiagonal coarsest solver (coarse_bt.cu) against the
    reference's banded LU (MgHierarchy::coarse_solve, src/multigrid.cpp:114-117);
    rows = "0": transposed planes + split-K GEMM (the large-plane layout) instead
    of the row-owner kernel; inverse = 40000: the explicit inverse formed from
    the plane factors; permute = "2": the sweep runs along the longest axis of
    the coarsest grid (y for 9x9x5, x for 17x9x9, y for 9x17x13) on re-indexed
    planes, "1" (default): the same for planes above the row-owner limit
    (with rows = "0": all), "0": along z; twisted = "1" (default): two-sided
    elimination meeting at the middle plane on two streams, "0": one-sided."""
    monkeypatch.setenv("HZ_COARSE", "bt")
    monkeypatch.setenv("HZ_BT_TWISTED", twisted)
    monkeypatch.setenv("HZ_BT_PERMUTE", permute)
    monkeypatch.setenv("HZ_BT_INVERSE_MAX", inverse)
    if rows is not None:
        monkeypatch.setenv("HZ_BT_ROWS_MAX", rows)
    cfg = configs.small_problem(3, n, seed=3)
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method="MgFgmres", nlevels=nl, shift_factor=0.5,
                                                       cycle=hz.CycleSpec("V")))
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, nl, 0.5)
    dims, _ = H.level_dims(nl - 1)
    nc = dims[0] * dims[1] * dims[2]
    for k in (1, 16):
        b = configs.random_block(nc, k, seed=21 + k)
        assert rel_err(S.coarse_solve(b), H.coarse_solve(b)) <= 1e-11
    b = configs.random_block(cfg.num_nodes, 4, seed=5)
    assert rel_err(S.cycle(b), H.cycle(b, kind="V")) <= 1e-11


@pytest.mark.parametrize("n,nl", [((33, 33, 17), 2), ((17, 33, 25), 2)])
def test_block_tridiagonal_prefetch_and_dependent_launch_bitwise(n, nl, monkeypatch):
    """The plane-step chain with the next factor block prefetched into L2
    (HZ_BT_L2PF = 1 next block, 2 own block) and with programmatic dependent
    launches (HZ_BT_PDL = 1: a step starts while its predecessor runs and waits
    for it only before touching the data) gives the bits of the plain chain,
    through direct launches and through the graph-replayed c64 cycle."""
    import torch
    monkeypatch.setenv("HZ_COARSE", "bt")
    cfg = configs.small_problem(3, n, seed=3)
    P = hz.HelmholtzProblem.from_config(cfg)
    outs = {}
    for pf, pdl, graph, res in (("0", "0", "0", None), ("0", "0", "1", None), ("1", "0", "1", None), ("1", "1", "1", None),
                                ("2", "1", "0", None), ("0", "1", "1", None), ("0", "0", "1", "0"), ("1", "1", "0", "0"),
                                ("0", "0", "1", "8:2:128")):
        monkeypatch.setenv("HZ_BT_L2PF", pf)
        monkeypatch.setenv("HZ_BT_PDL", pdl)
        monkeypatch.setenv("HZ_BT_GRAPH", graph)  # the chain replayed from its own CUDA graph (default) or launched directly
        # plane-step kernel: r resident in shared memory (default), its 8-warp shape, or the row-owner kernel ("0"):
        # the same per-lane and butterfly order, hence the same bits
        if res is None:
            monkeypatch.delenv("HZ_BT_RES", raising=False)
        else:
            monkeypatch.setenv("HZ_BT_RES", res)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method="MgFgmres", nlevels=nl, shift_factor=0.5,
                                                           cycle=hz.CycleSpec("V"), precond_precision="c64",
                                                           fgmres_restart=5, tol=1e-6, max_cycles=30))
        R = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method="MgFgmres", nlevels=nl, shift_factor=0.5,
                                                           cycle=hz.CycleSpec("V")))
        b = configs.random_block(cfg.num_nodes, 8, seed=5)
        cyc = [R.cycle(b)]
        for _ in range(3):
            cyc.append(R.cycle(b))  # repeated launches of the chain
        try:
            X, rep = S.solve_block(b)  # graph-replayed c64 cycles
        except hz.ConvergenceError:
            X = None
        outs[(pf, pdl, graph, res)] = (cyc, X)
    base = outs[("0", "0", "0", None)]
    for key, (cyc, X) in outs.items():
        for a, c in zip(cyc, base[0]):
            assert np.array_equal(a, c), key
        assert (X is None) == (base[1] is None)
        if X is not None:
            assert np.array_equal(X, base[1]), key


def test_config3_three_levels_block_tridiagonal(ref):
    """Config-3 recipe at 65x65x33 with the converging 3-level hierarchy: the
    coarsest level (17x17x9) is solved by the plane block-tridiagonal solver."""
    import os
    os.environ["HZ_COARSE"] = "bt"
    try:
        cfg = configs.config3(nlevels=3, n=(65, 65, 33), sgrid=2, layer=8)
        P = hz.HelmholtzProblem.from_config(cfg)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    finally:
        del os.environ["HZ_COARSE"]
    B = cfg.rhs_block()
    X, rep = S.solve_block(B)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, cfg.shift)
    Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=10, tol=1e-6, max_cycles=cfg.max_cycles)
    assert rep.all_converged() and rr.all_converged()
    assert abs(rep.cycles - rr.cycles) <= 0.05 * rr.cycles + 2
    for j in range(B.shape[1]):
        assert rel_err(X[:, j], Xr[:, j]) <= 1e-5


def test_fused_c64_cycle_matches_unfused():
    """The complex64 preconditioner with the casts fused into the fine-level
    sweeps (cycle_cast) against cast + cycle + cast (HZ_FUSED_CAST=0), in a
    fresh process each (the switch is read once)."""
    import subprocess, sys
    code = (
        "import sys; sys.path.insert(0, '.'); import numpy as np\n"
        "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
        "cfg = configs.config2(nlevels=4, k=8, nx=257, nz=129); cfg.precond_precision = 'c64'\n"
        "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))\n"
        "np.save(sys.argv[1], S.cycle(configs.random_block(cfg.num_nodes, 8, seed=4)))\n")
    with tempfile.TemporaryDirectory() as d:
        outs = []
        for flag in ("1", "0"):
            path = os.path.join(d, f"x{flag}.npy")
            env = dict(os.environ, HZ_FUSED_CAST=flag)
            r = subprocess.run([sys.executable, "-c", code, path], cwd=ROOT, env=env, capture_output=True, text=True)
            assert r.returncode == 0, r.stderr
            outs.append(np.load(path))
        assert rel_err(outs[0], outs[1]) <= 1e-5
