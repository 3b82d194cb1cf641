"""GPU tier: the FWI path either side of the solve and the wavefield output
 against the compiled reference: receiver sampling
P^T u / P d and the sensitivity right-hand side bitwise, the Jacobian
products to solver tolerance, Compact16 quantisation bitwise and the JSWF1
files byte for byte."""
import os
import tempfile

import numpy as np
import pytest

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _receivers(cfg, nrec, seed, on_nodes=0):
    """Random physical receiver points inside the grid, some exactly on nodes
    and on the boundary (zero multilinear weights are skipped)."""
    rng = np.random.default_rng(seed)
    xyz = np.zeros((nrec, 3))
    for a in range(cfg.ndim):
        xyz[:, a] = rng.uniform(0.0, (cfg.n[a] - 1) * cfg.h[a], nrec)
    for r in range(on_nodes):
        for a in range(cfg.ndim):
            xyz[r, a] = float(rng.integers(0, cfg.n[a])) * cfg.h[a]
    if nrec > on_nodes + 1:
        xyz[on_nodes] = xyz[on_nodes + 1]  # coincident receivers: scatter order matters
    return xyz


@pytest.mark.parametrize("ndim,n", [(2, (65, 33)), (3, (17, 17, 9))])
def test_sampling_operator_bitwise(ref, ndim, n):
    cfg = configs.small_problem(ndim, n, seed=5)
    P = hz.HelmholtzProblem.from_config(cfg)
    xyz = _receivers(cfg, 40, seed=9, on_nodes=6)
    S = hz.SamplingOperator(P, xyz)
    R = ref.RefSampling(ndim, cfg.n, cfg.h, xyz)
    for r in range(40):
        a, wa = S.receiver(r)
        b, wb = R.receiver(r)
        assert np.array_equal(a, b) and np.array_equal(wa, wb)
    U = configs.random_block(cfg.num_nodes, 3, seed=2)
    D = S.sample(U)
    for c in range(3):
        assert np.array_equal(D[:, c], R.sample(U[:, c]))
    W = configs.random_block(40, 3, seed=4)
    A = S.sample_adjoint(W)
    Ac = S.sample_adjoint(W, conj=True)
    for c in range(3):
        assert np.array_equal(A[:, c], R.sample_adjoint(W[:, c]))
        assert np.array_equal(Ac[:, c], R.sample_adjoint(np.conj(W[:, c])))
    with pytest.raises(hz.ValidationError):
        hz.SamplingOperator(P, [[-5.0, 0.0, 0.0]])


def test_sensitivity_rhs_bitwise(ref):
    cfg = configs.small_problem(2, (65, 33), seed=6)
    P = hz.HelmholtzProblem.from_config(cfg)
    Rp = ref.RefProblem.from_config(cfg)
    U = configs.random_block(cfg.num_nodes, 2, seed=1)
    v = np.random.default_rng(3).standard_normal(cfg.num_nodes)
    got = hz.fwi_sensitivity_rhs(P, U, v)
    for c in range(2):
        assert np.array_equal(got[:, c], ref.fwi_sensitivity_rhs(Rp, U[:, c], v))


def _fwi_setup(ref):
    cfg = configs.config1(nlevels=3, nx=65, k=3)
    P = hz.HelmholtzProblem.from_config(cfg)
    opts = hz.HelmholtzSolveOptions(method="MgBicgstab", nlevels=3, shift_factor=0.5)
    S = hz.HelmholtzSolver(P, opts)
    Rp = ref.RefProblem.from_config(cfg)
    Rs = ref.RefSolver(Rp, method="MgBicgstab", nlevels=3, shift=0.5)
    xyz = np.zeros((30, 3))
    xyz[:, 0] = np.linspace(2.0, cfg.n[0] - 3.0, 30) + 0.37
    xyz[:, 1] = 1.5
    Smp = hz.SamplingOperator(P, xyz)
    Rsmp = ref.RefSampling(2, cfg.n, cfg.h, xyz)
    U, rep = S.solve_block(cfg.rhs_block())  # stored forward fields
    assert rep.all_converged()
    return cfg, S, Rs, Smp, Rsmp, U


def test_fwi_jacobian_vec_matches_reference(ref):
    cfg, S, Rs, Smp, Rsmp, U = _fwi_setup(ref)
    v = np.random.default_rng(11).standard_normal(cfg.num_nodes) * 0.01
    for c in range(U.shape[1]):
        d = hz.fwi_jacobian_vec(S, U[:, c], Smp, v)
        dr = ref.fwi_jacobian_vec(Rs, U[:, c], Rsmp, v)
        assert rel_err(d, dr) <= 1e-6
    # batched over the k stored fields: one block solve
    D = hz.fwi_jacobian_vec(S, U, Smp, v)
    for c in range(U.shape[1]):
        assert rel_err(D[:, c], ref.fwi_jacobian_vec(Rs, U[:, c], Rsmp, v)) <= 1e-4


def test_fwi_jacobian_transpose_vec_matches_reference(ref):
    cfg, S, Rs, Smp, Rsmp, U = _fwi_setup(ref)
    W = configs.random_block(Smp.num_receivers, U.shape[1], seed=8)
    total = np.zeros(cfg.num_nodes)
    for c in range(U.shape[1]):
        g = hz.fwi_jacobian_transpose_vec(S, U[:, c], Smp, W[:, c])
        gr = ref.fwi_jacobian_transpose_vec(Rs, U[:, c], Rsmp, W[:, c])
        assert rel_err(g, gr) <= 1e-6
        total += gr
    G = hz.fwi_jacobian_transpose_vec(S, U, Smp, W)
    assert rel_err(G, total) <= 1e-4
    # device tensors, accumulating
    import torch
    g0 = torch.zeros(cfg.num_nodes, dtype=torch.float64, device="cuda")
    g1 = hz.fwi_jacobian_transpose_vec(S, torch.from_numpy(U).cuda(), Smp, torch.from_numpy(W).cuda(), g=g0)
    assert rel_err(g1.cpu().numpy(), G) <= 1e-12


def _fields(n, nsrc, seed):
    rng = np.random.default_rng(seed)
    F = (rng.standard_normal((nsrc, n)) + 1j * rng.standard_normal((nsrc, n))) * np.array(
        [1e-3, 1.0, 7.5e4, 3.0][:nsrc])[:, None]
    F[0, :5] = 0.0
    F[1, 7] = 1e-12  # below binary16 range after scaling: subnormal / zero
    F[-1] = 0.0      # all-zero field: scale 1
    return F


def test_compact16_quantisation_bitwise(ref):
    dims = (33, 17)
    n = dims[0] * dims[1]
    F = _fields(n, 4, seed=3)
    expect = ref.wavefield_roundtrip(F, dims, compact=True)
    B = hz.WavefieldBatch(n, hz.Compact16)
    B.append_block(list(range(4)), np.ascontiguousarray(F.T))
    for s in range(4):
        assert np.array_equal(B.field(s), expect[s])
    # full storage is lossless
    full = ref.wavefield_roundtrip(F, dims, compact=False)
    assert np.array_equal(full, F)


@pytest.mark.parametrize("compact", [False, True])
def test_jswf1_files_match_reference_bytes(ref, compact):
    dims = (33, 17)
    n = dims[0] * dims[1]
    F = _fields(n, 3, seed=5)
    with tempfile.TemporaryDirectory() as d:
        pr, pm = os.path.join(d, "ref.jswf"), os.path.join(d, "ours.jswf")
        ref.wavefield_roundtrip(F, dims, compact=compact, path=pr)
        B = hz.WavefieldBatch(n, hz.Compact16 if compact else hz.Full32)
        for s in range(3):
            B.append(s, F[s])
        B.save(pm)
        assert open(pr, "rb").read() == open(pm, "rb").read()
        L = hz.WavefieldBatch.load(pr, n)
        Lr = ref.wavefield_load(pr, dims, 3)
        for s in range(3):
            assert np.array_equal(L.field(s), Lr[s])
        with pytest.raises(hz.IoError):
            hz.WavefieldBatch.load(pr, n + 1)


def test_solve_helmholtz_compact16_end_to_end():
    cfg = configs.config1(nlevels=3, nx=65, k=4)
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    rhs = [cfg.rhs_block()[:, c] for c in range(4)]
    full = hz.solve_helmholtz(S, rhs)
    comp = hz.solve_helmholtz(S, rhs, precision=hz.Compact16)
    assert len(full) == len(comp) == 4
    for s in range(4):
        u, q = full.field(s), comp.field(s)
        peak = max(np.abs(u.real).max(), np.abs(u.imag).max())
        assert np.abs(q.real - u.real).max() <= 2.0 ** -10 * peak * 2
        assert np.abs(q.imag - u.imag).max() <= 2.0 ** -10 * peak * 2
    # the GPU quantisation of the same fields reproduces the solve's batch
    X = np.stack([full.field(s) for s in range(4)], axis=1)
    Q, scales = hz.compact16(X)
    for s in range(4):
        assert np.array_equal(Q[s], comp._q[s]) and scales[s] == comp._scale[s]


CPP_FWI = r"""
#include <cstdio>
#include <cmath>
#include "hz_b200.hpp"
using namespace hzb;
int main(int argc, char** argv) {
  RegularGrid g; g.ndim = 2; g.n = {65, 33, 1};
  const std::int64_t n = g.num_nodes();
  SlownessSquaredModel m{g, Field(n, 0.25)};
  const double omega = 2 * M_PI * 2.0 / 10.0 * (1 - 1e-9);
  AttenuationField a{g, 0.01 * omega, {}, Field(n, 0.0)};
  auto prob = std::make_shared<HelmholtzProblem>(m, omega, a);
  HelmholtzSolveOptions o;
  HelmholtzSolver solver(prob, o);
  std::vector<std::array<double, 3>> rec;
  for (int i = 0; i < 20; ++i) rec.push_back({2.0 + 3.0 * i + 0.25, 1.5, 0.0});
  AcquisitionGeometry geom({{32.0, 0.0, 0.0}}, rec, 0.0, 1e9, g);
  SamplingOperator P(geom, *prob);
  CField q(n, cplx(0.0));
  q[32] = 1.0;
  SolveReport rep;
  WavefieldBatch fw = solve_helmholtz(solver, {q}, StoragePrecision::Full32, &rep);
  WavefieldBatch cw = solve_helmholtz(solver, {q}, StoragePrecision::Compact16);
  const CField u = fw.field(0), uc = cw.field(0);
  double peak = 0, err = 0;
  for (std::int64_t i = 0; i < n; ++i) {
    peak = std::max({peak, std::abs(u[i].real()), std::abs(u[i].imag())});
    err = std::max({err, std::abs(u[i].real() - uc[i].real()), std::abs(u[i].imag() - uc[i].imag())});
  }
  Field v(n, 0.0);
  for (std::int64_t i = 0; i < n; ++i) v[i] = 1e-3 * std::sin(0.1 * i);
  auto d = fwi_jacobian_vec(solver, u, P, v);
  std::vector<cplx> w(P.num_receivers(), cplx(1.0, -0.5));
  Field gr = fwi_jacobian_transpose_vec(solver, u, P, w);
  // adjoint identity up to solver tolerance (A complex symmetric):
  // Re sum_r conj(w_r) (J v)_r = sum_i v_i (J^T w)_i
  double lhs = 0, rhs = 0;
  for (std::size_t r = 0; r < d.size(); ++r) lhs += (std::conj(w[r]) * d[r]).real();
  for (std::int64_t i = 0; i < n; ++i) rhs += v[i] * gr[i];
  cw.save(argv[1]);
  WavefieldBatch back = WavefieldBatch::load(argv[1], g);
  const CField ub = back.field(0);
  double ferr = 0;
  for (std::int64_t i = 0; i < n; ++i) ferr = std::max(ferr, std::abs(ub[i] - uc[i]));
  std::printf("cycles %d qerr %.3e peak %.3e adj %.6e %.6e ferr %.3e\n", rep.cycles, err, peak, lhs, rhs, ferr);
  const bool ok = rep.all_converged() && err <= 2 * std::ldexp(peak, -10) &&
                  std::abs(lhs - rhs) <= 1e-4 * std::abs(lhs) && ferr <= 1e-3 * peak;
  return ok ? 0 : 1;
}
"""


def test_cpp_dropin_fwi_and_wavefield_output():
    import subprocess
    from paper_1607_00968_b200 import _native
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "fwi.cpp"), os.path.join(d, "fwi")
        open(src, "w").write(CPP_FWI)
        libdir = os.path.dirname(_native.LIB_PATH)
        r = subprocess.run(["g++", "-std=c++17", "-O1", src, "-I", os.path.join(root, "include"), "-L", libdir,
                            "-lhz_b200", f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe, os.path.join(d, "w.jswf")], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
