// A seistomo caller, written against the reference's public C++ API only
// (proj/core/include/seistomo/*.hpp). It compiles UNCHANGED against
//   * the reference:  -I /root/reference/proj/core/include + its sources
//     (oracle/Makefile target sec33_ref), and
//   * the B200 drop-in: -I include/seistomo_compat + libhz_b200.so
//     (tests/test_dropin_cpp.py).
// It runs the SURVEY §3.3 composition (grid -> attenuation -> problem ->
// point_source -> build_hierarchy -> BlockOperator -> block_fgmres) plus the
// solver facade, and writes every result to one binary file the test
// compares across the two builds.
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "seistomo/attenuation.hpp"
#include "seistomo/grid.hpp"
#include "seistomo/helmholtz.hpp"
#include "seistomo/helmholtz_solver.hpp"
#include "seistomo/krylov.hpp"
#include "seistomo/model.hpp"
#include "seistomo/multigrid.hpp"

using namespace seistomo;

namespace {
std::FILE* out_file = nullptr;
void put_tag(const char* tag) { std::fwrite(tag, 1, 8, out_file); }
void put_i64(std::int64_t v) { std::fwrite(&v, sizeof v, 1, out_file); }
void put_f64s(const double* p, std::int64_t count) {
  put_i64(count);
  std::fwrite(p, sizeof(double), static_cast<std::size_t>(count), out_file);
}
void put_field(const char* tag, const Field& f) {
  put_tag(tag);
  put_f64s(f.data(), static_cast<std::int64_t>(f.size()));
}
void put_cfield(const char* tag, const std::vector<cplx>& f) {
  put_tag(tag);
  put_f64s(reinterpret_cast<const double*>(f.data()), 2 * static_cast<std::int64_t>(f.size()));
}
void put_report(const char* tag, const SolveReport& r) {
  put_tag(tag);
  Field v{static_cast<double>(r.cycles), r.all_converged() ? 1.0 : 0.0};
  for (int c : r.col_cycles) v.push_back(c);
  for (double x : r.rel_residual) v.push_back(x);
  put_f64s(v.data(), static_cast<std::int64_t>(v.size()));
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.bin\n", argv[0]);
    return 2;
  }
  out_file = std::fopen(argv[1], "wb");
  if (!out_file) return 2;

  // 2D grid, origin away from 0 (point_source / nearest_node use it)
  const RegularGrid g(2, {129, 65, 1}, {1.0, 1.0, 1.0}, {10.0, 20.0, 0.0});
  Field vel(static_cast<std::size_t>(g.num_nodes()));
  double vmin = 1e30;
  for (std::int64_t idx = 0; idx < g.num_nodes(); ++idx) {
    const auto c = g.unpack(idx);
    const double z = static_cast<double>(c[1]) / 64.0;
    const double v = (1.5 + 2.5 * z) * (1.0 + 0.05 * std::sin(0.21 * c[0]) * std::cos(0.13 * c[1]));
    vel[static_cast<std::size_t>(idx)] = v;
    vmin = std::min(vmin, v);
  }
  Field m(vel.size());
  for (std::size_t i = 0; i < m.size(); ++i) m[i] = 1.0 / (vel[i] * vel[i]);
  const SlownessSquaredModel M(g, m);
  const double omega = 2.0 * M_PI * vmin / 10.0 * (1.0 - 1e-9);
  PerSideWidths layer;
  layer.lo = {12, 0, 0};  // depth-low side: the free surface
  layer.hi = {12, 12, 0};
  AttenuationField att = assemble_attenuation(g, 0.01 * omega, layer);
  put_field("ramp    ", att.ramp);
  for (double& r : att.ramp) r *= 0.1;
  auto prob = std::make_shared<const HelmholtzProblem>(M, omega, att);
  put_cfield("mass    ", prob->mass());
  put_cfield("gfactor ", prob->gamma_factor());

  // four sources; two sit exactly half-way between nodes (ties go low)
  const std::vector<std::array<double, 3>> xs = {
      {10.0 + 20.5, 20.0, 0.0}, {10.0 + 50.25, 20.7, 0.0}, {10.0 + 80.0, 20.0, 0.0}, {10.0 + 100.5, 21.5, 0.0}};
  BlockVec<cplx> B(g.num_nodes(), static_cast<int>(xs.size()));
  Field nodes;
  for (std::size_t j = 0; j < xs.size(); ++j) {
    B.set_col(static_cast<int>(j), prob->point_source(xs[j], cplx(1.0, 0.5 * static_cast<double>(j))));
    nodes.push_back(static_cast<double>(g.nearest_node(xs[j])));
  }
  put_field("nodes   ", nodes);
  put_cfield("B       ", B.a);

  // the shifted operator, materialised
  const auto A = prob->to_csr(0.5);
  Field rp(A.rp.begin(), A.rp.end()), ci(A.ci.begin(), A.ci.end());
  put_field("csr_rp  ", rp);
  put_field("csr_ci  ", ci);
  put_cfield("csr_v   ", A.v);

  // build_hierarchy + MgHierarchy::cycle + block_fgmres(10)
  const MgHierarchy<cplx> hier = build_hierarchy(*prob, 3, 0.5);
  const CycleSpec spec{CycleKind::V, 2, 2, 0.8, 2};
  BlockVec<cplx> Z(B.n, B.k);
  hier.cycle(spec, B, Z);  // one cycle from zero
  put_cfield("cycle   ", Z.a);
  BlockOperator op;
  op.n = g.num_nodes();
  op.apply = [&](const BlockVec<cplx>& u, BlockVec<cplx>& v) { prob->apply_block(u, v); };
  op.prec = [&](const BlockVec<cplx>& r, BlockVec<cplx>& z) {
    z = BlockVec<cplx>(r.n, r.k);
    hier.cycle(spec, r, z);
  };
  auto [X, rep] = block_fgmres(op, B, 10, 1e-6, 400, true);
  put_cfield("X_fgmres", X.a);
  put_report("R_fgmres", rep);

  // the facade: W-cycle block BiCGSTAB (the reference defaults)
  HelmholtzSolveOptions o;
  o.max_cycles = 400;
  HelmholtzSolver S(prob, o);
  auto [X2, rep2] = S.solve_block(B);
  put_cfield("X_bicg  ", X2.a);
  put_report("R_bicg  ", rep2);

  // sensitivity pieces on fixed fields
  CField u(static_cast<std::size_t>(g.num_nodes())), lam(u.size());
  Field v(u.size());
  for (std::size_t i = 0; i < u.size(); ++i) {
    u[i] = cplx(std::sin(0.01 * i), std::cos(0.02 * i));
    lam[i] = cplx(std::cos(0.03 * i), std::sin(0.005 * i));
    v[i] = 0.5 + std::sin(0.07 * i);
  }
  put_field("sens_out", fwi_sensitivity_output(*prob, u, lam));
  put_cfield("sens_rhs", fwi_sensitivity_rhs(*prob, u, v));

  std::fclose(out_file);
  std::printf("fgmres cycles %d converged %d; bicgstab cycles %d converged %d\n", rep.cycles,
              rep.all_converged() ? 1 : 0, rep2.cycles, rep2.all_converged() ? 1 : 0);
  return 0;
}
