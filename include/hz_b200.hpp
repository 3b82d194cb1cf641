// hz_b200.hpp -- header-only C++ drop-in over the C ABI (hz_b200.h).
//
// Mirrors the reference's solver-facing C++ API (seistomo,
// proj/core/include/seistomo/{grid,model,attenuation,block,krylov,multigrid,
// helmholtz,helmholtz_solver}.hpp) with the same names, argument meaning and
// exception classes, so a caller of the reference's Helmholtz solve path can
// switch by changing the include and the namespace (or by defining
// HZ_B200_AS_SEISTOMO, which aliases namespace seistomo to this one when the
// reference headers are not also included). All computation happens in
// libhz_b200.so on the GPU; this header only marshals.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hz_b200.h"

namespace hzb {

using cplx = std::complex<double>;
using Field = std::vector<double>;
using CField = std::vector<cplx>;

// ---- errors (include/seistomo/errors.hpp:10-46)
class ValidationError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class ConvergenceError : public std::runtime_error {
 public:
  ConvergenceError(const std::string& what, std::vector<double> history)
      : std::runtime_error(what), residual_history(std::move(history)) {}
  std::vector<double> residual_history;
};
class BreakdownError : public std::runtime_error {
 public:
  BreakdownError(const std::string& what, int iteration) : std::runtime_error(what), iteration(iteration) {}
  int iteration;
};
class FactorizationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class StateError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int st, std::vector<double> history = {}) {
  if (st == HZ_OK) return;
  const std::string msg = hz_last_error_message();
  switch (st) {
    case HZ_VALIDATION: throw ValidationError(msg);
    case HZ_CONVERGENCE: throw ConvergenceError(msg, std::move(history));
    case HZ_BREAKDOWN: throw BreakdownError(msg, -1);
    case HZ_FACTORIZATION: throw FactorizationError(msg);
    case HZ_STATE: throw StateError(msg);
    case HZ_IO: throw IoError(msg);
    default: throw CudaError(msg);
  }
}

// ---- inputs (grid.hpp:26-35, model.hpp:10-18, attenuation.hpp:11-22)
struct RegularGrid {
  int ndim = 2;
  std::array<std::int64_t, 3> n{1, 1, 1};
  std::array<double, 3> h{1.0, 1.0, 1.0};
  std::int64_t num_nodes() const { return n[0] * n[1] * n[2]; }
};

struct SlownessSquaredModel {
  RegularGrid grid;
  Field values;
};

struct AttenuationField {
  RegularGrid grid;
  double base = 0.0;
  Field ramp;
  Field gamma_at(double omega) const {
    Field g(ramp.size());
    for (std::size_t i = 0; i < g.size(); ++i) g[i] = base + omega * ramp[i];
    return g;
  }
};

// ---- node-major block (block.hpp:17-39)
template <class S>
struct BlockVec {
  std::int64_t n = 0;
  int k = 0;
  std::vector<S> a;
  BlockVec() = default;
  BlockVec(std::int64_t n_, int k_) : n(n_), k(k_), a(static_cast<std::size_t>(n_) * k_, S{}) {}
  S& operator()(std::int64_t i, int j) { return a[i * k + j]; }
  const S& operator()(std::int64_t i, int j) const { return a[i * k + j]; }
  void set_col(int j, const std::vector<S>& v) {
    for (std::int64_t i = 0; i < n; ++i) a[i * k + j] = v[i];
  }
  std::vector<S> col(int j) const {
    std::vector<S> v(n);
    for (std::int64_t i = 0; i < n; ++i) v[i] = a[i * k + j];
    return v;
  }
};

// ---- options / report (multigrid.hpp:17-23, helmholtz_solver.hpp:12-24, krylov.hpp:19-40)
enum class CycleKind { V, W, K };
struct CycleSpec {
  CycleKind kind = CycleKind::W;
  int pre = 2;
  int post = 2;
  double jacobi_weight = 0.8;
  int k_inner = 2;
};
enum class HelmholtzMethod { MgBicgstab, MgFgmresW, MgFgmresK, DenseLuSmall, MgFgmres, MgBicgstabCycle };
enum class PreconditionerPrecision { C128, C64 };
struct HelmholtzSolveOptions {
  HelmholtzMethod method = HelmholtzMethod::MgBicgstab;
  double tol = 1e-6;
  int max_cycles = 200;
  int nlevels = 3;
  double shift_factor = 0.2;
  CycleSpec cycle{};
  int fgmres_restart = 5;
  std::int64_t dense_threshold = 3000;
  bool allow_coarse_ppw = false;
  PreconditionerPrecision precond_precision = PreconditionerPrecision::C128;
};

struct SolveReport {
  int cycles = 0;
  std::vector<int> col_cycles;
  std::vector<double> rel_residual;
  std::vector<char> converged;
  std::vector<double> history;
  double wall_s = 0.0;
  int qr_factorizations = 0;
  std::int64_t block_gram_products = 0;
  bool all_converged() const {
    for (char c : converged)
      if (!c) return false;
    return !converged.empty();
  }
};

// ---- operator (helmholtz.hpp:19-57)
class HelmholtzProblem {
 public:
  HelmholtzProblem(SlownessSquaredModel m_padded, double omega, AttenuationField gamma,
                   bool allow_coarse_ppw = false, int device = 0)
      : m_(std::move(m_padded)), omega_(omega), gamma_(std::move(gamma)) {
    if (gamma_.grid.n != m_.grid.n) throw ValidationError("helmholtz: attenuation grid mismatch");
    hz_problem* p = nullptr;
    check(hz_problem_create(m_.grid.ndim, m_.grid.n.data(), m_.grid.h.data(), m_.values.data(), omega,
                            gamma_.base, gamma_.ramp.data(), allow_coarse_ppw ? 1 : 0, device, &p));
    h_.reset(p, [](hz_problem* q) { hz_problem_destroy(q); });
  }
  const RegularGrid& grid() const { return m_.grid; }
  const SlownessSquaredModel& model() const { return m_; }
  const AttenuationField& attenuation() const { return gamma_; }
  double omega() const { return omega_; }
  double points_per_wavelength() const {
    double v = 0;
    check(hz_problem_ppw(h_.get(), &v));
    return v;
  }
  void apply_block(const BlockVec<cplx>& u, BlockVec<cplx>& out) const {
    if (out.n != u.n || out.k != u.k) out = BlockVec<cplx>(u.n, u.k);
    check(hz_apply_block(h_.get(), u.n, u.k, reinterpret_cast<const double*>(u.a.data()),
                         reinterpret_cast<double*>(out.a.data())));
  }
  void apply(const CField& u, CField& out) const {
    BlockVec<cplx> U(static_cast<std::int64_t>(u.size()), 1), V;
    U.a = u;
    apply_block(U, V);
    out = std::move(V.a);
  }
  hz_problem* handle() const { return h_.get(); }

 private:
  SlownessSquaredModel m_;
  double omega_;
  AttenuationField gamma_;
  std::shared_ptr<hz_problem> h_;
};

// ---- solver facade (helmholtz_solver.hpp:30-79)
class HelmholtzSolver {
 public:
  HelmholtzSolver(std::shared_ptr<const HelmholtzProblem> problem, HelmholtzSolveOptions opts)
      : problem_(std::move(problem)), opts_(opts) {
    hz_options o;
    hz_options_default(&o);
    o.method = static_cast<int>(opts.method);
    o.tol = opts.tol;
    o.max_cycles = opts.max_cycles;
    o.nlevels = opts.nlevels;
    o.shift_factor = opts.shift_factor;
    o.cycle_kind = static_cast<int>(opts.cycle.kind);
    o.pre = opts.cycle.pre;
    o.post = opts.cycle.post;
    o.jacobi_weight = opts.cycle.jacobi_weight;
    o.k_inner = opts.cycle.k_inner;
    o.fgmres_restart = opts.fgmres_restart;
    o.dense_threshold = opts.dense_threshold;
    o.precond_precision = opts.precond_precision == PreconditionerPrecision::C64 ? HZ_C64 : HZ_C128;
    hz_solver* s = nullptr;
    check(hz_solver_create(problem_->handle(), &o, &s));
    h_.reset(s, [](hz_solver* q) { hz_solver_destroy(q); });
  }
  const HelmholtzProblem& problem() const { return *problem_; }
  const HelmholtzSolveOptions& options() const { return opts_; }
  void set_tolerance(double tol) {
    opts_.tol = tol;
    check(hz_solver_set_tolerance(h_.get(), tol));
  }
  std::pair<BlockVec<cplx>, SolveReport> solve_block(const BlockVec<cplx>& B) const {
    BlockVec<cplx> X(B.n, B.k);
    SolveReport rep;
    std::vector<int> cc(B.k), cv(B.k);
    rep.rel_residual.resize(B.k);
    std::vector<double> hist(static_cast<std::size_t>(opts_.max_cycles) + 8);
    hz_report r{};
    r.col_cycles = cc.data();
    r.rel_residual = rep.rel_residual.data();
    r.converged = cv.data();
    r.history = hist.data();
    r.history_cap = static_cast<int>(hist.size());
    check(hz_solve_block(h_.get(), B.n, B.k, reinterpret_cast<const double*>(B.a.data()),
                         reinterpret_cast<double*>(X.a.data()), &r));
    rep.cycles = r.cycles;
    rep.qr_factorizations = r.qr_factorizations;
    rep.block_gram_products = r.block_gram_products;
    rep.wall_s = r.wall_s;
    rep.col_cycles = cc;
    rep.converged.assign(cv.begin(), cv.end());
    hist.resize(std::min<std::size_t>(hist.size(), static_cast<std::size_t>(r.history_len)));
    rep.history = std::move(hist);
    return {std::move(X), std::move(rep)};
  }
  std::pair<CField, SolveReport> solve(const CField& rhs) const {
    BlockVec<cplx> B(static_cast<std::int64_t>(rhs.size()), 1);
    B.set_col(0, rhs);
    auto res = solve_block(B);
    return {res.first.col(0), std::move(res.second)};
  }

 private:
  std::shared_ptr<const HelmholtzProblem> problem_;
  HelmholtzSolveOptions opts_;
  std::shared_ptr<hz_solver> h_;
};

// solve_helmholtz (src/helmholtz_solver.cpp:81-93), Full storage: one
// solution field per right-hand side; ConvergenceError if any column misses tol.
inline std::vector<CField> solve_helmholtz(const HelmholtzSolver& solver, const std::vector<CField>& rhs,
                                           SolveReport* report = nullptr) {
  const std::int64_t n = solver.problem().grid().num_nodes();
  BlockVec<cplx> B(n, static_cast<int>(rhs.size()));
  for (std::size_t s = 0; s < rhs.size(); ++s) B.set_col(static_cast<int>(s), rhs[s]);
  auto res = solver.solve_block(B);
  if (!res.second.all_converged())
    throw ConvergenceError("helmholtz solve: tolerance not met within cycle cap", res.second.history);
  std::vector<CField> out(rhs.size());
  for (std::size_t s = 0; s < rhs.size(); ++s) out[s] = res.first.col(static_cast<int>(s));
  if (report) *report = res.second;
  return out;
}

}  // namespace hzb

#ifdef HZ_B200_AS_SEISTOMO
namespace seistomo = hzb;
#endif
