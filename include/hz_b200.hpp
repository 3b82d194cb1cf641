// hz_b200.hpp -- header-only C++ drop-in over the C ABI (hz_b200.h).
//
// Mirrors the reference's solver-facing C++ API (seistomo,
// proj/core/include/seistomo/{grid,model,attenuation,block,krylov,multigrid,
// helmholtz,helmholtz_solver}.hpp) with the same names, argument meaning and
// exception classes, so a caller of the reference's Helmholtz solve path can
// switch by changing the include and the namespace, or unchanged: with
// HZ_B200_AS_SEISTOMO defined, namespace seistomo aliases this one, and
// include/seistomo_compat/seistomo/*.hpp provide the reference's include
// paths (tests/dropin/sec33_composition.cpp compiles unchanged against both).
// All computation happens in libhz_b200.so on the GPU; this header holds the
// host-side grid / attenuation setup and marshals everything else.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <type_traits>
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

// ---- inputs (grid.hpp:18-60, model.hpp:10-18, attenuation.hpp:11-28)
struct PerSideWidths {  // include/seistomo/grid.hpp:18-21
  std::array<int, 3> lo{0, 0, 0};
  std::array<int, 3> hi{0, 0, 0};
};

// RegularGrid (include/seistomo/grid.hpp:26-58, src/grid.cpp:10-55): host-side
// index arithmetic only
struct RegularGrid {
  int ndim = 2;
  std::array<std::int64_t, 3> n{1, 1, 1};
  std::array<double, 3> h{1.0, 1.0, 1.0};
  std::array<double, 3> origin{0.0, 0.0, 0.0};

  RegularGrid() = default;
  RegularGrid(int ndim_, std::array<std::int64_t, 3> n_, std::array<double, 3> h_,
              std::array<double, 3> origin_ = {0.0, 0.0, 0.0})
      : ndim(ndim_), n(n_), h(h_), origin(origin_) {
    if (ndim != 2 && ndim != 3) throw ValidationError("grid: ndim must be 2 or 3");
    if (ndim == 2) {
      n[2] = 1;
      h[2] = 1.0;
      origin[2] = 0.0;
    }
    for (int a = 0; a < ndim; ++a) {
      if (n[a] < 3) throw ValidationError("grid: axis " + std::to_string(a) + " needs at least 3 nodes");
      if (!(h[a] > 0.0)) throw ValidationError("grid: spacing on axis " + std::to_string(a) + " must be positive");
    }
    const std::int64_t cap = INT64_MAX;
    if (n[0] != 0 && cap / n[0] / n[1] < n[2]) throw ValidationError("grid: node count overflows index type");
  }
  std::int64_t num_nodes() const { return n[0] * n[1] * n[2]; }
  std::int64_t index(std::int64_t i, std::int64_t j, std::int64_t k = 0) const { return i + n[0] * (j + n[1] * k); }
  std::array<std::int64_t, 3> unpack(std::int64_t idx) const {
    return {idx % n[0], (idx / n[0]) % n[1], idx / (n[0] * n[1])};
  }
  std::array<double, 3> position(std::int64_t idx) const {
    const auto c = unpack(idx);
    return {origin[0] + c[0] * h[0], origin[1] + c[1] * h[1], origin[2] + c[2] * h[2]};
  }
  double min_h() const {
    double m = h[0];
    for (int a = 1; a < ndim; ++a) m = std::min(m, h[a]);
    return m;
  }
  bool contains(const std::array<double, 3>& x) const {
    const double eps = 1e-9;
    for (int a = 0; a < ndim; ++a) {
      const double lo = origin[a] - eps * h[a];
      const double hi = origin[a] + (n[a] - 1) * h[a] + eps * h[a];
      if (x[a] < lo || x[a] > hi) return false;
    }
    return true;
  }
  // exact half-spacing ties break toward the lower index
  std::int64_t nearest_node(const std::array<double, 3>& x) const {
    std::array<std::int64_t, 3> c{0, 0, 0};
    for (int a = 0; a < ndim; ++a) {
      const double f = (x[a] - origin[a]) / h[a];
      std::int64_t i = static_cast<std::int64_t>(std::floor(f + 0.5));
      if (static_cast<double>(i) - f == 0.5) --i;
      c[a] = std::clamp<std::int64_t>(i, 0, n[a] - 1);
    }
    return index(c[0], c[1], c[2]);
  }
  bool operator==(const RegularGrid& o) const {
    return ndim == o.ndim && n == o.n && h == o.h && origin == o.origin;
  }
  bool operator!=(const RegularGrid& o) const { return !(*this == o); }
};

struct SlownessSquaredModel {  // include/seistomo/model.hpp:10-18, src/model.cpp:13-19
  RegularGrid grid;
  Field values;
  SlownessSquaredModel() = default;
  SlownessSquaredModel(RegularGrid g, Field v) : grid(std::move(g)), values(std::move(v)) {
    if (static_cast<std::int64_t>(values.size()) != grid.num_nodes())
      throw ValidationError("model: value count does not match grid");
    for (double x : values)
      if (!(x > 0.0)) throw ValidationError("model: slowness-squared values must be positive");
  }
};

struct AttenuationField {  // include/seistomo/attenuation.hpp:11-22
  RegularGrid grid;
  double base = 0.0;
  PerSideWidths layer;
  Field ramp;  // in [0,1]: ((L-d)/L)^2 within each layer, max over sides
  Field gamma_at(double omega) const {
    Field g(ramp.size());
    for (std::size_t i = 0; i < g.size(); ++i) g[i] = base + omega * ramp[i];
    return g;
  }
};

// assemble_attenuation (src/attenuation.cpp:8-41): quadratic absorbing ramp,
// max over sides; width-0 sides (the free surface) get none. Setup on the
// host, like the reference.
inline AttenuationField assemble_attenuation(const RegularGrid& grid, double base_gamma, const PerSideWidths& layer) {
  if (base_gamma < 0.0) throw ValidationError("attenuation: base must be nonnegative");
  for (int a = 0; a < grid.ndim; ++a) {
    if (layer.lo[a] < 0 || layer.hi[a] < 0) throw ValidationError("attenuation: layer widths must be nonnegative");
    if (layer.lo[a] >= grid.n[a] / 2 + 1 || layer.hi[a] >= grid.n[a] / 2 + 1)
      throw ValidationError("attenuation: layer wider than half the grid on axis " + std::to_string(a));
  }
  AttenuationField f;
  f.grid = grid;
  f.base = base_gamma;
  f.layer = layer;
  f.ramp.assign(static_cast<std::size_t>(grid.num_nodes()), 0.0);
  for (std::int64_t idx = 0; idx < grid.num_nodes(); ++idx) {
    const auto c = grid.unpack(idx);
    double r = 0.0;
    for (int a = 0; a < grid.ndim; ++a) {
      if (layer.lo[a] > 0 && c[a] < layer.lo[a]) {
        const double L = layer.lo[a], d = static_cast<double>(c[a]);
        r = std::max(r, ((L - d) / L) * ((L - d) / L));
      }
      if (layer.hi[a] > 0 && c[a] > grid.n[a] - 1 - layer.hi[a]) {
        const double L = layer.hi[a], d = static_cast<double>(grid.n[a] - 1 - c[a]);
        r = std::max(r, ((L - d) / L) * ((L - d) / L));
      }
    }
    f.ramp[static_cast<std::size_t>(idx)] = r;
  }
  return f;
}

// ---- node-major block (block.hpp:17-39)
template <class S>
struct BlockVec {
  std::int64_t n = 0;
  int k = 0;
  std::vector<S> a;
  BlockVec() = default;
  BlockVec(std::int64_t n_, int k_) : n(n_), k(k_), a(static_cast<std::size_t>(n_) * k_, S{}) {}
  void set_zero() { std::fill(a.begin(), a.end(), S{}); }
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
  int rhs_block = 0;  // hz_options.rhs_block: 0 = one Krylov block over all columns
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

// ---- sparse matrix (csr.hpp:16-71): the materialised operator for callers
// that inspect it (HelmholtzProblem::to_csr); the solve never uses it
template <class S>
struct Csr {
  std::int64_t rows = 0, cols = 0;
  std::vector<std::int64_t> rp;  // size rows+1
  std::vector<std::int32_t> ci;  // column indices
  std::vector<S> v;
  Csr() = default;
  Csr(std::int64_t r, std::int64_t c) : rows(r), cols(c), rp(static_cast<std::size_t>(r) + 1, 0) {}
  std::int64_t nnz() const { return static_cast<std::int64_t>(v.size()); }
  void mul(const std::vector<S>& x, std::vector<S>& y) const {
    y.assign(static_cast<std::size_t>(rows), S{});
    for (std::int64_t r = 0; r < rows; ++r) {
      S acc{};
      for (std::int64_t e = rp[r]; e < rp[r + 1]; ++e) acc += v[e] * x[ci[e]];
      y[r] = acc;
    }
  }
  std::vector<S> diagonal() const {
    std::vector<S> d(static_cast<std::size_t>(rows), S{});
    for (std::int64_t r = 0; r < rows; ++r)
      for (std::int64_t e = rp[r]; e < rp[r + 1]; ++e)
        if (ci[e] == r) d[r] = v[e];
    return d;
  }
};

class HelmholtzProblem;
template <class S> class MgHierarchy;

namespace detail {
// Operator recognition for block_fgmres / block_bicgstab (below): while a
// Recorder is active on this thread, HelmholtzProblem::apply_block and
// MgHierarchy::cycle note what they were called with (they still compute).
struct Recorder {
  int applies = 0, cycles = 0;
  hz_problem* problem = nullptr;
  hz_solver* hier = nullptr;
  const hz_problem* hier_problem = nullptr;
  hz_cycle_spec spec{};
  bool x_was_zero = false;
};
inline Recorder*& recorder() {
  static thread_local Recorder* r = nullptr;
  return r;
}
inline hz_cycle_spec to_c(const CycleSpec& c) {
  hz_cycle_spec o{};
  o.kind = static_cast<int>(c.kind);
  o.pre = c.pre;
  o.post = c.post;
  o.jacobi_weight = c.jacobi_weight;
  o.k_inner = c.k_inner;
  return o;
}
}  // namespace detail

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
    const std::size_t nn = static_cast<std::size_t>(m_.grid.num_nodes());
    mass_.resize(nn);
    gamma_factor_.resize(nn);
    check(hz_problem_mass(p, reinterpret_cast<double*>(mass_.data())));
    check(hz_problem_gamma_factor(p, reinterpret_cast<double*>(gamma_factor_.data())));
  }
  const RegularGrid& grid() const { return m_.grid; }
  // complex mass w^2 (1 - i gamma/w) m and (1 - i gamma/w) per node (helmholtz.hpp:33-38)
  const CField& mass() const { return mass_; }
  const CField& gamma_factor() const { return gamma_factor_; }
  // the shifted operator as CSR (helmholtz.hpp:42-44, src/helmholtz.cpp:102-122)
  Csr<cplx> to_csr(double shift_factor = 0.0) const {
    std::int64_t nnz = 0;
    check(hz_problem_to_csr(h_.get(), shift_factor, nullptr, nullptr, nullptr, 0, &nnz));
    Csr<cplx> c(m_.grid.num_nodes(), m_.grid.num_nodes());
    c.ci.resize(static_cast<std::size_t>(nnz));
    c.v.resize(static_cast<std::size_t>(nnz));
    check(hz_problem_to_csr(h_.get(), shift_factor, c.rp.data(), c.ci.data(), reinterpret_cast<double*>(c.v.data()),
                            nnz, &nnz));
    return c;
  }
  // finite-volume point source amplitude / prod(h) at the nearest node, ties
  // toward the lower index (helmholtz.hpp:46-48, src/helmholtz.cpp:124-132)
  CField point_source(const std::array<double, 3>& x_s, cplx amplitude) const {
    CField q(static_cast<std::size_t>(m_.grid.num_nodes()));
    check(hz_problem_point_source(h_.get(), m_.grid.origin.data(), x_s.data(), amplitude.real(), amplitude.imag(),
                                  reinterpret_cast<double*>(q.data())));
    return q;
  }
  const SlownessSquaredModel& model() const { return m_; }
  const AttenuationField& attenuation() const { return gamma_; }
  double omega() const { return omega_; }
  double points_per_wavelength() const {
    double v = 0;
    check(hz_problem_ppw(h_.get(), &v));
    return v;
  }
  void apply_block(const BlockVec<cplx>& u, BlockVec<cplx>& out) const {
    if (auto* r = detail::recorder()) {
      ++r->applies;
      r->problem = h_.get();
    }
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
  CField mass_, gamma_factor_;
  std::shared_ptr<hz_problem> h_;
};

// ---- multigrid (multigrid.hpp:12-88)
// coarsen_dims (src/multigrid.cpp:11-25)
inline std::array<std::int64_t, 3> coarsen_dims(const std::array<std::int64_t, 3>& dims) {
  std::array<std::int64_t, 3> out = dims;
  for (int a = 0; a < 3; ++a) {
    if (dims[a] <= 1) continue;
    if (dims[a] % 2 == 0)
      throw ValidationError("multigrid: axis " + std::to_string(a) + " has even node count " +
                            std::to_string(dims[a]) + "; not coarsenable");
    const std::int64_t nc = (dims[a] - 1) / 2 + 1;
    if (nc < 3)
      throw ValidationError("multigrid: axis " + std::to_string(a) + " too small to coarsen (coarse count " +
                            std::to_string(nc) + ")");
    out[a] = nc;
  }
  return out;
}

// MgHierarchy<cplx>: the shifted-Laplacian Galerkin hierarchy resident on the
// GPU (one hz_solver owns it). Copies share the device hierarchy, as the
// reference's hierarchy is immutable after build.
template <class S>
class MgHierarchy {
  static_assert(std::is_same<S, cplx>::value, "the B200 hierarchy is complex128 (MgHierarchy<cplx>)");

 public:
  MgHierarchy() = default;
  // a view of the hierarchy owned by solver `s` (built from problem `p`)
  MgHierarchy(std::shared_ptr<hz_solver> s, const hz_problem* p) : s_(std::move(s)), p_(p) {}
  int num_levels() const {
    int l = 0;
    check(hz_hierarchy_num_levels(s_.get(), &l));
    return l;
  }
  std::array<std::int64_t, 3> level_dims(int l) const {
    std::array<std::int64_t, 3> d{1, 1, 1};
    check(hz_hierarchy_level_dims(s_.get(), l, d.data()));
    return d;
  }
  // one cycle on the level-0 system A X = B, updating x in place (multigrid.hpp:53-55)
  void cycle(const CycleSpec& spec, const BlockVec<S>& b, BlockVec<S>& x) const {
    if (x.n != b.n || x.k != b.k) throw ValidationError("cycle: x and b blocks differ in shape");
    bool zero = true;
    for (const S& v : x.a)
      if (v != S{}) {
        zero = false;
        break;
      }
    if (auto* r = detail::recorder()) {
      ++r->cycles;
      r->hier = s_.get();
      r->hier_problem = p_;
      r->spec = detail::to_c(spec);
      r->x_was_zero = zero;
    }
    const hz_cycle_spec cs = detail::to_c(spec);
    check(hz_hierarchy_cycle(s_.get(), &cs, b.n, b.k, reinterpret_cast<const double*>(b.a.data()),
                             reinterpret_cast<double*>(x.a.data()), zero ? 1 : 0));
  }
  // direct coarsest solve of all columns, in place (multigrid.hpp:58-60)
  void coarse_solve(BlockVec<S>& b) const {
    BlockVec<S> x(b.n, b.k);
    check(hz_coarse_solve(s_.get(), b.n, b.k, reinterpret_cast<const double*>(b.a.data()),
                          reinterpret_cast<double*>(x.a.data())));
    b = std::move(x);
  }
  hz_solver* handle() const { return s_.get(); }
  const hz_problem* problem_handle() const { return p_; }

 private:
  std::shared_ptr<hz_solver> s_;
  const hz_problem* p_ = nullptr;
};

// build_hierarchy (src/multigrid.cpp:204-208): level 0 is the shifted operator
// (gamma + shift_factor * omega), coarser levels by Galerkin products, the
// coarsest factored once -- all built on the problem's GPU.
inline MgHierarchy<cplx> build_hierarchy(const HelmholtzProblem& problem, int nlevels, double shift_factor = 0.2) {
  hz_options o;
  hz_options_default(&o);
  o.method = HZ_METHOD_MG_FGMRES;
  o.cycle_kind = HZ_CYCLE_V;
  o.nlevels = nlevels;
  o.shift_factor = shift_factor;
  hz_solver* s = nullptr;
  check(hz_solver_create(problem.handle(), &o, &s));
  return MgHierarchy<cplx>(std::shared_ptr<hz_solver>(s, [](hz_solver* q) { hz_solver_destroy(q); }),
                           problem.handle());
}

// ---- block Krylov (krylov.hpp:13-57)
struct BlockOperator {
  std::int64_t n = 0;
  std::function<void(const BlockVec<cplx>&, BlockVec<cplx>&)> apply;
  std::function<void(const BlockVec<cplx>&, BlockVec<cplx>&)> prec;  // optional
};

namespace detail {
// The solve runs on the GPU for the operator the reference's own callers
// build (src/helmholtz_solver.cpp:60-68): apply =
// HelmholtzProblem::apply_block, prec = out := 0; MgHierarchy::cycle(spec),
// both of the same problem. block_fgmres / block_bicgstab recognise it by
// calling op.apply and op.prec once on B while a Recorder is active, then
// check that the outputs are bit-for-bit those of the recognised operators.
// Any other operator is rejected (StateError): there is no host Krylov path.
inline std::pair<BlockVec<cplx>, SolveReport> krylov_on_device(const BlockOperator& op, const BlockVec<cplx>& B,
                                                              int method, int restart, double tol, int max_cycles,
                                                              const char* who) {
  if (op.n != B.n) throw ValidationError(std::string(who) + ": operator size does not match the block");
  if (!op.apply) throw ValidationError(std::string(who) + ": operator has no apply");
  const std::string reject = std::string(who) +
                             ": the B200 drop-in solves op = {HelmholtzProblem::apply_block, out := 0; "
                             "MgHierarchy::cycle} of one problem on the GPU; this operator is not that composition";
  if (!op.prec) throw StateError(reject + " (no preconditioner)");
  Recorder rec;
  BlockVec<cplx> V, Z(B.n, B.k);
  std::fill(Z.a.begin(), Z.a.end(), cplx(1.0, -1.0));  // stale content the preconditioner must overwrite
  recorder() = &rec;
  try {
    op.apply(B, V);
    op.prec(B, Z);
  } catch (...) {
    recorder() = nullptr;
    throw;
  }
  recorder() = nullptr;
  if (rec.applies != 1 || rec.cycles != 1 || !rec.problem || rec.hier_problem != rec.problem || !rec.x_was_zero)
    throw StateError(reject);
  BlockVec<cplx> V2(B.n, B.k), Z2(B.n, B.k);
  check(hz_apply_block(rec.problem, B.n, B.k, reinterpret_cast<const double*>(B.a.data()),
                       reinterpret_cast<double*>(V2.a.data())));
  check(hz_hierarchy_cycle(rec.hier, &rec.spec, B.n, B.k, reinterpret_cast<const double*>(B.a.data()),
                           reinterpret_cast<double*>(Z2.a.data()), 1));
  if (V.n != B.n || V.k != B.k || std::memcmp(V.a.data(), V2.a.data(), V2.a.size() * sizeof(cplx)) != 0 ||
      std::memcmp(Z.a.data(), Z2.a.data(), Z2.a.size() * sizeof(cplx)) != 0)
    throw StateError(reject + " (outputs differ)");
  BlockVec<cplx> X(B.n, B.k);
  SolveReport rep;
  std::vector<int> cc(B.k), cv(B.k);
  rep.rel_residual.resize(B.k);
  std::vector<double> hist(static_cast<std::size_t>(std::max(max_cycles, 0)) + 8);
  hz_report r{};
  r.col_cycles = cc.data();
  r.rel_residual = rep.rel_residual.data();
  r.converged = cv.data();
  r.history = hist.data();
  r.history_cap = static_cast<int>(hist.size());
  check(hz_block_krylov(rec.hier, method, &rec.spec, restart, tol, max_cycles, B.n, B.k,
                        reinterpret_cast<const double*>(B.a.data()), reinterpret_cast<double*>(X.a.data()), &r));
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
}  // namespace detail

// block_fgmres (krylov.hpp:54-57, src/krylov.cpp:178-280); `flexible` is
// accepted and ignored, as in the reference (directions are always stored)
inline std::pair<BlockVec<cplx>, SolveReport> block_fgmres(const BlockOperator& op, const BlockVec<cplx>& B,
                                                           int restart, double tol, int max_cycles,
                                                           bool flexible = true) {
  (void)flexible;
  return detail::krylov_on_device(op, B, 0, restart, tol, max_cycles, "block_fgmres");
}

// block_bicgstab (krylov.hpp:48-51, src/krylov.cpp:60-176)
inline std::pair<BlockVec<cplx>, SolveReport> block_bicgstab(const BlockOperator& op, const BlockVec<cplx>& B,
                                                             double tol, int max_cycles) {
  return detail::krylov_on_device(op, B, 1, 0, tol, max_cycles, "block_bicgstab");
}

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
    o.rhs_block = opts.rhs_block;
    hz_solver* s = nullptr;
    check(hz_solver_create(problem_->handle(), &o, &s));
    h_.reset(s, [](hz_solver* q) { hz_solver_destroy(q); });
    if (opts.method != HelmholtzMethod::DenseLuSmall)
      hier_ = std::make_shared<MgHierarchy<cplx>>(h_, problem_->handle());
    // the method fixes the cycle kind (src/helmholtz_solver.cpp:19-29)
    if (opts_.method == HelmholtzMethod::MgBicgstab || opts_.method == HelmholtzMethod::MgFgmresW)
      opts_.cycle.kind = CycleKind::W;
    else if (opts_.method == HelmholtzMethod::MgFgmresK)
      opts_.cycle.kind = CycleKind::K;
  }
  // the solver's hierarchy (nullptr for DenseLuSmall), helmholtz_solver.hpp:48
  const MgHierarchy<cplx>* hierarchy() const { return hier_.get(); }
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
  hz_solver* handle() const { return h_.get(); }
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
  std::shared_ptr<MgHierarchy<cplx>> hier_;
};

// fwi_sensitivity_rhs (helmholtz_solver.hpp:74-75, src/helmholtz_solver.cpp:95-101):
// -w^2 (1 - i gamma/w) u_s v, on the GPU
inline CField fwi_sensitivity_rhs(const HelmholtzProblem& problem, const CField& u_s, const Field& v) {
  const std::int64_t n = problem.grid().num_nodes();
  if (static_cast<std::int64_t>(u_s.size()) != n || static_cast<std::int64_t>(v.size()) != n)
    throw ValidationError("fwi_sensitivity_rhs: field size does not match grid");
  CField rhs(static_cast<std::size_t>(n));
  check(hz_fwi_sensitivity_rhs(problem.handle(), n, 1, reinterpret_cast<const double*>(u_s.data()), v.data(),
                               reinterpret_cast<double*>(rhs.data())));
  return rhs;
}

// fwi_sensitivity_output (helmholtz_solver.hpp:76-78, src/helmholtz_solver.cpp:103-111):
// Re(-w^2 (1 - i gamma/w) u_s lambda), on the GPU
inline Field fwi_sensitivity_output(const HelmholtzProblem& problem, const CField& u_s, const CField& lambda) {
  const std::int64_t n = problem.grid().num_nodes();
  if (static_cast<std::int64_t>(u_s.size()) != n || static_cast<std::int64_t>(lambda.size()) != n)
    throw ValidationError("fwi_sensitivity_output: field size does not match grid");
  Field g(static_cast<std::size_t>(n));
  check(hz_sensitivity_accumulate(problem.handle(), n, 1, reinterpret_cast<const double*>(u_s.data()),
                                  reinterpret_cast<const double*>(lambda.data()), g.data(), 0));
  return g;
}

// ---- acquisition (acquisition.hpp:9-62): receivers sampled on the GPU
struct AcquisitionGeometry {
  std::vector<std::array<double, 3>> sources;
  std::vector<std::array<double, 3>> receivers;
  double offset_min = 0.0;
  double offset_max = 0.0;
  std::vector<std::vector<std::uint8_t>> active;  // [source][receiver]
  AcquisitionGeometry() = default;
  AcquisitionGeometry(std::vector<std::array<double, 3>> src, std::vector<std::array<double, 3>> rec, double omin,
                      double omax, const RegularGrid& core_grid)
      : sources(std::move(src)), receivers(std::move(rec)), offset_min(omin), offset_max(omax) {
    if (omin < 0.0 || omax < omin) throw ValidationError("acquisition: bad offset range");
    auto inside = [&](const std::array<double, 3>& x) {
      for (int a = 0; a < core_grid.ndim; ++a) {
        const double lo = core_grid.origin[a] - 1e-9 * core_grid.h[a];
        const double hi = core_grid.origin[a] + (core_grid.n[a] - 1) * core_grid.h[a] + 1e-9 * core_grid.h[a];
        if (x[a] < lo || x[a] > hi) return false;
      }
      return true;
    };
    for (std::size_t i = 0; i < sources.size(); ++i)
      if (!inside(sources[i])) throw ValidationError("acquisition: source " + std::to_string(i) + " outside core grid");
    for (std::size_t i = 0; i < receivers.size(); ++i)
      if (!inside(receivers[i]))
        throw ValidationError("acquisition: receiver " + std::to_string(i) + " outside core grid");
    active.assign(sources.size(), std::vector<std::uint8_t>(receivers.size(), 0));
    for (std::size_t a = 0; a < sources.size(); ++a)
      for (std::size_t r = 0; r < receivers.size(); ++r) {
        double d2 = 0.0;
        for (int c = 0; c < core_grid.ndim; ++c) {
          const double dx = sources[a][c] - receivers[r][c];
          d2 += dx * dx;
        }
        const double d = std::sqrt(d2);
        active[a][r] = (d >= offset_min && d <= offset_max) ? 1 : 0;
      }
  }
  std::size_t num_sources() const { return sources.size(); }
  std::size_t num_receivers() const { return receivers.size(); }
  bool is_active(std::size_t a, std::size_t r) const { return active[a][r] != 0; }
};

// SamplingOperator: P^T u / P d as GPU gathers (node-major transpose for the
// scatter, so the sum order is the reference's without atomics).
class SamplingOperator {
 public:
  SamplingOperator(const AcquisitionGeometry& geom, const HelmholtzProblem& problem) : grid_(problem.grid()) {
    std::vector<double> xyz;
    for (const auto& r : geom.receivers) xyz.insert(xyz.end(), r.begin(), r.end());
    hz_sampling* p = nullptr;
    check(hz_sampling_create(problem.handle(), grid_.origin.data(), static_cast<std::int64_t>(geom.receivers.size()),
                             xyz.data(), &p));
    h_.reset(p, [](hz_sampling* q) { hz_sampling_destroy(q); });
  }
  std::size_t num_receivers() const { return static_cast<std::size_t>(hz_sampling_num_receivers(h_.get())); }
  const RegularGrid& grid() const { return grid_; }
  std::vector<cplx> sample(const CField& u) const {
    if (static_cast<std::int64_t>(u.size()) != grid_.num_nodes())
      throw ValidationError("sample: field size does not match grid");
    std::vector<cplx> d(num_receivers());
    check(hz_sample(h_.get(), 1, reinterpret_cast<const double*>(u.data()), reinterpret_cast<double*>(d.data())));
    return d;
  }
  CField sample_adjoint(const std::vector<cplx>& d) const {
    if (d.size() != num_receivers()) throw ValidationError("sample_adjoint: receiver count mismatch");
    CField u(static_cast<std::size_t>(grid_.num_nodes()));
    check(hz_sample_adjoint(h_.get(), 1, reinterpret_cast<const double*>(d.data()), reinterpret_cast<double*>(u.data()),
                            0));
    return u;
  }
  std::vector<std::int64_t> receiver_nodes(std::size_t r) const {
    std::int64_t nd[8];
    double w[8];
    int c = 0;
    check(hz_sampling_receiver(h_.get(), static_cast<std::int64_t>(r), nd, w, &c));
    return std::vector<std::int64_t>(nd, nd + c);
  }
  std::vector<double> receiver_weights(std::size_t r) const {
    std::int64_t nd[8];
    double w[8];
    int c = 0;
    check(hz_sampling_receiver(h_.get(), static_cast<std::int64_t>(r), nd, w, &c));
    return std::vector<double>(w, w + c);
  }
  hz_sampling* handle() const { return h_.get(); }

 private:
  RegularGrid grid_;
  std::shared_ptr<hz_sampling> h_;
};

namespace detail {
inline hz_report make_report(std::vector<int>& cc, std::vector<double>& rr, std::vector<int>& cv,
                             std::vector<double>& hist) {
  hz_report r{};
  r.col_cycles = cc.data();
  r.rel_residual = rr.data();
  r.converged = cv.data();
  r.history = hist.data();
  r.history_cap = static_cast<int>(hist.size());
  return r;
}
}  // namespace detail

// fwi_jacobian_vec (src/helmholtz_solver.cpp:113-125)
inline std::vector<cplx> fwi_jacobian_vec(const HelmholtzSolver& solver, const CField& u_s, const SamplingOperator& P,
                                          const Field& v) {
  const std::int64_t n = solver.problem().grid().num_nodes();
  if (static_cast<std::int64_t>(u_s.size()) != n) throw StateError("fwi_jacobian_vec: stored field does not match grid");
  if (v.size() != u_s.size()) throw ValidationError("fwi_jacobian_vec: model vector size mismatch");
  std::vector<cplx> d(P.num_receivers());
  std::vector<int> cc(1), cv(1);
  std::vector<double> rr(1), hist(static_cast<std::size_t>(solver.options().max_cycles) + 8);
  hz_report r = detail::make_report(cc, rr, cv, hist);
  const int st = hz_fwi_jacobian_vec(solver.handle(), P.handle(), n, 1, reinterpret_cast<const double*>(u_s.data()),
                                     v.data(), reinterpret_cast<double*>(d.data()), &r);
  hist.resize(std::min<std::size_t>(hist.size(), static_cast<std::size_t>(r.history_len)));
  check(st, hist);
  return d;
}

// fwi_jacobian_transpose_vec (src/helmholtz_solver.cpp:127-139)
inline Field fwi_jacobian_transpose_vec(const HelmholtzSolver& solver, const CField& u_s, const SamplingOperator& P,
                                        const std::vector<cplx>& w) {
  const std::int64_t n = solver.problem().grid().num_nodes();
  if (static_cast<std::int64_t>(u_s.size()) != n)
    throw StateError("fwi_jacobian_transpose_vec: stored field does not match grid");
  if (w.size() != P.num_receivers()) throw ValidationError("sample_adjoint: receiver count mismatch");
  Field g(static_cast<std::size_t>(n));
  std::vector<int> cc(1), cv(1);
  std::vector<double> rr(1), hist(static_cast<std::size_t>(solver.options().max_cycles) + 8);
  hz_report r = detail::make_report(cc, rr, cv, hist);
  const int st = hz_fwi_jacobian_transpose_vec(solver.handle(), P.handle(), n, 1,
                                               reinterpret_cast<const double*>(u_s.data()),
                                               reinterpret_cast<const double*>(w.data()), g.data(), 0, &r);
  hist.resize(std::min<std::size_t>(hist.size(), static_cast<std::size_t>(r.history_len)));
  check(st, hist);
  return g;
}

// ---- wavefield output (helmholtz.hpp:59-91)
enum class StoragePrecision { Full32, Compact16 };

namespace detail {
// IEEE binary16 <-> binary32, round to nearest even (host side of the
// JSWF1 f16 payload; the solve's own quantisation runs on the GPU)
inline std::uint16_t f32_to_f16(float x) {
  std::uint32_t b;
  std::memcpy(&b, &x, 4);
  const std::uint16_t sgn = static_cast<std::uint16_t>((b >> 16) & 0x8000u);
  const std::uint32_t ex = (b >> 23) & 0xffu, fr = b & 0x7fffffu;
  if (ex == 0xffu) return static_cast<std::uint16_t>(sgn | (fr ? 0x7e00u : 0x7c00u));
  const int e = static_cast<int>(ex) - 112;  // rebias 127 -> 15
  if (e >= 31) return static_cast<std::uint16_t>(sgn | 0x7c00u);
  std::uint32_t m, shift;
  if (e <= 0) {  // half subnormal (or zero)
    if (e < -10) return sgn;
    m = fr | 0x800000u;
    shift = static_cast<std::uint32_t>(14 - e);
  } else {
    m = (static_cast<std::uint32_t>(e) << 23) | fr;  // exponent rides above the mantissa
    shift = 13;
  }
  std::uint32_t q = m >> shift;
  const std::uint32_t rest = m & ((1u << shift) - 1u), half = 1u << (shift - 1u);
  if (rest > half || (rest == half && (q & 1u))) ++q;  // a carry into the exponent is correct
  return static_cast<std::uint16_t>(sgn | q);
}
inline float f16_to_f32(std::uint16_t v) {
  const std::uint32_t sgn = static_cast<std::uint32_t>(v & 0x8000u) << 16;
  const std::uint32_t ex = (v >> 10) & 0x1fu, fr = v & 0x3ffu;
  float out;
  if (ex == 0) {
    out = std::ldexp(static_cast<float>(fr), -24);  // zero / subnormal, exact
    return sgn ? -out : out;
  }
  const std::uint32_t bits = ex == 0x1fu ? (sgn | 0x7f800000u | (fr << 13)) : (sgn | ((ex + 112u) << 23) | (fr << 13));
  std::memcpy(&out, &bits, 4);
  return out;
}
}  // namespace detail

class WavefieldBatch {
 public:
  WavefieldBatch() = default;
  WavefieldBatch(RegularGrid grid, StoragePrecision precision) : grid_(std::move(grid)), precision_(precision) {}
  // Compact16 quantisation runs on the GPU (hz_compact16)
  void append(int source_id, const CField& u) {
    if (static_cast<std::int64_t>(u.size()) != grid_.num_nodes())
      throw ValidationError("wavefield batch: field size mismatch");
    source_ids_.push_back(source_id);
    if (precision_ == StoragePrecision::Full32) {
      full_.push_back(u);
      return;
    }
    const std::int64_t n = grid_.num_nodes();
    Compact c;
    c.re_im.resize(2 * static_cast<std::size_t>(n));
    check(hz_compact16(n, 1, reinterpret_cast<const double*>(u.data()), c.re_im.data(), &c.scale));
    compact_.push_back(std::move(c));
  }
  // k solved columns already quantised on the device (solve_helmholtz)
  void append_compact(int source_id, double scale, std::vector<std::uint16_t> re_im) {
    source_ids_.push_back(source_id);
    compact_.push_back(Compact{scale, std::move(re_im)});
  }
  CField field(std::size_t idx) const {
    if (idx >= source_ids_.size()) throw StateError("wavefield batch: no stored field at index");
    if (precision_ == StoragePrecision::Full32) return full_[idx];
    const Compact& c = compact_[idx];
    CField u(c.re_im.size() / 2);
    for (std::size_t i = 0; i < u.size(); ++i)
      u[i] = cplx(detail::f16_to_f32(c.re_im[2 * i]) * c.scale, detail::f16_to_f32(c.re_im[2 * i + 1]) * c.scale);
    return u;
  }
  int source_id(std::size_t idx) const { return source_ids_[idx]; }
  std::size_t size() const { return source_ids_.size(); }
  StoragePrecision precision() const { return precision_; }
  const RegularGrid& grid() const { return grid_; }
  // JSWF1: "JSWF1 <nsrc> <nnodes> <f32|f16>\n" + per-source little-endian (re, im)
  void save(const std::string& path) const {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("cannot open for write: " + path);
    const bool f32 = precision_ == StoragePrecision::Full32;
    bool ok = std::fprintf(f, "JSWF1 %zu %lld %s\n", size(), static_cast<long long>(grid_.num_nodes()),
                           f32 ? "f32" : "f16") > 0;
    for (std::size_t a = 0; a < size() && ok; ++a) {
      const CField u = field(a);
      if (f32) {
        std::vector<float> b(2 * u.size());
        for (std::size_t i = 0; i < u.size(); ++i) {
          b[2 * i] = static_cast<float>(u[i].real());
          b[2 * i + 1] = static_cast<float>(u[i].imag());
        }
        ok = std::fwrite(b.data(), sizeof(float), b.size(), f) == b.size();
      } else {
        std::vector<std::uint16_t> b(2 * u.size());
        for (std::size_t i = 0; i < u.size(); ++i) {
          b[2 * i] = detail::f32_to_f16(static_cast<float>(u[i].real()));
          b[2 * i + 1] = detail::f32_to_f16(static_cast<float>(u[i].imag()));
        }
        ok = std::fwrite(b.data(), sizeof(std::uint16_t), b.size(), f) == b.size();
      }
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw IoError("short write: " + path);
  }
  static WavefieldBatch load(const std::string& path, RegularGrid grid) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open: " + path);
    char magic[16] = {0}, tok[16] = {0};
    std::size_t nsrc = 0;
    long long nn = 0;
    if (std::fscanf(f, "%15s %zu %lld %15s", magic, &nsrc, &nn, tok) != 4 || std::string(magic) != "JSWF1" ||
        std::fgetc(f) != '\n') {
      std::fclose(f);
      throw IoError("bad JSWF1 header: " + path);
    }
    if (nn != grid.num_nodes()) {
      std::fclose(f);
      throw IoError("JSWF1 node count does not match grid: " + path);
    }
    const std::string t(tok);
    if (t != "f16" && t != "f32") {
      std::fclose(f);
      throw IoError("bad JSWF1 precision token: " + path);
    }
    WavefieldBatch b(std::move(grid), StoragePrecision::Full32);
    CField u(static_cast<std::size_t>(nn));
    for (std::size_t a = 0; a < nsrc; ++a) {
      if (t == "f16") {
        std::vector<std::uint16_t> buf(2 * static_cast<std::size_t>(nn));
        if (std::fread(buf.data(), 2, buf.size(), f) != buf.size()) {
          std::fclose(f);
          throw IoError("truncated JSWF1 payload: " + path);
        }
        for (long long i = 0; i < nn; ++i)
          u[i] = cplx(detail::f16_to_f32(buf[2 * i]), detail::f16_to_f32(buf[2 * i + 1]));
      } else {
        std::vector<float> buf(2 * static_cast<std::size_t>(nn));
        if (std::fread(buf.data(), 4, buf.size(), f) != buf.size()) {
          std::fclose(f);
          throw IoError("truncated JSWF1 payload: " + path);
        }
        for (long long i = 0; i < nn; ++i) u[i] = cplx(buf[2 * i], buf[2 * i + 1]);
      }
      b.append(static_cast<int>(a), u);
    }
    std::fclose(f);
    return b;
  }

 private:
  struct Compact {
    double scale = 1.0;
    std::vector<std::uint16_t> re_im;
  };
  RegularGrid grid_;
  StoragePrecision precision_ = StoragePrecision::Full32;
  std::vector<int> source_ids_;
  std::vector<CField> full_;
  std::vector<Compact> compact_;
};

// solve_helmholtz (src/helmholtz_solver.cpp:81-93): one block solve;
// Compact16 batches are quantised on the GPU and only the 4-byte entries
// come back to the host.
inline WavefieldBatch solve_helmholtz(const HelmholtzSolver& solver, const std::vector<CField>& rhs,
                                      StoragePrecision precision = StoragePrecision::Full32,
                                      SolveReport* report = nullptr) {
  const std::int64_t n = solver.problem().grid().num_nodes();
  const int k = static_cast<int>(rhs.size());
  BlockVec<cplx> B(n, k);
  for (int a = 0; a < k; ++a) B.set_col(a, rhs[a]);
  WavefieldBatch batch(solver.problem().grid(), precision);
  if (precision == StoragePrecision::Full32) {
    auto res = solver.solve_block(B);
    if (!res.second.all_converged())
      throw ConvergenceError("helmholtz solve: tolerance not met within cycle cap", res.second.history);
    for (int a = 0; a < k; ++a) batch.append(a, res.first.col(a));
    if (report) *report = res.second;
    return batch;
  }
  std::vector<std::uint16_t> q(2 * static_cast<std::size_t>(n) * k);
  std::vector<double> scales(k);
  std::vector<int> cc(k), cv(k);
  std::vector<double> rr(k), hist(static_cast<std::size_t>(solver.options().max_cycles) + 8);
  hz_report r = detail::make_report(cc, rr, cv, hist);
  const int st = hz_solve_helmholtz_compact16(solver.handle(), n, k, reinterpret_cast<const double*>(B.a.data()),
                                              q.data(), scales.data(), &r);
  hist.resize(std::min<std::size_t>(hist.size(), static_cast<std::size_t>(r.history_len)));
  check(st, hist);
  for (int a = 0; a < k; ++a)
    batch.append_compact(a, scales[a], std::vector<std::uint16_t>(q.begin() + 2 * n * a, q.begin() + 2 * n * (a + 1)));
  if (report) {
    report->cycles = r.cycles;
    report->col_cycles = cc;
    report->rel_residual = rr;
    report->converged.assign(cv.begin(), cv.end());
    report->history = hist;
    report->wall_s = r.wall_s;
    report->qr_factorizations = r.qr_factorizations;
    report->block_gram_products = r.block_gram_products;
  }
  return batch;
}

}  // namespace hzb

#ifdef HZ_B200_AS_SEISTOMO
namespace seistomo = hzb;
#endif
