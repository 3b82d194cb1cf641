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

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
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
  std::array<double, 3> origin{0.0, 0.0, 0.0};
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
    o.rhs_block = opts.rhs_block;
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
};

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
