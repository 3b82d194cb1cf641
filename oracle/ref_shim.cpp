// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference C++ library (seistomo, compiled
// from /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).
// It lets the Python tests, smoke() and bench.py's cpu_baseline / --impl
// reference arm drive the reference's own public API through ctypes with
// plain pointers. Every entry point names the reference symbol it forwards to.
//
// Layout conventions match the reference: complex blocks are node-major
// (a[i*k + j], inc/block.hpp:13-27), interleaved (re, im) doubles.

#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "seistomo/acquisition.hpp"
#include "seistomo/attenuation.hpp"
#include "seistomo/errors.hpp"
#include "seistomo/grid.hpp"
#include "seistomo/helmholtz.hpp"
#include "seistomo/helmholtz_solver.hpp"
#include "seistomo/krylov.hpp"
#include "seistomo/model.hpp"
#include "seistomo/multigrid.hpp"
#include "seistomo/parallel.hpp"

using namespace seistomo;

namespace {

thread_local std::string g_err;

int map_exception() {
  try {
    throw;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return 2;
  } catch (const BreakdownError& e) {
    g_err = e.what();
    return 3;
  } catch (const FactorizationError& e) {
    g_err = e.what();
    return 4;
  } catch (const StateError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

BlockVec<cplx> to_block(std::int64_t n, int k, const double* a) {
  BlockVec<cplx> b(n, k);
  std::memcpy(b.a.data(), a, sizeof(double) * 2 * n * k);
  return b;
}

void from_block(const BlockVec<cplx>& b, double* out) {
  std::memcpy(out, b.a.data(), sizeof(double) * 2 * b.n * b.k);
}

struct RefProblem {
  std::shared_ptr<const HelmholtzProblem> p;
};

struct RefHier {
  MgHierarchy<cplx> h;
};

struct RefSolver {
  std::unique_ptr<HelmholtzSolver> s;
};

}  // namespace

extern "C" {

// Plain report mirror of seistomo::SolveReport (inc/krylov.hpp:19-40).
struct ref_report {
  int cycles;
  int qr_factorizations;
  long long block_gram_products;
  double wall_s;
  int history_len;  // entries written to history (capped by history_cap)
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_num_threads(int n) { set_num_threads(n); }  // inc/parallel.hpp:14
int ref_num_threads() { return num_threads(); }

// HelmholtzProblem ctor (src/helmholtz.cpp:16-38) over SlownessSquaredModel
// and AttenuationField{base, ramp} (inc/attenuation.hpp:11-22).
int ref_problem_create(int ndim, const long long* n, const double* h, const double* m,
                       double omega, double gamma_base, const double* ramp, int allow_coarse,
                       void** out) {
  try {
    RegularGrid g(ndim, {n[0], n[1], n[2]}, {h[0], h[1], h[2]});
    const std::int64_t nn = g.num_nodes();
    SlownessSquaredModel model(g, Field(m, m + nn));
    AttenuationField att;
    att.grid = g;
    att.base = gamma_base;
    att.ramp.assign(ramp, ramp + nn);
    auto* rp = new RefProblem;
    rp->p = std::make_shared<HelmholtzProblem>(std::move(model), omega, std::move(att),
                                               allow_coarse != 0);
    *out = rp;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ref_problem_destroy(void* p) { delete static_cast<RefProblem*>(p); }

double ref_problem_ppw(void* p) { return static_cast<RefProblem*>(p)->p->points_per_wavelength(); }

// mass_ = omega^2 (1 - i gamma/omega) m  (src/helmholtz.cpp:31-37)
void ref_problem_mass(void* p, double* out) {
  const CField& m = static_cast<RefProblem*>(p)->p->mass();
  std::memcpy(out, m.data(), sizeof(cplx) * m.size());
}

// HelmholtzProblem::apply_block (src/helmholtz.cpp:71-100)
int ref_apply_block(void* p, long long n, int k, const double* u, double* out) {
  try {
    auto U = to_block(n, k, u);
    BlockVec<cplx> V;
    static_cast<RefProblem*>(p)->p->apply_block(U, V);
    from_block(V, out);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// HelmholtzProblem::point_source (src/helmholtz.cpp:124-132)
int ref_point_source(void* p, const double* x, double amp_re, double amp_im, double* out) {
  try {
    CField q = static_cast<RefProblem*>(p)->p->point_source({x[0], x[1], x[2]},
                                                            cplx(amp_re, amp_im));
    std::memcpy(out, q.data(), sizeof(cplx) * q.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// build_hierarchy (src/multigrid.cpp:204-208) -> MgHierarchy::build (:76-112)
int ref_hier_create(void* p, int nlevels, double shift, void** out) {
  try {
    auto* rh = new RefHier{build_hierarchy(*static_cast<RefProblem*>(p)->p, nlevels, shift)};
    *out = rh;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ref_hier_destroy(void* h) { delete static_cast<RefHier*>(h); }

int ref_hier_num_levels(void* h) { return static_cast<RefHier*>(h)->h.num_levels(); }

// MgHierarchy::level(l) (inc/multigrid.hpp:49): dims and CSR sizes of A_l
void ref_hier_level_info(void* h, int l, long long* dims, long long* nnz) {
  const auto& lev = static_cast<RefHier*>(h)->h.level(l);
  for (int a = 0; a < 3; ++a) dims[a] = lev.dims[a];
  *nnz = lev.A.nnz();
}

void ref_hier_level_csr(void* h, int l, long long* rp, int* ci, double* v) {
  const auto& A = static_cast<RefHier*>(h)->h.level(l).A;
  for (std::int64_t r = 0; r <= A.rows; ++r) rp[r] = A.rp[r];
  std::memcpy(ci, A.ci.data(), sizeof(int) * A.ci.size());
  std::memcpy(v, A.v.data(), sizeof(cplx) * A.v.size());
}

long long ref_hier_coarse_lu_bytes(void* h) { return static_cast<RefHier*>(h)->h.coarse_lu_bytes(); }

// MgHierarchy::cycle (inc/multigrid.hpp:53-55 -> src/multigrid.cpp:162-199).
// kind: 0 V, 1 W, 2 K.  x is updated in place (pass zeros for x0 = 0).
int ref_hier_cycle(void* h, int kind, int pre, int post, double wj, int k_inner, long long n,
                   int k, const double* b, double* x) {
  try {
    CycleSpec spec;
    spec.kind = kind == 0 ? CycleKind::V : (kind == 1 ? CycleKind::W : CycleKind::K);
    spec.pre = pre;
    spec.post = post;
    spec.jacobi_weight = wj;
    spec.k_inner = k_inner;
    auto B = to_block(n, k, b);
    auto X = to_block(n, k, x);
    static_cast<RefHier*>(h)->h.cycle(spec, B, X);
    from_block(X, x);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// MgHierarchy::coarse_solve (src/multigrid.cpp:114-117), in place
int ref_hier_coarse_solve(void* h, long long n, int k, double* b) {
  try {
    auto B = to_block(n, k, b);
    static_cast<RefHier*>(h)->h.coarse_solve(B);
    from_block(B, b);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

static void fill_report(const SolveReport& rep, int k, ref_report* out, int* col_cycles,
                        double* rel_res, int* converged, double* history, int history_cap) {
  out->cycles = rep.cycles;
  out->qr_factorizations = rep.qr_factorizations;
  out->block_gram_products = rep.block_gram_products;
  out->wall_s = rep.wall_s;
  const int hl = std::min<int>(history_cap, static_cast<int>(rep.history.size()));
  out->history_len = static_cast<int>(rep.history.size());
  for (int i = 0; i < hl; ++i) history[i] = rep.history[i];
  for (int j = 0; j < k; ++j) {
    col_cycles[j] = rep.col_cycles[j];
    rel_res[j] = rep.rel_residual[j];
    converged[j] = rep.converged[j];
  }
}

// The V-cycle + FGMRES(restart) composition of SURVEY §3.3:
// BlockOperator{apply = HelmholtzProblem::apply_block, prec = out:=0; cycle}
// (src/helmholtz_solver.cpp:60-68) -> block_fgmres (src/krylov.cpp:178-280)
// or block_bicgstab (src/krylov.cpp:60-176) when method == 1.
int ref_krylov_solve(void* p, void* h, int method, int kind, int pre, int post, double wj,
                     int k_inner, int restart, double tol, int max_cycles, long long n, int k,
                     const double* b, double* x, ref_report* rep_out, int* col_cycles,
                     double* rel_res, int* converged, double* history, int history_cap) {
  try {
    const HelmholtzProblem& prob = *static_cast<RefProblem*>(p)->p;
    const MgHierarchy<cplx>* hier = h ? &static_cast<RefHier*>(h)->h : nullptr;
    CycleSpec spec;
    spec.kind = kind == 0 ? CycleKind::V : (kind == 1 ? CycleKind::W : CycleKind::K);
    spec.pre = pre;
    spec.post = post;
    spec.jacobi_weight = wj;
    spec.k_inner = k_inner;
    BlockOperator op;
    op.n = n;
    op.apply = [&prob](const BlockVec<cplx>& v, BlockVec<cplx>& out) { prob.apply_block(v, out); };
    if (hier)
      op.prec = [hier, spec](const BlockVec<cplx>& v, BlockVec<cplx>& out) {
        out = BlockVec<cplx>(v.n, v.k);
        hier->cycle(spec, v, out);
      };
    auto B = to_block(n, k, b);
    auto res = method == 1 ? block_bicgstab(op, B, tol, max_cycles)
                           : block_fgmres(op, B, restart, tol, max_cycles, true);
    from_block(res.first, x);
    fill_report(res.second, k, rep_out, col_cycles, rel_res, converged, history, history_cap);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// HelmholtzSolver (src/helmholtz_solver.cpp:7-33) with HelmholtzSolveOptions
// (inc/helmholtz_solver.hpp:14-24). method: 0 MgBicgstab, 1 MgFgmresW,
// 2 MgFgmresK, 3 DenseLuSmall.
int ref_solver_create(void* p, int method, double tol, int max_cycles, int nlevels,
                      double shift, int pre, int post, double wj, int k_inner, int restart,
                      long long dense_threshold, void** out) {
  try {
    HelmholtzSolveOptions o;
    o.method = static_cast<HelmholtzMethod>(method);
    o.tol = tol;
    o.max_cycles = max_cycles;
    o.nlevels = nlevels;
    o.shift_factor = shift;
    o.cycle.pre = pre;
    o.cycle.post = post;
    o.cycle.jacobi_weight = wj;
    o.cycle.k_inner = k_inner;
    o.fgmres_restart = restart;
    o.dense_threshold = dense_threshold;
    auto* rs = new RefSolver;
    rs->s = std::make_unique<HelmholtzSolver>(static_cast<RefProblem*>(p)->p, o);
    *out = rs;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ref_solver_destroy(void* s) { delete static_cast<RefSolver*>(s); }

// HelmholtzSolver::solve_block (src/helmholtz_solver.cpp:35-72)
int ref_solver_solve_block(void* s, long long n, int k, const double* b, double* x,
                           ref_report* rep_out, int* col_cycles, double* rel_res, int* converged,
                           double* history, int history_cap) {
  try {
    auto B = to_block(n, k, b);
    auto res = static_cast<RefSolver*>(s)->s->solve_block(B);
    from_block(res.first, x);
    fill_report(res.second, k, rep_out, col_cycles, rel_res, converged, history, history_cap);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// fwi_sensitivity_output (src/helmholtz_solver.cpp:103-111)
int ref_sensitivity_output(void* p, const double* u, const double* lambda, double* g) {
  try {
    const HelmholtzProblem& prob = *static_cast<RefProblem*>(p)->p;
    const std::int64_t n = prob.grid().num_nodes();
    CField U(reinterpret_cast<const cplx*>(u), reinterpret_cast<const cplx*>(u) + n);
    CField L(reinterpret_cast<const cplx*>(lambda), reinterpret_cast<const cplx*>(lambda) + n);
    Field out = fwi_sensitivity_output(prob, U, L);
    std::memcpy(g, out.data(), sizeof(double) * n);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Block kernels of inc/block.hpp for unit-level pins.
void ref_gram(long long n, int kx, int ky, const double* x, const double* y, double* g) {
  auto X = to_block(n, kx, x);
  auto Y = to_block(n, ky, y);
  DenseMat<cplx> G = gram(X, Y);
  std::memcpy(g, G.a.data(), sizeof(cplx) * G.a.size());
}

int ref_thin_qr(long long n, int k, double* w, double* r) {
  auto W = to_block(n, k, w);
  DenseMat<cplx> R;
  bool rd = false;
  thin_qr(W, R, &rd);
  from_block(W, w);
  std::memcpy(r, R.a.data(), sizeof(cplx) * R.a.size());
  return rd ? 1 : 0;
}

// least_squares (inc/dense.hpp:118-175): A rows x cols, B rows x nrhs (row-major)
int ref_least_squares(long long rows, long long cols, long long nrhs, const double* a,
                      const double* b, double* y, double* res) {
  try {
    DenseMat<cplx> A(rows, cols), B(rows, nrhs);
    std::memcpy(A.a.data(), a, sizeof(cplx) * rows * cols);
    std::memcpy(B.a.data(), b, sizeof(cplx) * rows * nrhs);
    std::vector<double> rn;
    DenseMat<cplx> Y = least_squares(std::move(A), std::move(B), &rn);
    std::memcpy(y, Y.a.data(), sizeof(cplx) * cols * nrhs);
    std::memcpy(res, rn.data(), sizeof(double) * nrhs);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// assemble_attenuation (src/attenuation.cpp:8-41): ramp profile only.
int ref_attenuation_ramp(int ndim, const long long* n, const int* lo, const int* hi, double* ramp) {
  try {
    RegularGrid g(ndim, {n[0], n[1], n[2]}, {1.0, 1.0, 1.0});
    PerSideWidths w;
    for (int a = 0; a < 3; ++a) {
      w.lo[a] = lo[a];
      w.hi[a] = hi[a];
    }
    AttenuationField f = assemble_attenuation(g, 0.0, w);
    std::memcpy(ramp, f.ramp.data(), sizeof(double) * f.ramp.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// ---- FWI path either side of the solve
// SamplingOperator(AcquisitionGeometry, grid) (src/acquisition.cpp:10-62):
// receivers only (no sources), full offset range.
int ref_sampling_create(int ndim, const long long* n, const double* h, const double* origin, long long nrec,
                        const double* xyz, void** out) {
  try {
    RegularGrid g(ndim, {n[0], n[1], n[2]}, {h[0], h[1], h[2]}, {origin[0], origin[1], origin[2]});
    std::vector<std::array<double, 3>> rec(nrec);
    for (long long r = 0; r < nrec; ++r) rec[r] = {xyz[3 * r], xyz[3 * r + 1], xyz[3 * r + 2]};
    AcquisitionGeometry geom({}, rec, 0.0, 1e300, g);
    *out = new SamplingOperator(geom, g);
    return 0;
  } catch (...) {
    return map_exception();
  }
}
void ref_sampling_destroy(void* s) { delete static_cast<SamplingOperator*>(s); }
int ref_sampling_receiver(void* s, long long r, long long* nodes, double* w) {
  const auto* P = static_cast<SamplingOperator*>(s);
  const auto& nd = P->receiver_nodes(r);
  const auto& ww = P->receiver_weights(r);
  for (size_t q = 0; q < nd.size(); ++q) {
    nodes[q] = nd[q];
    w[q] = ww[q];
  }
  return int(nd.size());
}
// SamplingOperator::sample / sample_adjoint (inc/acquisition.hpp:40-61), one field
int ref_sample(void* s, const double* u, double* d) {
  try {
    const auto* P = static_cast<SamplingOperator*>(s);
    const std::int64_t n = P->grid().num_nodes();
    CField U(reinterpret_cast<const cplx*>(u), reinterpret_cast<const cplx*>(u) + n);
    auto D = P->sample(U);
    std::memcpy(d, D.data(), sizeof(cplx) * D.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}
int ref_sample_adjoint(void* s, const double* d, double* u) {
  try {
    const auto* P = static_cast<SamplingOperator*>(s);
    std::vector<cplx> D(reinterpret_cast<const cplx*>(d), reinterpret_cast<const cplx*>(d) + P->num_receivers());
    auto U = P->sample_adjoint(D);
    std::memcpy(u, U.data(), sizeof(cplx) * U.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}
// fwi_sensitivity_rhs (src/helmholtz_solver.cpp:95-101)
int ref_fwi_sensitivity_rhs(void* p, const double* u, const double* v, double* rhs) {
  try {
    const HelmholtzProblem& prob = *static_cast<RefProblem*>(p)->p;
    const std::int64_t n = prob.grid().num_nodes();
    CField U(reinterpret_cast<const cplx*>(u), reinterpret_cast<const cplx*>(u) + n);
    Field V(v, v + n);
    CField R = fwi_sensitivity_rhs(prob, U, V);
    std::memcpy(rhs, R.data(), sizeof(cplx) * n);
    return 0;
  } catch (...) {
    return map_exception();
  }
}
// fwi_jacobian_vec / fwi_jacobian_transpose_vec (src/helmholtz_solver.cpp:113-139)
int ref_fwi_jacobian_vec(void* solver, void* sampling, const double* u, const double* v, double* d) {
  try {
    const HelmholtzSolver& S = *static_cast<RefSolver*>(solver)->s;
    const auto* P = static_cast<SamplingOperator*>(sampling);
    const std::int64_t n = S.problem().grid().num_nodes();
    CField U(reinterpret_cast<const cplx*>(u), reinterpret_cast<const cplx*>(u) + n);
    Field V(v, v + n);
    auto D = fwi_jacobian_vec(S, U, *P, V);
    std::memcpy(d, D.data(), sizeof(cplx) * D.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}
int ref_fwi_jacobian_transpose_vec(void* solver, void* sampling, const double* u, const double* w, double* g) {
  try {
    const HelmholtzSolver& S = *static_cast<RefSolver*>(solver)->s;
    const auto* P = static_cast<SamplingOperator*>(sampling);
    const std::int64_t n = S.problem().grid().num_nodes();
    CField U(reinterpret_cast<const cplx*>(u), reinterpret_cast<const cplx*>(u) + n);
    std::vector<cplx> W(reinterpret_cast<const cplx*>(w), reinterpret_cast<const cplx*>(w) + P->num_receivers());
    Field G = fwi_jacobian_transpose_vec(S, U, *P, W);
    std::memcpy(g, G.data(), sizeof(double) * n);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// ---- wavefield output: WavefieldBatch (src/helmholtz.cpp:137-233)
// fields[s] (n0 x n1 2D grid) -> append (Full32 or Compact16) -> field(s)
// into out[s][n];
// optionally save(path) as JSWF1.
int ref_wavefield_roundtrip(long long n0, long long n1, int nsrc, const double* fields, int compact, double* out,
                            const char* path) {
  try {
    RegularGrid g(2, {n0, n1, 1}, {1.0, 1.0, 1.0});
    const long long n = n0 * n1;
    WavefieldBatch b(g, compact ? StoragePrecision::Compact16 : StoragePrecision::Full32);
    for (int s = 0; s < nsrc; ++s) {
      const cplx* f = reinterpret_cast<const cplx*>(fields) + size_t(s) * n;
      b.append(s, CField(f, f + n));
    }
    for (int s = 0; s < nsrc; ++s) {
      CField u = b.field(s);
      std::memcpy(out + 2 * size_t(s) * n, u.data(), sizeof(cplx) * n);
    }
    if (path && path[0]) b.save(path);
    return 0;
  } catch (...) {
    return map_exception();
  }
}
// WavefieldBatch::load (src/helmholtz.cpp:197-233) -> out[s][n]
int ref_wavefield_load(const char* path, long long n0, long long n1, int max_src, double* out, int* nsrc) {
  try {
    RegularGrid g(2, {n0, n1, 1}, {1.0, 1.0, 1.0});
    const long long n = n0 * n1;
    WavefieldBatch b = WavefieldBatch::load(path, g);
    *nsrc = int(b.size());
    for (int s = 0; s < int(b.size()) && s < max_src; ++s) {
      CField u = b.field(s);
      std::memcpy(out + 2 * size_t(s) * n, u.data(), sizeof(cplx) * n);
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
