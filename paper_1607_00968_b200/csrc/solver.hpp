// Host-side C++ driver of the B200 solver: the Helmholtz problem, the
// shifted-Laplacian multigrid hierarchy and the block Krylov methods. The
// control flow (cycle recursion, Krylov iterations, k x k algebra) runs on the
// host; every grid- or block-sized operation is an sm_100a kernel enqueued on
// the solver's stream.
#pragma once

#include <array>
#include <complex>
#include <functional>
#include <map>
#include <tuple>
#include <memory>
#include <vector>

#include "devbuf.hpp"
#include "kernels.hpp"
#include "slabs.hpp"

namespace hz {

using cplx = std::complex<double>;

// ------------------------------------------------------------------ problem
// Mirrors seistomo::HelmholtzProblem (inc/helmholtz.hpp:19-57,
// src/helmholtz.cpp:16-43): A = Lap_h + omega^2 (1 - i gamma/omega) m with
// gamma = base + omega * ramp (AttenuationField, inc/attenuation.hpp:11-22).
struct Problem {
  int ndim = 2;
  std::array<int64_t, 3> n{1, 1, 1};
  std::array<double, 3> h{1, 1, 1};
  double omega = 0, gamma_base = 0;
  std::vector<double> m, ramp;
  std::vector<cplx> mass, gamma_factor;  // host copies (reference arithmetic)
  double inv_h2[3] = {0, 0, 0};
  double center_lap = 0;
  int device = 0;
  // fine stencil: 7 = the reference's 5-point (2D) / 7-point (3D) operator;
  // 27 = the compact 27-point operator of config 4 (3D, uniform spacing; no
  // reference counterpart, weights from scripts/design_27pt.py)
  int stencil = 7;
  // device: centre of the unshifted operator (center_lap + mass) and (1 - i gamma/omega)
  DevBuf<double2> d_center, d_gf;
  // stencil 27: the mass and m on the device (couplings computed on the fly)
  DevBuf<double2> d_mass;
  DevBuf<double> d_m;

  Problem(int ndim, const int64_t* n, const double* h, const double* m, double omega,
          double gamma_base, const double* ramp, bool allow_coarse, int device, int stencil = 7);
  // 27 coefficient planes of the operator with gamma shifted by shift * omega
  void build_coef27(double shift, double2* planes, cudaStream_t s) const;
  // kFine27 weights {lap[0..3], mu[0..3]}
  void weights27(double* w8) const;
  int64_t num_nodes() const { return n[0] * n[1] * n[2]; }
  double points_per_wavelength() const;
  double min_h() const;
  // shifted centre (HelmholtzProblem::to_csr diagonal, src/helmholtz.cpp:108)
  std::vector<cplx> shifted_center(double shift) const;
  LevelOp<double> fine_op(int k) const;  // unshifted, for apply / residual
};

// explicit inverse of a 3D coarse level (transposed, row stride inv_ld(n))
// from its block-tridiagonal plane factors (coarse_bt.cu)
DevBuf<double2> bt_explicit_inverse(const LevelGeom& g, const double2* coef, const double2* ET, const double2* FT,
                                    cudaStream_t s);

// ------------------------------------------------------------------ cycles
enum class CycleKind : int { V = 0, W = 1, K = 2 };

struct CycleSpec {  // inc/multigrid.hpp:17-23
  CycleKind kind = CycleKind::W;
  int pre = 2;
  int post = 2;
  double jacobi_weight = 0.8;
  int k_inner = 2;
};

template <class T> class Fgmres;

// Per-level device storage of one precision.
template <class T>
struct MgLevelDev {
  using V = cplx_t<T>;
  std::array<int64_t, 3> dims{1, 1, 1};
  int kind = kFine;
  DevBuf<V> center;    // level 0: shifted centre
  DevBuf<V> coef;      // levels >= 1: [S][n] Galerkin planes
  DevBuf<V> inv_diag;  // D^{-1}
  DevBuf<V> cd;        // level 0 of the c64 hierarchy: (centre, D^{-1}) interleaved per node (fused k = 8 kernels)
  T w27[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // kFine27 weights (center = shifted per-node mass)
  T w[3] = {0, 0, 0};
  int64_t nodes() const { return dims[0] * dims[1] * dims[2]; }
};

// Shifted-Laplacian Galerkin hierarchy (MgHierarchy, inc/multigrid.hpp:44-80)
// held on the device in precision T, with the coarsest operator applied as
// an explicit inverse formed from the reference's banded LU factors.
template <class T>
class Hierarchy {
 public:
  using V = cplx_t<T>;
  Hierarchy() = default;
  Hierarchy(const Hierarchy&) = delete;
  Hierarchy& operator=(const Hierarchy&) = delete;
  ~Hierarchy();
  // Build from f64 setup data (the f64 hierarchy is always built first; the
  // c64 one is a rounded copy so both apply the same operators).
  static std::unique_ptr<Hierarchy<double>> build(const Problem& p, int nlevels, double shift,
                                                  cudaStream_t s);
  static std::unique_ptr<Hierarchy<float>> rounded(const Hierarchy<double>& h64, cudaStream_t s);

  int num_levels() const { return int(levels_.size()); }
  const MgLevelDev<T>& level(int l) const { return levels_[l]; }
  int ndim() const { return ndim_; }
  int64_t coarse_n() const { return levels_.back().nodes(); }
  int64_t coarse_band() const { return band_; }

  LevelOp<T> op(int l, int k) const;
  // One cycle on the level-0 system A X = B (x updated in place; x_zero
  // means the caller guarantees x == 0 on entry, as the preconditioner
  // application does, src/helmholtz_solver.cpp:65-68).
  void cycle(const CycleSpec& spec, int k, const V* b, V* x, bool x_zero, cudaStream_t s);
  void coarse_solve(int k, const V* b, V* x, cudaStream_t s);
  // complex64 hierarchy as the preconditioner of a complex128 block (casts
  // fused into the fine-level sweeps where possible)
  // (XO = double2: widened result; XO = float2: the complex64 result as is)
  template <class XO>
  void cycle_cast(const CycleSpec& spec, int k, const double2* b64, XO* x64, cudaStream_t s);
  // cycle_cast replayed from a CUDA graph per (b64, x64, k, spec) after its
  // first direct run (V / W cycles, not in slab mode or while profiling;
  // HZ_CYCLE_GRAPHS=0 disables): one launch instead of ~50 per cycle
  template <class XO>
  void cycle_cast_graph(const CycleSpec& spec, int k, const double2* b64, XO* x64, cudaStream_t s);
  // Galerkin planes / diagonal of level l (host copy, f64) for parity checks
  void download_level(int l, std::vector<cplx>& coef_or_center) const;
  // copy of the level operators (not the coarsest solver) on another GPU
  std::unique_ptr<Hierarchy<T>> replica(int device, cudaStream_t s) const;
  // same operators (aliased, not copied), private cycle workspace: one per
  // concurrently cycling RHS group
  std::unique_ptr<Hierarchy<T>> share() const;
  // Slab mode (slabs.hpp): levels below sl->agg_level() run on every part,
  // each part computing its own planes with the operators of reps[p] (a
  // hierarchy resident on part p's GPU); coarser levels and the coarsest
  // solve run on part 0. cycle() must then be called on part 0's stream
  // with b, x spanning level-0 vectors.
  void attach_slabs(const Slabs* sl, std::vector<const Hierarchy<T>*> reps);
  const Slabs* slabs() const { return sl_; }

  std::vector<MgLevelDev<T>> levels_;
  DevBuf<V> ainvT_;  // coarsest inverse, transposed [n_c][inv_ld(n_c)]
  DevBuf<V> cpart_;  // split-K partials of the coarse solve
  // block-tridiagonal plane solver of a large 3D coarsest level
  bool bt_ = false;
  DevBuf<V> bt_ET_, bt_FT_, bt_r_;
  // sweep-axis permutation of the plane solver (identity: planes of axis 2);
  // bt_coef_ = the coarsest operator's planes on the permuted grid, bt_b_ /
  // bt_x_ = the re-indexed right-hand side / solution of a solve
  BtAux bt_aux_;
  int bt_perm_[3] = {0, 1, 2};
  DevBuf<V> bt_coef_, bt_b_, bt_x_;
  bool bt_permuted() const { return bt_perm_[0] != 0 || bt_perm_[1] != 1 || bt_perm_[2] != 2; }
  int ndim_ = 2;
  int64_t band_ = 0;

 private:
  void ensure_ws(int k);
  void cycle_rec(int l, const CycleSpec& spec, int k, const V* b, V* x, bool x_zero,
                 cudaStream_t s);
  void relax(int l, const CycleSpec& spec, int sweeps, int k, const V* b, V*& cur, V*& other,
             bool& cur_zero, cudaStream_t s);
  void kcycle_coarse(int l, const CycleSpec& spec, int k, const V* b, V* x, cudaStream_t s);
  void coarse_correction(int l, const CycleSpec& spec, int k, const V* b, V* cur, bool cur_zero,
                         cudaStream_t s);
  // the coarse visit(s) of level l's correction: level l+1 solved from
  // wb_[l+1] into wx_[l+1] (V / W / K per spec.kind)
  void coarse_visit(int l, const CycleSpec& spec, int k, cudaStream_t s);
  void coarse_visit_on(int l, const CycleSpec& spec, int k, cudaStream_t s);
  bool fused_level0(const CycleSpec& spec, int k) const;
  bool slab_level(int l) const { return sl_ && l < sl_->agg_level(); }
  // f(op, stream, row0, rows) once per part owning level l (slab levels), or
  // once on stream s over the whole grid
  template <class F>
  void on_level(int l, int k, cudaStream_t s, F&& f);
  const Slabs* sl_ = nullptr;
  std::vector<const Hierarchy<T>*> reps_;
  int ws_k_ = 0;
  std::vector<DevBuf<V>> wx_, wt_, wb_, wr_;  // per level: solution, ping-pong, rhs, residual
  std::vector<std::unique_ptr<Fgmres<T>>> kfgm_;
  struct GraphKey {
    const void* b;
    const void* x;
    int k, kind, pre, post;
    double wj;
    bool operator<(const GraphKey& o) const {
      return std::tie(b, x, k, kind, pre, post, wj) < std::tie(o.b, o.x, o.k, o.kind, o.pre, o.post, o.wj);
    }
  };
  struct GraphRec {
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
  };
  std::map<GraphKey, GraphRec> graphs_;
  void clear_graphs();
  // the plane-solver chain of a coarsest-level solve (≈ 130-260 dependent
  // launches) as its own graph per (b, x, k), replayed wherever the cycle
  // itself is not graph-replayed (complex128 cycles, profiled runs)
  std::map<std::tuple<const void*, const void*, int>, GraphRec> bt_graphs_;
  void coarse_solve_bt(int k, const V* b, V* x, cudaStream_t s);
  // high-priority stream of the coarse part of the cycle (coarse_visit)
  cudaStream_t hp_ = nullptr;
  cudaEvent_t hp_fork_ = nullptr, hp_join_ = nullptr;
};

// explicit inverse of the unshifted operator (HelmholtzMethod::DenseLuSmall)
DevBuf<double2> dense_inverse(const Problem& p, cudaStream_t s);

// ------------------------------------------------------------------ Krylov
struct Report {  // seistomo::SolveReport (inc/krylov.hpp:19-40)
  int cycles = 0;
  std::vector<int> col_cycles;
  std::vector<double> rel_residual;
  std::vector<char> converged;
  std::vector<double> history;
  double wall_s = 0;
  int qr_factorizations = 0;
  int64_t block_gram_products = 0;
  bool all_converged() const {
    for (char c : converged)
      if (!c) return false;
    return !converged.empty();
  }
};

// Matrix-free block operator on device blocks (BlockOperator, inc/krylov.hpp:13-17).
template <class T>
struct DevOp {
  using V = cplx_t<T>;
  int64_t n = 0;
  std::function<void(const V* in, V* out, int k, cudaStream_t)> apply;
  std::function<void(const V* in, V* out, int k, cudaStream_t)> prec;  // optional
  // optional fused true residual r = b - A x (bitwise apply + axpby)
  std::function<void(const V* x, const V* b, V* r, int k, cudaStream_t)> resid;
  // optional complex64 preconditioner output (a c64 cycle's result before
  // its exact widening) + the operator applied to such a block: FGMRES then
  // keeps its Z blocks in complex64 -- the same values at half the bytes
  std::function<void(const V* in, float2* out, int k, cudaStream_t)> prec_lo;
  std::function<void(const float2* in, V* out, int k, cudaStream_t)> apply_lo;
  // optional: block widths apply_lo supports (unset: all)
  std::function<bool(int k)> lo_ok;
  // optional apply_lo fused with the Arnoldi Gram: W = A Z and the partial
  // Grams of [X_0..X_{nb-2}, W]^H W (k = 8); returns the slots written
  std::function<int(const float2* Z, V* W, const BlockTab<T>& X, int nb, V* partials, int max_slots, cudaStream_t)>
      apply_lo_gram;
};

// Device block algebra shared by the Krylov methods.
template <class T>
class BlockAlgebra {
 public:
  using V = cplx_t<T>;
  // sl: rows of level 0 split over slab parts (nullptr: one stream)
  void ensure(int64_t n, int k, int max_blocks, const Slabs* sl = nullptr);
  // G_i = X_i^H Y for nb blocks, result on device (nb k^2, row-major tiles)
  void gram(const BlockTab<T>& tab, int nb, const V* Y, V* out, cudaStream_t s);
  // W = A Z with the Gram [X_0..X_{nb-2}, W]^H W into out (op.apply_lo_gram)
  void gram_apply(const DevOp<T>& op, const BlockTab<T>& tab, int nb, const float2* Z, V* W, V* out,
                  cudaStream_t s);
  // per-column 2-norms to host
  void col_norms(const V* X, std::vector<double>& out, cudaStream_t s);
  // CholQR2 thin QR of W in place (inc/block.hpp:104-137 semantics):
  // enqueues the work; R (k x k, row-major) and the rank-deficient flag are
  // available after sync in host_R()/host_deficient().
  void thin_qr_enqueue(V* W, cudaStream_t s);
  void thin_qr_finish(std::vector<cplx>& R, bool& deficient);  // after stream sync
  // G = W^H W on device (kept for thin_qr_from) and the column 2-norms
  // sqrt(diag G) to host: one pass over W instead of col_norms + a QR Gram
  void self_gram_norms(const V* W, std::vector<double>& out, cudaStream_t s);
  // thin QR of src into dst (dst != src) from the Gram G = src^H src
  // already on device: one CholQR pass when every Cholesky pivot keeps eta2
  // of its column's norm^2 (then Q^H Q = I to ~eps/eta2), else CholQR2, or
  // the column Gram-Schmidt for near rank deficiency; R / deficient as
  // thin_qr_finish. Synchronises the stream.
  void thin_qr_from(const V* src, V* dst, std::vector<cplx>& R, bool& deficient, double eta2, cudaStream_t s);

  int64_t n = 0;
  int k = 0;
  int nslots = 0;
  DevBuf<V> partials, tmp_blk, G, R1, R1i, R2, R2i;
  DevBuf<T> rpart, rnorm;
  DevBuf<int> flags;
  DevBuf<V> dbuf;         // column Gram-Schmidt dot products
  bool mgs_used = false;  // last thin_qr took the column Gram-Schmidt path
  PinnedBuf<T> h_norm;
  PinnedBuf<V> h_R;     // [R1 | R2 | G]
  PinnedBuf<int> h_flags;

  // ---- slab mode: row-local work runs per part on the part's rows; the
  // k x k partials of all parts are summed on part 0 (stream s) in a fixed
  // slot order
  const Slabs* sl = nullptr;
  std::vector<int> pslots;  // partial slots per part
  template <class F>
  void each(cudaStream_t s, F&& f) const {
    if (!sl) {
      f(0, int64_t(0), n, s);
      return;
    }
    sl->each(0, [&](int p, int64_t r0, int64_t nr, cudaStream_t st) { f(p, r0, nr, st); });
  }
  void join() const {
    if (sl) sl->join();
  }
  void fork() const {
    if (sl) sl->fork();
  }
  static BlockTab<T> shift(const BlockTab<T>& t, int nb, int64_t off) {
    BlockTab<T> r{};
    for (int i = 0; i < nb; ++i) r.p[i] = t.p[i] ? t.p[i] + off : nullptr;
    return r;
  }
  // row-split block update: Yout = (Yin ? Yin : 0) + sign * sum_i X_i H_i
  void update(int nb, const BlockTab<T>& X, const V* H, const V* Yin, V* Yout, T sign, cudaStream_t s);

 private:
  const Slabs* sl_alloc_ = nullptr;
};

template <class T>
class Fgmres {
 public:
  using V = cplx_t<T>;
  // block_fgmres (src/krylov.cpp:178-280): X = 0 start, flexible, restart m.
  Report solve(const DevOp<T>& op, int k, const V* B, V* X, int restart, double tol,
               int max_cycles, cudaStream_t s);
  // slab mode: B, X and the basis span the parts; s must be part 0's stream
  void set_slabs(const Slabs* sl) {
    if (sl != sl_) {  // re-laid out at the next solve: free the old basis now
      n_ = 0;
      Vb_.clear();
      Zb_.clear();
      Zlo_.clear();
      R_.release();
      Qs_.release();
      alg_.tmp_blk.release();
    }
    sl_ = sl;
  }

 private:
  void ensure(int64_t n, int k, int restart, bool lo);
  const Slabs* sl_ = nullptr;
  int64_t n_ = 0;
  int k_ = 0, m_ = 0;
  std::vector<DevBuf<V>> Vb_, Zb_;
  std::vector<DevBuf<float2>> Zlo_;  // complex64 Z blocks (DevOp::prec_lo)
  bool lo_ = false;
  BlockTab<float> zlotab_{};
  DevBuf<V> R_;
  DevBuf<V> Qs_;  // spare block: the speculative one-pass Q of an Arnoldi step
  BlockTab<T> vtab_{}, ztab_{};
  // marks the D2H copies of a step's acceptance flag / H column, so the host
  // waits for them without draining the speculative work behind them
  struct Event {
    cudaEvent_t e = nullptr;
    ~Event() {
      if (e) cudaEventDestroy(e);
    }
    cudaEvent_t get() {
      if (!e) HZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      return e;
    }
  } ev_;
  DevBuf<V> hcol1_, hcol2_, ydev_, ccoef_;
  // Gram of the next step computed with its matvec (DevOp::apply_lo_gram)
  DevBuf<V> hcol_next_;
  bool gram_next_ = false, ga_ = false;
  // Pythagorean one-pass orthogonalisation with CGS2 fallback (HZ_ORTHO=cgs2
  // forces the two-pass path everywhere)
  bool pip_ = true;
  // accept the one-pass block when ||W'_c||^2 >= eta2 ||W_c||^2 for every
  // column: the Pythagorean S then has relative error <= eps/eta2 and Q is
  // orthogonal to V to eps/sqrt(eta2) (1e-4 -> ~1e-14), far below what a
  // 1e-6 solve can see; below it the step falls back to CGS2 + CholQR2
  double pip_eta2_ = 1e-4;

 public:
  int64_t pip_accepted_ = 0, pip_rejected_ = 0;

 private:
  PinnedBuf<V> h_hcol_, h_y_;
  BlockAlgebra<T> alg_;
};

// block_bicgstab (src/krylov.cpp:60-176), f64.
class Bicgstab {
 public:
  using V = double2;
  Report solve(const DevOp<double>& op, int k, const V* B, V* X, double tol, int max_cycles,
               cudaStream_t s);

 private:
  void ensure(int64_t n, int k);
  int64_t n_ = 0;
  int k_ = 0;
  DevBuf<V> R_, Rt_, P_, ZP_, V_, S_, ZS_, T_, PmV_, cdev_, fpart_, fsum_;
  PinnedBuf<V> h_small_;
  BlockAlgebra<double> alg_;
};

}  // namespace hz
