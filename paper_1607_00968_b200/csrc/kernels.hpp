// Launch wrappers for the sm_100a kernels (declarations). Every wrapper
// enqueues on the given stream and never synchronises.
#pragma once

#include "common.cuh"

namespace hz {

// One level operator as the kernels see it.
//  * kind == kFine: the 5-point (2D) / 7-point (3D) fine operator with a
//    per-node complex centre and constant off-diagonals w[a] = 1/h_a^2
//    (HelmholtzProblem, src/helmholtz.cpp:45-122).
//  * kind == kStencil: a Galerkin coarse operator stored as S = 3^ndim
//    complex coefficient planes coef[s][node], s = (dz+1)*9 + (dy+1)*3 + (dx+1)
//    -- ascending s is ascending CSR column, so sums run in the reference's
//    Csr::mul_block order (inc/csr.hpp:40-54).
//  * kind == kFine27: the compact 27-point fine operator (config 4) with its
//    couplings computed on the fly, lap[q] + mu[q] (M_i + M_j)/2 from the
//    per-node mass M (`center`, gamma already shifted) and the 8 weights
//    w27 = {lap[0..3], mu[0..3]} -- 1 complex per node instead of 27 planes.
enum OpKind : int { kFine = 0, kStencil = 1, kFine27 = 2 };

template <class T>
struct LevelOp {
  using V = cplx_t<T>;
  int kind = kFine;
  int ndim = 2;
  LevelGeom g;                 // k is set per launch
  const V* center = nullptr;   // kFine: diagonal (centre) per node
  const V* coef = nullptr;     // kStencil: [S][nodes]
  const V* inv_diag = nullptr; // Jacobi D^{-1} per node
  const V* cd = nullptr;       // optional: (centre, D^{-1}) per node (kFine), (9 planes, D^{-1}) per node (2D kStencil)
  T w[3] = {0, 0, 0};          // kFine off-diagonal weights (0 on flat axes)
  T w27[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // kFine27: lap[0..3], mu[0..3]
  int level = 0;               // multigrid level (profiling names only)
};

// out = A u                                    (K1: apply_block)
template <class T>
void launch_apply(const LevelOp<T>& op, const cplx_t<T>* u, cplx_t<T>* out, cudaStream_t s);
// complex128 fine apply of a complex64 block (widened on load; the values
// and arithmetic of launch_apply<double> on the widened block)
void launch_apply_lo(const LevelOp<double>& op, const float2* u, double2* out, cudaStream_t s);
// r = b - A x                                  (residual, src/multigrid.cpp:173-175)
template <class T>
void launch_residual(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* r,
                     cudaStream_t s);
// r = b - A x for the fine operator with A x in apply_block order: the
// fused, bitwise-identical form of apply + axpby(-1, r, 1, b) (the true
// residual of block_fgmres / finalize, src/krylov.cpp:35-37,270-271)
template <class T>
void launch_apply_residual(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* r,
                           cudaStream_t s);
// xout = x + (wj D^{-1}) (b - A x)             (K2: relax, src/multigrid.cpp:119-136)
template <class T>
void launch_jacobi(const LevelOp<T>& op, T wj, const cplx_t<T>* x, const cplx_t<T>* b,
                   cplx_t<T>* xout, cudaStream_t s);
// xout = (wj D^{-1}) b  -- the first sweep from x = 0, bitwise the same as
// b - A*0 = b. In may be a wider type (c128 -> c64 cast).
template <class T, class In>
void launch_jacobi_zero(const LevelOp<T>& op, T wj, const In* b, cplx_t<T>* xout, cudaStream_t s);
// bc = P^T r   (R unscaled, src/multigrid.cpp:87-88,176-178)
template <class T>
void launch_restrict(const LevelGeom& gf, const LevelGeom& gc, int ndim, const cplx_t<T>* r,
                     cplx_t<T>* bc, cudaStream_t s);
// x += P ec    (bi/trilinear, src/multigrid.cpp:27-69,195-197)
template <class T>
void launch_prolong_correct(const LevelGeom& gf, const LevelGeom& gc, int ndim,
                            const cplx_t<T>* ec, cplx_t<T>* x, cudaStream_t s);
// Galerkin A_c = P^T A_f P as 3^ndim stencil planes, in the reference's
// sparse triple-product summation order (src/multigrid.cpp:85-93,
// inc/csr.hpp:130-160). Always f64.
void launch_galerkin(const LevelOp<double>& fine, const LevelGeom& gc, double2* coef_c,
                     cudaStream_t s);

// complex64 preconditioner of a complex128 block, finest level: the
// zero-start sweep fused with the c128 -> c64 cast of the right-hand side
// (b32 is written for the rest of the cycle; k % 4 == 0) ...
bool cast_zero_ok(const LevelOp<float>& op);
void launch_jacobi_zero_cast(const LevelOp<float>& op, float wj, const double2* b64, float2* b32, float2* x1,
                             cudaStream_t s);
// ... and the last post-smoothing sweep writing the c128 result directly
// (kFine, k % 4 == 0)
bool fused_fine_ok(const LevelOp<float>& op);
void launch_jacobi_out64(const LevelOp<float>& op, float wj, const float2* x, const float2* b, double2* out,
                         cudaStream_t s);

// Fused finest-level V(2,2) smoothing on a 2D grid (fused.cu): the zero-start
// pre-smoothing sweeps + residual + restriction in one streaming kernel
// (x2 = the pre-smoothed iterate, rc = P^T r), and the prolongated correction
// + both post-smoothing sweeps in another (out = x after the visit, cast to
// Out). Bitwise equal to the unfused sequence. HZ_FUSED_VCYCLE=0 disables.
template <class T>
bool fused_fine_vcycle_ok(const LevelOp<T>& op);
template <class T, class In>
void launch_fused_pre(const LevelOp<T>& op, const LevelGeom& gc, T wj, const In* b, cplx_t<T>* x2,
                      cplx_t<T>* rc, cudaStream_t s);
template <class T, class In, class Out>
void launch_fused_post(const LevelOp<T>& op, const LevelGeom& gc, T wj, const cplx_t<T>* x2,
                       const cplx_t<T>* ec, const In* b, Out* out, cudaStream_t s);

// Plane-streaming 3D fine-level kernels for 8-column blocks (stream3d.cu):
// 7-point (bitwise equal to the element kernels) and compact 27-point
// (separable class sums), bulk-copy tile staging with an mbarrier ring.
// mode 0 apply, 1 residual, 2 damped Jacobi (Out may be double2 for the
// complex64 level: the cycle's last sweep), 3 residual in apply_block order.
// Return false when they do not apply (HZ_STREAM3D=0, other k, slab ranges).
template <class T>
bool stream3d_ok(const LevelOp<T>& op);
template <class T, class Out>
bool launch_stream3d(const LevelOp<T>& op, int mode, T wj, const cplx_t<T>* x, const cplx_t<T>* b, Out* out,
                     cudaStream_t s);
// complex128 fine operator applied to a complex64 block (widened on load)
bool launch_stream3d_lo(const LevelOp<double>& op, const float2* x, double2* out, cudaStream_t s);

// Compact 27-point operator (3D, uniform spacing h): planes[s][i],
// s = (dz+1)*9 + (dy+1)*3 + (dx+1). Laplacian weights lap[q] for neighbour
// class q = |dx|+|dy|+|dz| (lap[0] is the centre), mass weights mu[q]; the
// coupling of i and j is lap[q] + mu[q] (M_i + M_j)/2, the centre
// lap[0] + mu[0] M_i, with M = mass - i shift_w2 m (gamma + shift omega);
// neighbours outside the grid get 0 (Dirichlet truncation).
void launch_build27(const LevelGeom& g, const double* lap, const double* mu, const double2* mass, const double* m,
                    double shift_w2, double2* planes, cudaStream_t s);
// Ms[i] = mass[i] - i shift_w2 m[i] (the shifted per-node mass of kFine27)
void launch_shift_mass(int64_t n, const double2* mass, const double* m, double shift_w2, double2* ms, cudaStream_t s);
// inv[i] = 1 / (lap0 + mu0 Ms[i]) (Jacobi D^-1 of a kFine27 level)
void launch_inv_centre27(int64_t n, double lap0, double mu0, const double2* ms, double2* inv, cudaStream_t s);
// inv[i] = 1 / planes[centre][i] (Jacobi D^-1 of a stencil level)
void launch_inv_plane(int64_t n, const double2* centre, double2* inv, cudaStream_t s);

// complex64 2D Galerkin level, k = 8, with bulk-copy row staging (fused.cu):
// MODE 0 apply, 1 residual, 2 damped Jacobi, bitwise equal to the stencil_v4
// kernels; returns false when it does not apply (then use dispatch_level)
bool launch_stencil9_k8(const LevelOp<float>& op, int mode, float wj, const float2* x, const float2* b, float2* out,
                        cudaStream_t s);

// two damped-Jacobi sweeps of a complex64 2D Galerkin level (k = 8) in one
// launch, the intermediate iterate in shared memory (fused.cu); x == nullptr:
// the sweeps start from x = 0. out must not alias x. Bitwise equal to two
// launch_jacobi calls (or launch_jacobi_zero + launch_jacobi); false when it
// does not apply (small levels, other k / layouts, HZ_S9_PAIR=0)
bool launch_stencil9_pair_k8(const LevelOp<float>& op, float wj, const float2* x, const float2* b, float2* out,
                             cudaStream_t s);

// zero-start pre-smoothing visit of a complex64 2D Galerkin level (k = 8) in
// one launch: both sweeps from x = 0, the residual and its restriction
// (x2 = the pre-smoothed iterate, rc = P^T (b - A x2)); bitwise equal to
// jacobi_zero + jacobi + residual + restrict. False when it does not apply.
bool launch_stencil9_pre_k8(const LevelOp<float>& op, const LevelGeom& gc, float wj, const float2* b, float2* x2,
                            float2* rc, cudaStream_t s);

// plane-streaming kernel of a complex64 3D Galerkin level, k = 8
// (galerkin3d.cu): mode 0 apply, 1 residual, 2 damped Jacobi, bitwise equal
// to the stencil_v4 kernels. op.cd = the level's three record groups
// [3][nodes][10] (launch_galerkin3d_records), kept for levels of at least
// galerkin3d_min_nodes() nodes. False when it does not apply (HZ_G3=0, ...).
int64_t galerkin3d_min_nodes();
void launch_galerkin3d_records(int64_t nodes, const float2* coef, const float2* inv_diag, float2* rec,
                               cudaStream_t s);
bool launch_galerkin3d(const LevelOp<float>& op, int mode, float wj, const float2* x, const float2* b, float2* out,
                       cudaStream_t s);

// elementwise casts / copies
template <class Dst, class Src>
void launch_cast(int64_t count, const Src* in, Dst* out, cudaStream_t s);

// ---- coarsest level (K5)
// Columns of A^{-1} from banded LU factors (gbtrf storage as in
// BandedLU, inc/dense.hpp:179-216): one warp per column, written as
// ainvT[c][i] = (A^{-1})[i][c].
void launch_banded_inverse(int64_t n, int64_t kl, int64_t ku, int64_t ld, const double2* ab,
                           const int64_t* piv, double2* ainvT, cudaStream_t s);
// Row stride of ainvT (even, so complex64 rows stay 16-byte aligned).
__host__ __device__ inline int64_t inv_ld(int64_t n) { return n + (n & 1); }
// Split-K factor of the tiled coarse solve (0: k not tiled). The tiled path
// needs `part` with coarse_split(n, k) * n * k entries when the split is > 1.
int coarse_split(int64_t n, int k);
// X[i][:] = sum_l ainvT[l][i] * B[l][:]   (dense coarse solve, all k columns)
template <class T>
void launch_coarse_solve(int64_t n, int k, const cplx_t<T>* ainvT, const cplx_t<T>* b,
                         cplx_t<T>* x, cplx_t<T>* part, cudaStream_t s);
// general form: x = (c_in ? c_in : 0) + sign * (A b), A given transposed with
// row stride ld (x may alias c_in)
template <class T>
void launch_coarse_gemm(int64_t n, int k, const cplx_t<T>* ainvT, int64_t ld, const cplx_t<T>* b, cplx_t<T>* x,
                        const cplx_t<T>* c_in, T sign, cplx_t<T>* part, cudaStream_t s);

// Block-tridiagonal (plane) direct solver of a 3D coarsest Galerkin operator
// (coarse_bt.cu): ET/FT = [n2][m][inv_ld(m)] plane blocks E_j, F_j: row-major
// when bt_rowmajor(m) (the row-owner kernel), else transposed (coarse GEMM);
// m = n0*n1; g.k unused. Solve scratch: r (m*k), part (split partials).
// planes up to 2 x 148 x 8 nodes (HZ_BT_ROWS_MAX overrides) use the row-major
// layout; read when the factor is built and at every solve
bool bt_rowmajor(int64_t m);
void bt_factor(const LevelGeom& g, const double2* coef, double2* ET, double2* FT, cudaStream_t s);

// sweep-axis permutation of the plane solver: perm[a] = old axis of new axis
// a, the longest axis last (HZ_BT_PERMUTE=0: identity); the operator planes
// and the right-hand side / solution blocks are re-indexed onto that grid
void bt_sweep_perm(const int64_t* dims, int* perm);
LevelGeom bt_permuted_geom(const LevelGeom& g, const int* perm);
void bt_permute_coef(const LevelGeom& g, const int* perm, const double2* coef, double2* coefT, cudaStream_t s);
template <class T>
void bt_permute_vec(const LevelGeom& g, const int* perm, int k, bool inverse, const cplx_t<T>* src, cplx_t<T>* dst,
                    cudaStream_t s);

// second stream + fork / join events of the two-sided (twisted) sweep; one
// per concurrently solving hierarchy view
struct BtAux {
  cudaStream_t s2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  BtAux() = default;
  BtAux(const BtAux&) = delete;
  BtAux& operator=(const BtAux&) = delete;
  ~BtAux();
  void ensure();
};
// planes [0, mid) are eliminated top-down, (mid, n2) bottom-up (HZ_BT_TWISTED=0: mid = n2 - 1)
int bt_mid(int np);
// scratch: r = 2 m k entries, part = 2 coarse_split(m, k) m k entries
template <class T>
void bt_solve(const LevelGeom& g, const cplx_t<T>* coef, const cplx_t<T>* ET, const cplx_t<T>* FT, int k,
              const cplx_t<T>* b, cplx_t<T>* x, cplx_t<T>* r, cplx_t<T>* part, const BtAux& aux, cudaStream_t s);

// ---- block (tall-skinny) kernels, node-major [n][k] blocks (inc/block.hpp)
// Tables of block pointers travel by value in the kernel parameters (no
// device-side pointer arrays, no host round trip to build them).
constexpr int kMaxBlocks = 48;
template <class T>
struct BlockTab {
  const cplx_t<T>* p[kMaxBlocks];
};
// W = A Z (fine complex128 operator, Z complex64, k = 8) fused with the
// partial Grams of [X_0..X_{nb-2}, W]^H W (gram8 slot layout); returns the
// number of partial slots written (<= max_slots)
int launch_gram8_apply(const LevelOp<double>& op, int nb, const BlockTab<double>& X, const float2* Z, double2* W,
                       double2* partials, int max_slots, cudaStream_t s);
// Y += sum_i Z_i H_i with complex64 blocks Z_i widened on load (FGMRES's
// restart update X += Z Y over complex64 Z blocks)
void launch_update_lo(int64_t n, int k, int nb, const BlockTab<float>& Z, const double2* H, double2* Y,
                      cudaStream_t s);
// Stage 1 of a deterministic two-stage reduction: per-CTA partial Grams
// G_i = X_i^H Y for nb blocks X_i against one Y (k x k each).
// Returns the number of partial slices written to `partials`
// (partials must hold gram_partial_slots(n) * nb * k * k entries).
int gram_partial_slots(int64_t n, int k);
template <class T>
int launch_multi_gram(int64_t n, int k, int nb, const BlockTab<T>& X, const cplx_t<T>* Y,
                       cplx_t<T>* partials, int nslots, cudaStream_t s);
// Yout = (Yin ? Yin : 0) + sign * sum_i X_i H_i  (H_i k x k row-major, on
// device). Yout may alias Yin but not any X_i.
template <class T>
void launch_multi_update(int64_t n, int k, int nb, const BlockTab<T>& X, const cplx_t<T>* H,
                         const cplx_t<T>* Yin, cplx_t<T>* Yout, T sign, cudaStream_t s);
// sum over slots: out[e] = sum_s partials[s][e], fixed slot order
template <class T>
void launch_reduce_partials(int64_t count, int nslots, const cplx_t<T>* partials, cplx_t<T>* out,
                            cudaStream_t s);
// per-column sums of |x|^2 (partials per slot, then reduce)
template <class T>
void launch_colnorm2_partial(int64_t n, int k, const cplx_t<T>* X, T* partials, int nslots,
                             cudaStream_t s);
template <class T>
void launch_reduce_real(int64_t count, int nslots, const T* partials, T* out, cudaStream_t s);
// Y = a*Y + b*X (complex scalars, host values)
template <class T>
void launch_axpby(int64_t count, cplx_t<T> a, cplx_t<T>* Y, cplx_t<T> b, const cplx_t<T>* X,
                  cudaStream_t s);
// X += omega ZS ; R = S - omega T   (block BiCGSTAB update, src/krylov.cpp:140-145)
template <class T>
void launch_bicgstab_update(int64_t count, cplx_t<T> omega, cplx_t<T>* X, const cplx_t<T>* ZS,
                            cplx_t<T>* R, const cplx_t<T>* S, const cplx_t<T>* Tt, cudaStream_t s);
// partial sums of conj(T).S and conj(T).T over all entries (Frobenius)
template <class T>
void launch_frob2_partial(int64_t count, const cplx_t<T>* Tt, const cplx_t<T>* S,
                          cplx_t<T>* partials, int nslots, cudaStream_t s);

// upper-triangular Cholesky factor of a k x k Hermitian Gram on device:
// R (k x k), Rinv, and flag[0] = first failing column + 1 (0 = ok). A failing
// pivot marks the column collapsed exactly as thin_qr does
// (inc/block.hpp:126-131): zero row in R, zero column in Q = W Rinv.
template <class T>
void launch_small_cholesky(int k, const cplx_t<T>* G, cplx_t<T>* R, cplx_t<T>* Rinv, int* flag,
                           T rel_tol, cudaStream_t s);

// Column-by-column Gram-Schmidt with re-orthogonalisation, the reference's
// thin_qr (inc/block.hpp:104-137), fully on the device: W <- Q, R (k x k),
// flag = 1 if a column collapsed (zeroed, R_jj = 0). dbuf >= 192 entries,
// partials >= max_slots * 64 entries. Used when CholQR cannot resolve the
// block (near rank deficiency).
template <class T>
void launch_mgs_qr(int64_t n, int k, cplx_t<T>* W, cplx_t<T>* R, cplx_t<T>* dbuf, cplx_t<T>* partials,
                   int max_slots, int* flag, cudaStream_t s);

// Pythagorean block CholQR of one Arnoldi step from Hc = [H_0..H_{nb-1}, G]
// (one Gram pass [V_0..V_{nb-1}, W]^H W): R, R^{-1} and the block-update
// coefficients C (nb + 1 tiles) of Q = (W - V H) R^{-1}; flag 0 accepted,
// 1 rejected (severe cancellation: caller falls back to CGS2 + CholQR2).
template <class T>
void launch_pip_factor(int k, int nb, const cplx_t<T>* Hc, cplx_t<T>* R, cplx_t<T>* Rinv,
                       cplx_t<T>* C, int* flag, T eta2, cudaStream_t s);

// FP64 tensor-pipe (DMMA) peak of the current device, TFLOP/s (diagnostic)
double measure_dmma_tflops();

// sensitivity: g[i] (+)= sum_s Re(-omega^2 gf[i] u[i][s] lam[i][s])  (K13)
void launch_sensitivity(int64_t n, int k, double w2, const double2* gf, const double2* U,
                        const double2* L, double* g, int accumulate, cudaStream_t s);

}  // namespace hz
