// Tall-skinny block kernels for the block Krylov methods (K6-K10) over
// node-major [n][k] blocks: Gram products X^H Y, block updates Y -= X H,
// column norms, Frobenius inner products and the block axpby
// (inc/block.hpp:42-98, src/krylov.cpp:129-145).
//
// Reductions are deterministic two-stage: each CTA ("slot") writes a
// private partial, and a second kernel sums the slots in fixed order -- no
// floating-point atomics, so runs are bitwise reproducible.
#include "kernels.hpp"
#include "profile.hpp"
#include "block_tiled.cuh"
#include "block_dmma.cuh"
#include "block_k8.cuh"
#include "devbuf.hpp"

#include <cstdlib>
#include <type_traits>

namespace hz {

namespace {

constexpr int kBlk = 256;

int slots_for(int64_t n) {
  // ~4 CTAs per SM, at least 64 rows each
  int64_t s = (n + 63) / 64;
  if (s > 4 * kNumSMs) s = 4 * kNumSMs;
  return int(s < 1 ? 1 : s);
}


// CTA (i = blockIdx.x, slot = blockIdx.y) computes the slot's partial of
// X_i^H Y over its row range. Thread t owns a TP x TQ tile of (p, q) pairs;
// when k*k/(TP*TQ) < 256 the CTA splits into row groups reduced in smem.
template <class T, int TP, int TQ>
__global__ void __launch_bounds__(kBlk)
multi_gram_kernel(int64_t n, int k, const BlockTab<T> X,
                  const cplx_t<T>* __restrict__ Y, cplx_t<T>* __restrict__ partials, int nslots) {
  using V = cplx_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* red = reinterpret_cast<V*>(smem_raw);
  const int i = blockIdx.x, slot = blockIdx.y, nb = gridDim.x;
  const V* __restrict__ Xi = X.p[i];
  const int tp_count = (k + TP - 1) / TP, tq_count = (k + TQ - 1) / TQ;
  const int tiles = tp_count * tq_count;
  const int groups = max(1, kBlk / tiles);
  const int tid = threadIdx.x;
  const int g = tid / tiles, tile = tid - g * tiles;
  const bool active = g < groups && tid < groups * tiles;
  const int p0 = (tile / tq_count) * TP, q0 = (tile % tq_count) * TQ;
  V acc[TP][TQ];
#pragma unroll
  for (int a = 0; a < TP; ++a)
#pragma unroll
    for (int b = 0; b < TQ; ++b) acc[a][b] = czero<V>();
  const int64_t rows_per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(slot) * rows_per, r1 = min(n, r0 + rows_per);
  if (active) {
    for (int64_t r = r0 + g; r < r1; r += groups) {
      const V* xr = Xi + r * k;
      const V* yr = Y + r * k;
      V xv[TP], yv[TQ];
#pragma unroll
      for (int a = 0; a < TP; ++a) xv[a] = (p0 + a < k) ? __ldg(&xr[p0 + a]) : czero<V>();
#pragma unroll
      for (int b = 0; b < TQ; ++b) yv[b] = (q0 + b < k) ? __ldg(&yr[q0 + b]) : czero<V>();
#pragma unroll
      for (int a = 0; a < TP; ++a)
#pragma unroll
        for (int b = 0; b < TQ; ++b) acc[a][b] = cfmac(xv[a], yv[b], acc[a][b]);
    }
  }
  // reduce row groups through smem in fixed group order
  V* out = partials + (int64_t(slot) * nb + i) * k * k;
  if (groups == 1) {
    if (active) {
#pragma unroll
      for (int a = 0; a < TP; ++a)
#pragma unroll
        for (int b = 0; b < TQ; ++b)
          if (p0 + a < k && q0 + b < k) out[(p0 + a) * k + q0 + b] = acc[a][b];
    }
    return;
  }
  // smem layout [groups][k*k]
  if (active) {
#pragma unroll
    for (int a = 0; a < TP; ++a)
#pragma unroll
      for (int b = 0; b < TQ; ++b)
        if (p0 + a < k && q0 + b < k) red[g * k * k + (p0 + a) * k + q0 + b] = acc[a][b];
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += kBlk) {
    V s = red[e];
    for (int gg = 1; gg < groups; ++gg) s = cadd(s, red[gg * k * k + e]);
    out[e] = s;
  }
}

// out = (Yin ? Yin : 0) + sign * sum_i X_i H_i ; H_i row-major k x k.
// Thread per (row, q) element; H_i staged in smem one block at a time.
template <class T>
__global__ void __launch_bounds__(kBlk)
multi_update_kernel(int64_t n, int k, int nb, const BlockTab<T> X,
                    const cplx_t<T>* __restrict__ H, const cplx_t<T>* Yin, cplx_t<T>* Yout, T sign) {
  using V = cplx_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* Hs = reinterpret_cast<V*>(smem_raw);  // [k][k]
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  const bool valid = e < n * k;
  const int64_t r = valid ? e / k : 0;
  const int q = valid ? int(e - r * k) : 0;
  V acc = czero<V>();
  for (int i = 0; i < nb; ++i) {
    __syncthreads();
    for (int t = threadIdx.x; t < k * k; t += kBlk) Hs[t] = H[int64_t(i) * k * k + t];
    __syncthreads();
    if (valid) {
      const V* xr = X.p[i] + r * k;
      for (int p = 0; p < k; ++p) acc = cfma(__ldg(&xr[p]), Hs[p * k + q], acc);
    }
  }
  if (valid) {
    V y = Yin ? Yin[e] : czero<V>();
    y.x += sign * acc.x;
    y.y += sign * acc.y;
    Yout[e] = y;
  }
}

template <class T>
__global__ void __launch_bounds__(kBlk)
reduce_partials_kernel(int64_t count, int nslots, const cplx_t<T>* __restrict__ partials,
                       cplx_t<T>* __restrict__ out) {
  // CTA = 32 consecutive outputs x 8 slot groups; each group sums a strided
  // subset of the slots, then the 8 group sums are added in fixed order.
  using V = cplx_t<T>;
  __shared__ V red[8][32];
  const int o = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int64_t e = int64_t(blockIdx.x) * 32 + o;
  V s = czero<V>();
  if (e < count)
    for (int t = sg; t < nslots; t += 8) s = cadd(s, partials[int64_t(t) * count + e]);
  red[sg][o] = s;
  __syncthreads();
  if (sg == 0 && e < count) {
    V r = red[0][o];
#pragma unroll
    for (int gg = 1; gg < 8; ++gg) r = cadd(r, red[gg][o]);
    out[e] = r;
  }
}

template <class T>
__global__ void __launch_bounds__(kBlk)
reduce_real_kernel(int64_t count, int nslots, const T* __restrict__ partials, T* __restrict__ out) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= count) return;
  T s = partials[e];
  for (int t = 1; t < nslots; ++t) s += partials[int64_t(t) * count + e];
  out[e] = s;
}

// per-slot per-column sum |x|^2; thread handles column q = tid % k on rows
// of its row group.
template <class T>
__global__ void __launch_bounds__(kBlk)
colnorm2_kernel(int64_t n, int k, const cplx_t<T>* __restrict__ X, T* __restrict__ partials,
                int nslots) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* red = reinterpret_cast<T*>(smem_raw);
  const int slot = blockIdx.x;
  const int groups = max(1, kBlk / k);
  const int tid = threadIdx.x, g = tid / k, q = tid - g * k;
  const bool active = g < groups;
  const int64_t rows_per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(slot) * rows_per, r1 = min(n, r0 + rows_per);
  T acc[4] = {0, 0, 0, 0};  // k > 256 handled by striding q
  const int qstride = kBlk;
  if (k <= kBlk) {
    if (active)
      for (int64_t r = r0 + g; r < r1; r += groups) acc[0] += cabs2(__ldg(&X[r * k + q]));
    red[tid] = active ? acc[0] : T(0);
    __syncthreads();
    if (tid < k) {
      T s = red[tid];
      for (int gg = 1; gg < groups; ++gg) s += red[gg * k + tid];
      partials[int64_t(slot) * k + tid] = s;
    }
  } else {
    for (int qq = tid; qq < k; qq += qstride) {
      T s = 0;
      for (int64_t r = r0; r < r1; ++r) s += cabs2(X[r * k + qq]);
      partials[int64_t(slot) * k + qq] = s;
    }
  }
}

template <class T>
__global__ void __launch_bounds__(kBlk)
axpby_kernel(int64_t count, cplx_t<T> a, cplx_t<T>* Y, cplx_t<T> b, const cplx_t<T>* X) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= count) return;
  Y[e] = cadd(cmul(a, Y[e]), cmul(b, X[e]));
}

template <class T>
__global__ void __launch_bounds__(kBlk)
bicgstab_update_kernel(int64_t count, cplx_t<T> omega, cplx_t<T>* __restrict__ X,
                       const cplx_t<T>* __restrict__ ZS, cplx_t<T>* __restrict__ R,
                       const cplx_t<T>* __restrict__ S, const cplx_t<T>* __restrict__ Tt) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= count) return;
  X[e] = cadd(X[e], cmul(omega, ZS[e]));
  R[e] = csub(S[e], cmul(omega, Tt[e]));
}

// partial[slot] = (sum conj(T) S, sum conj(T) T)
template <class T>
__global__ void __launch_bounds__(kBlk)
frob2_kernel(int64_t count, const cplx_t<T>* __restrict__ Tt, const cplx_t<T>* __restrict__ S,
             cplx_t<T>* __restrict__ partials, int nslots) {
  using V = cplx_t<T>;
  __shared__ V red_a[kBlk], red_b[kBlk];
  const int slot = blockIdx.x;
  const int64_t per = (count + nslots - 1) / nslots;
  const int64_t e0 = int64_t(slot) * per, e1 = min(count, e0 + per);
  V a = czero<V>(), b = czero<V>();
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kBlk) {
    const V t = Tt[e];
    a = cfmac(t, S[e], a);
    b.x += cabs2(t);
  }
  red_a[threadIdx.x] = a;
  red_b[threadIdx.x] = b;
  __syncthreads();
  for (int o = kBlk / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red_a[threadIdx.x] = cadd(red_a[threadIdx.x], red_a[threadIdx.x + o]);
      red_b[threadIdx.x] = cadd(red_b[threadIdx.x], red_b[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * slot] = red_a[0];
    partials[2 * slot + 1] = red_b[0];
  }
}

// ---- k x k factorisations on one CTA (k <= 64, up to 1024 threads).
// In-place right-looking Cholesky of the Hermitian A (upper triangle) in
// shared memory, A <- R (upper, real positive diagonal). Element (a, c) is
// owned by thread (a k + c) mod nt for the whole factorisation, so step j
// needs ONE barrier: every thread reads the pivot and row j, updates its own
// trailing elements in place, and the row-j owners publish the scaled row
// after the barrier. Pivot test: PIP -- stop at the first d_j < thr G_jj;
// else (CholQR) collapse the column (zero row of R) and go on. Returns the
// first failing column + 1 (0: none).
template <class T, bool PIP>
__device__ int chol_upper_smem(cplx_t<T>* A, int k, const cplx_t<T>* G, T thr) {
  using V = cplx_t<T>;
  const int tid = threadIdx.x, nt = blockDim.x;
  constexpr int MAXE = 4;  // owned elements per thread: k^2 <= 4 * nt
  int fail = 0;
  int ea[MAXE], ec[MAXE], ne = 0;
#pragma unroll
  for (int q = 0; q < MAXE; ++q) {
    const int e = tid + q * nt;
    if (e < k * k) {
      ea[q] = e / k;
      ec[q] = e - ea[q] * k;
      ne = q + 1;
    }
  }
  for (int j = 0; j < k; ++j) {
    const T d = A[j * k + j].x;
    const T g0 = G[j * k + j].x;
    const bool dead = PIP ? (!(d >= thr * g0) || !(d > T(0)))
                          : (!(d > thr * (g0 > T(0) ? g0 : T(1))) || !(d > T(0)));
    if (dead && fail == 0) fail = j + 1;
    if (PIP && dead) return fail;  // the same decision in every thread
    const T piv = dead ? T(0) : sqrt(d);
    const T inv = piv > T(0) ? T(1) / piv : T(0);
    V rowv[MAXE];
    int rowc[MAXE];
    int nrow = 0;
#pragma unroll
    for (int q = 0; q < MAXE; ++q) {
      if (q >= ne) break;
      const int a = ea[q], c = ec[q], e = a * k + c;
      if (a == j && c >= j) {
        rowv[nrow] = c == j ? mk(piv, T(0)) : cscale(inv, A[e]);
        rowc[nrow++] = c;
      } else if (a > j && c >= a) {
        const V ra = cscale(inv, A[j * k + a]), rc = cscale(inv, A[j * k + c]);
        A[e] = csub(A[e], cmulc(ra, rc));
      }
    }
    __syncthreads();
    for (int q = 0; q < nrow; ++q) A[j * k + rowc[q]] = rowv[q];
  }
  __syncthreads();
  return fail;
}

template <class V>
__device__ __forceinline__ V warp_allsum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Ri = R^{-1} for upper R in shared memory (k <= 64): one warp per column,
// column-oriented back substitution (x = e_c; for l = c..0: x_l /= d_l, then
// every lane i < l subtracts A[i][l] x_l) -- one shuffle per step, no
// reductions on the dependency chain. A column whose pivot is not positive
// (collapsed) is zero, as are rows with d_i <= 0.
template <class T>
__device__ void tri_inv_upper(const cplx_t<T>* A, cplx_t<T>* Ri, int k) {
  using V = cplx_t<T>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // reciprocal pivots of this lane's rows (0 for non-positive pivots)
  const T d0 = lane < k ? A[lane * k + lane].x : T(0);
  const T d1 = lane + 32 < k ? A[(lane + 32) * k + lane + 32].x : T(0);
  const T r0 = d0 > T(0) ? T(1) / d0 : T(0), r1 = d1 > T(0) ? T(1) / d1 : T(0);
  for (int c = warp; c < k; c += nw) {
    const bool live = A[c * k + c].x > T(0);
    V x0 = (lane == c && live) ? mk(T(1), T(0)) : czero<V>();
    V x1 = (lane + 32 == c && live) ? mk(T(1), T(0)) : czero<V>();
    for (int l = c; l >= 0 && live; --l) {
      // finalise x_l on its lane, then broadcast it
      if (lane == l) x0 = cscale(r0, x0);
      if (lane + 32 == l) x1 = cscale(r1, x1);
      const V src = l < 32 ? x0 : x1;
      V xl;
      xl.x = __shfl_sync(0xffffffffu, src.x, l & 31);
      xl.y = __shfl_sync(0xffffffffu, src.y, l & 31);
      if (lane < l) x0 = csub(x0, cmul(A[lane * k + l], xl));
      if (lane + 32 < l) x1 = csub(x1, cmul(A[(lane + 32) * k + l], xl));
    }
    if (lane < k) Ri[lane * k + c] = x0;
    if (lane + 32 < k) Ri[(lane + 32) * k + c] = x1;
  }
}

// Single-CTA Cholesky G = R^H R (upper R, real positive diagonal) and R^{-1}.
// flag = first column j whose pivot fails d_j > rel_tol^2 * G_jj (+1), else 0.
template <class T>
__global__ void __launch_bounds__(1024)
small_cholesky_kernel(int k, const cplx_t<T>* __restrict__ G, cplx_t<T>* __restrict__ R,
                      cplx_t<T>* __restrict__ Rinv, int* flag, T rel_tol) {
  using V = cplx_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* A = reinterpret_cast<V*>(smem_raw);  // [k][k]
  V* Ri = A + k * k;                      // [k][k]
  const int tid = threadIdx.x;
  for (int e = tid; e < k * k; e += blockDim.x) A[e] = G[e];
  __syncthreads();
  const int fl = chol_upper_smem<T, false>(A, k, G, rel_tol * rel_tol);
  tri_inv_upper<T>(A, Ri, k);
  __syncthreads();
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int a = e / k, c = e - a * k;
    R[e] = c >= a ? A[e] : czero<V>();
    Rinv[e] = Ri[e];
  }
  if (tid == 0) *flag = fl;
}

// ---- column-wise Gram-Schmidt with one re-orthogonalisation: the
// reference's thin_qr (inc/block.hpp:104-137) for blocks CholQR cannot
// resolve (near rank-deficient: a column collapsing below ~1e-5 of its
// norm). One column at a time, entirely on the device:
//   d1 = W[:, :j+1]^H w_j (self entry = norm0^2); w_j -= W[:, :j] d1[:j]
//   d2 = ...;                                     w_j -= W[:, :j] d2[:j]
//   d3 = ... (self entry = norm^2); collapse if norm <= 1e-12 norm0.
template <class T>
__global__ void __launch_bounds__(256)
col_dots_kernel(int64_t n, int k, const cplx_t<T>* __restrict__ W, int j, cplx_t<T>* __restrict__ partials,
                int nslots) {
  using V = cplx_t<T>;
  __shared__ V red[4][64];
  const int p = threadIdx.x & 63, g = threadIdx.x >> 6;
  const int slot = blockIdx.x;
  const int64_t per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(slot) * per, r1 = (r0 + per) < n ? (r0 + per) : n;
  V s = czero<V>();
  if (p <= j)
    for (int64_t r = r0 + g; r < r1; r += 4) s = cfmac(W[r * k + p], W[r * k + j], s);
  red[g][p] = s;
  __syncthreads();
  if (g == 0 && p <= j) {
    V t = red[0][p];
    for (int gg = 1; gg < 4; ++gg) t = cadd(t, red[gg][p]);
    partials[int64_t(slot) * (j + 1) + p] = t;
  }
}

template <class T>
__global__ void __launch_bounds__(256)
col_update_kernel(int64_t n, int k, cplx_t<T>* __restrict__ W, int j, const cplx_t<T>* __restrict__ d) {
  using V = cplx_t<T>;
  const int64_t r = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (r >= n) return;
  V w = W[r * k + j];
  for (int p = 0; p < j; ++p) w = csub(w, cmul(d[p], W[r * k + p]));
  W[r * k + j] = w;
}

template <class T>
__global__ void __launch_bounds__(256)
col_finish_kernel(int64_t n, int k, cplx_t<T>* __restrict__ W, int j, const cplx_t<T>* __restrict__ d1,
                  const cplx_t<T>* __restrict__ d2, const cplx_t<T>* __restrict__ d3, cplx_t<T>* __restrict__ R,
                  int* flag, T tol) {
  using V = cplx_t<T>;
  const T norm0 = sqrt(d1[j].x), norm = sqrt(d3[j].x);
  const bool dead = norm <= tol * (norm0 > T(0) ? norm0 : T(1));
  const int64_t r = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (r < n) W[r * k + j] = dead ? czero<V>() : cscale(T(1) / norm, W[r * k + j]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int p = 0; p < j; ++p) R[p * k + j] = cadd(cadd(czero<V>(), d1[p]), d2 ? d2[p] : czero<V>());
    R[j * k + j] = dead ? czero<V>() : mk(norm, T(0));
    if (dead) *flag = 1;
  }
}

}  // namespace

template <class T>
void launch_mgs_qr(int64_t n, int k, cplx_t<T>* W, cplx_t<T>* R, cplx_t<T>* dbuf, cplx_t<T>* partials,
                   int max_slots, int* flag, cudaStream_t s) {
  using V = cplx_t<T>;
  const int nslots = int(std::max<int64_t>(1, std::min<int64_t>(max_slots, (n + 255) / 256)));
  ProfScope prof("mgs_qr", 6.0 * n * k * sizeof(V), s);
  HZ_CUDA(cudaMemsetAsync(R, 0, sizeof(V) * size_t(k) * k, s));
  HZ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const T tol = sizeof(T) == 8 ? T(1e-12) : T(1e-6);
  V* d1 = dbuf;
  V* d2 = dbuf + 64;
  V* d3 = dbuf + 128;
  auto dots = [&](int j, V* out) {
    col_dots_kernel<T><<<nslots, 256, 0, s>>>(n, k, W, j, partials, nslots);
    launch_reduce_partials<T>(j + 1, nslots, partials, out, s);
  };
  for (int j = 0; j < k; ++j) {
    dots(j, d1);
    if (j > 0) {
      col_update_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(n, k, W, j, d1);
      dots(j, d2);
      col_update_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(n, k, W, j, d2);
    }
    dots(j, d3);
    col_finish_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(n, k, W, j, d1, j > 0 ? d2 : nullptr, d3, R, flag,
                                                          tol);
  }
  HZ_LAUNCH_CHECK();
}
template void launch_mgs_qr<double>(int64_t, int, double2*, double2*, double2*, double2*, int, int*,
                                    cudaStream_t);
template void launch_mgs_qr<float>(int64_t, int, float2*, float2*, float2*, float2*, int, int*, cudaStream_t);

namespace {

// Pythagorean block CholQR factor for one Arnoldi step (single CTA of
// 1024 threads, operands staged in shared memory when they fit):
// Hc = [H_0 .. H_{nb-1}, G] from one Gram pass [V_0..V_{nb-1}, W]^H W.
// S = G - sum_i H_i^H H_i (= W'^H W' for W' = W - V H, V orthonormal);
// accepted when every Cholesky pivot keeps eta2 of its column's norm^2 (no
// severe cancellation, so the Pythagorean subtraction keeps full relative
// accuracy -- otherwise the caller re-orthogonalises with CGS2 + CholQR2);
// then S = R^H R and C_i = -H_i R^{-1}, C_nb = R^{-1}, so that
// Q = sum_i V_i C_i + W C_nb = (W - V H) R^{-1} in one block update.
// flag: 0 accepted, 1 rejected.
template <class T>
__global__ void __launch_bounds__(1024)
pip_factor_kernel(int k, int nb, const cplx_t<T>* __restrict__ Hc, cplx_t<T>* __restrict__ R,
                  cplx_t<T>* __restrict__ Rinv, cplx_t<T>* __restrict__ C, int* flag, T eta2, int staged) {
  using V = cplx_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int kk = k * k;
  V* A = reinterpret_cast<V*>(smem_raw);  // [k][k] S, then R
  V* Ri = A + kk;                         // [k][k] R^{-1}
  V* Hs = Ri + kk;                        // [nb+1][k][k] when staged
  const int tid = threadIdx.x, nt = blockDim.x;
  const V* H = Hc;
  if (staged) {
    for (int e = tid; e < (nb + 1) * kk; e += nt) Hs[e] = Hc[e];
    H = Hs;
  }
  __syncthreads();
  const V* G = H + int64_t(nb) * kk;
  for (int e = tid; e < kk; e += nt) {
    const int a = e / k, b = e - a * k;
    if (b < a) continue;  // upper triangle suffices
    V s = G[e];
    for (int i = 0; i < nb; ++i) {
      const V* Hi = H + int64_t(i) * kk;
#pragma unroll 4
      for (int p = 0; p < k; ++p) s = csub(s, cmulc(Hi[p * k + a], Hi[p * k + b]));
    }
    A[e] = s;
  }
  __syncthreads();
  // every pivot (squared norm of column j after projecting out V and the
  // earlier columns) must keep eta2 of the column's norm^2
  if (chol_upper_smem<T, true>(A, k, G, eta2)) {
    if (tid == 0) *flag = 1;
    return;
  }
  tri_inv_upper<T>(A, Ri, k);
  __syncthreads();
  for (int e = tid; e < kk; e += nt) {
    const int a = e / k, c = e % k;
    R[e] = c >= a ? A[e] : czero<V>();
    Rinv[e] = Ri[e];
  }
  for (int e = tid; e < (nb + 1) * kk; e += nt) {
    const int i = e / kk, r = e - i * kk, a = r / k, b = r - a * k;
    if (i == nb) {
      C[e] = Ri[r];
    } else {
      const V* Hi = H + int64_t(i) * kk;
      V s = czero<V>();
      for (int l = 0; l <= b; ++l) s = cfma(Hi[a * k + l], Ri[l * k + b], s);
      C[e] = mk(-s.x, -s.y);
    }
  }
  if (tid == 0) *flag = 0;
}

__global__ void __launch_bounds__(kBlk)
sensitivity_kernel(int64_t n, int k, double w2, const double2* __restrict__ gf,
                   const double2* __restrict__ U, const double2* __restrict__ L,
                   double* __restrict__ g, int accumulate) {
  const int64_t i = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (i >= n) return;
  const double2 f = gf[i];
  // reference per source: Re(-w2 * gf * u * lam), (-w2*gf) first
  const double2 c = make_double2(-w2 * f.x, -w2 * f.y);
  double s = accumulate ? g[i] : 0.0;
  for (int q = 0; q < k; ++q) {
    const double2 cu = cmul(c, U[i * k + q]);
    s += cu.x * L[i * k + q].x - cu.y * L[i * k + q].y;
  }
  g[i] = s;
}

template <class T, int TP, int TQ>
void gram_launch(int64_t n, int k, int nb, const BlockTab<T>& X, const cplx_t<T>* Y,
                 cplx_t<T>* partials, int nslots, cudaStream_t s) {
  const int tiles = ((k + TP - 1) / TP) * ((k + TQ - 1) / TQ);
  const int groups = std::max(1, kBlk / tiles);
  const size_t smem = groups > 1 ? sizeof(cplx_t<T>) * size_t(groups) * k * k : 0;
  auto kern = multi_gram_kernel<T, TP, TQ>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  dim3 grid(nb, nslots);
  kern<<<grid, kBlk, smem, s>>>(n, k, X, Y, partials, nslots);
}

}  // namespace

int gram_partial_slots(int64_t n, int k) {
  (void)k;
  return slots_for(n);
}

// FP64 tensor-core (DMMA) path for complex128; HZ_DMMA=0 selects the FFMA
// tiles instead (for comparison).
bool use_dmma() {
  static const bool on = [] {
    const char* e = std::getenv("HZ_DMMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int K>
void gram_dmma_launch(int64_t n, int nb, const BlockTab<double>& X, const double2* Y, double2* partials,
                      int nslots, cudaStream_t s) {
  const size_t smem = dmma::gram_smem<K>();
  auto kern = dmma::gram_kernel<K>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  kern<<<dim3(nb, nslots), 256, smem, s>>>(n, X, Y, partials, nslots);
}

template <int K>
void update_dmma_launch(int64_t n, int nb, const BlockTab<double>& X, const double2* H, const double2* Yin,
                        double2* Yout, double sign, cudaStream_t s) {
  const size_t smem = dmma::update_smem<K>();
  auto kern = dmma::update_kernel<K>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  kern<<<grid_for(n, dmma::UpdateCfg<K>::RC), dmma::UpdateCfg<K>::THREADS, smem, s>>>(n, nb, X, H, Yin, Yout,
                                                                                    sign);
}

template <class T, int K>
void gram_tiled_launch(int64_t n, int nb, const BlockTab<T>& X, const cplx_t<T>* Y,
                       cplx_t<T>* partials, int nslots, cudaStream_t s) {
  if constexpr (std::is_same<T, double>::value) {
    if (use_dmma()) return gram_dmma_launch<K>(n, nb, X, Y, partials, nslots, s);
  }
  const size_t smem = tiled::gram_smem<T, K>();
  auto kern = tiled::gram_kernel<T, K>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  kern<<<dim3(nb, nslots), 256, smem, s>>>(n, X, Y, partials, nslots);
}

template <class T, int K>
void update_tiled_launch(int64_t n, int nb, const BlockTab<T>& X, const cplx_t<T>* H,
                         const cplx_t<T>* Yin, cplx_t<T>* Yout, T sign, cudaStream_t s) {
  if constexpr (std::is_same<T, double>::value) {
    if (use_dmma()) return update_dmma_launch<K>(n, nb, X, H, Yin, Yout, sign, s);
  }
  constexpr int RC = tiled::update_rows<K>();
  const size_t smem = tiled::update_smem<T, K>();
  auto kern = tiled::update_kernel<T, K>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  kern<<<grid_for(n, RC), 256, smem, s>>>(n, nb, X, H, Yin, Yout, sign);
}

// K = 8 register-direct DMMA kernels (block_k8.cuh) for nb <= kK8MaxNb
constexpr int kK8MaxNb = 12;

template <int NB>
void gram8_dispatch(int nb, int64_t n, const BlockTab<double>& X, const double2* Y, double2* partials, int nslots,
                    cudaStream_t s) {
  if constexpr (NB <= kK8MaxNb) {
    if (nb == NB) {
      k8::gram8_kernel<NB><<<nslots, k8::kThreads, 0, s>>>(n, X, Y, partials);
      return;
    }
    gram8_dispatch<NB + 1>(nb, n, X, Y, partials, nslots, s);
  }
}

template <int NB, class TT>
void update8_dispatch(int nb, int64_t n, const BlockTab<TT>& X, const double2* H, const double2* Yin,
                      double2* Yout, double sign, cudaStream_t s) {
  if constexpr (NB <= kK8MaxNb) {
    if (nb == NB) {
      const int64_t tiles = (n + 7) / 8;
      const int grid =
          int(std::max<int64_t>(1, std::min<int64_t>(HZ_UPDATE8_MINB * kNumSMs, (tiles + 7) / 8)));
      k8::update8_kernel<NB, TT><<<grid, k8::kThreads, 0, s>>>(n, X, H, Yin, Yout, sign);
      return;
    }
    update8_dispatch<NB + 1, TT>(nb, n, X, H, Yin, Yout, sign, s);
  }
}

// Y += sum_i Z_i H_i, Z_i complex64 (widened), any k: one thread per output
// element, H tiles in shared memory, complex products in the reference's
// order (sum over i, then the k entries of a row)
__global__ void __launch_bounds__(kBlk)
update_lo_kernel(int64_t n, int k, int nb, const BlockTab<float> Z, const double2* __restrict__ H, double2* Y) {
  extern __shared__ double2 hsm[];
  for (int e = threadIdx.x; e < nb * k * k; e += kBlk) hsm[e] = H[e];
  __syncthreads();
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= n * k) return;
  const int64_t row = e / k;
  const int q = int(e - row * k);
  double2 acc = Y[e];
  for (int i = 0; i < nb; ++i) {
    const float2* z = Z.p[i] + row * k;
    const double2* h = hsm + size_t(i) * k * k;
    for (int p = 0; p < k; ++p) {
      const float2 zf = __ldg(z + p);
      acc = cfma(make_double2(double(zf.x), double(zf.y)), h[p * k + q], acc);
    }
  }
  Y[e] = acc;
}

template <int NB>
void gram16_dispatch(int nb, int64_t n, const BlockTab<double>& X, const double2* Y, double2* partials, int nslots,
                     cudaStream_t s) {
  if constexpr (NB <= kK8MaxNb) {
    if (nb == NB) {
      k16::gram16_kernel<NB><<<nslots, k8::kThreads, 0, s>>>(n, X, Y, partials);
      return;
    }
    gram16_dispatch<NB + 1>(nb, n, X, Y, partials, nslots, s);
  }
}

template <int NB, class TT>
void update16_dispatch(int nb, int64_t n, const BlockTab<TT>& X, const double2* H, const double2* Yin,
                       double2* Yout, double sign, cudaStream_t s) {
  if constexpr (NB <= kK8MaxNb) {
    if (nb == NB) {
      const int64_t tiles = (n + 7) / 8;
      const int grid = int(std::max<int64_t>(1, std::min<int64_t>(2 * kNumSMs, (tiles + 7) / 8)));
      k16::update16_kernel<NB, TT><<<grid, k8::kThreads, 0, s>>>(n, X, H, Yin, Yout, sign);
      return;
    }
    update16_dispatch<NB + 1, TT>(nb, n, X, H, Yin, Yout, sign, s);
  }
}

bool use_k8() {
  static const bool on = [] {
    const char* e = std::getenv("HZ_K8");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class T>
int launch_multi_gram(int64_t n, int k, int nb, const BlockTab<T>& X, const cplx_t<T>* Y,
                      cplx_t<T>* partials, int max_slots, cudaStream_t s) {
  if (k > 64) throw HzError(kValidation, "block width k > 64 unsupported");
  if (nb > kMaxBlocks) throw HzError(kValidation, "too many blocks in one Gram");
  // Y is usually the last X block (the Arnoldi step's [V_0..V_j, W]^H W):
  // then nb blocks are read, not nb + 1
  const double blocks = (nb > 0 && X.p[nb - 1] == Y) ? double(nb) : double(nb + 1);
  ProfScope prof(sizeof(T) == 8 ? "multi_gram_c128" : "multi_gram_c64", blocks * n * k * sizeof(cplx_t<T>), s,
                 8.0 * double(n) * k * k * nb);
  // ~4 CTAs per SM in total over the nb blocks; at least 32 rows per slot
  // exactly one wave of resident CTAs (3 per SM for the tiled / DMMA Grams)
  // over the nb blocks: a partial last wave would idle up to 2/3 of the GPU
  if constexpr (std::is_same<T, double>::value) {
    if ((k == 8 || k == 16) && nb >= 1 && nb <= kK8MaxNb && use_dmma() && use_k8()) {
      // one pass over all nb blocks per CTA: one wave of 2 CTAs per SM
      int64_t want = std::min<int64_t>(2 * kNumSMs, (n + 31) / 32);
      const int nslots = int(std::max<int64_t>(1, std::min<int64_t>(want, max_slots)));
      if (k == 8)
        gram8_dispatch<1>(nb, n, X, Y, partials, nslots, s);
      else
        gram16_dispatch<1>(nb, n, X, Y, partials, nslots, s);
      HZ_LAUNCH_CHECK();
      return nslots;
    }
  }
  int64_t want = std::max<int64_t>(1, (3 * kNumSMs) / nb);
  want = std::min<int64_t>(want, (n + 31) / 32);
  const int nslots = int(std::max<int64_t>(1, std::min<int64_t>(want, max_slots)));
  if (k == 32)
    gram_tiled_launch<T, 32>(n, nb, X, Y, partials, nslots, s);
  else if (k == 16)
    gram_tiled_launch<T, 16>(n, nb, X, Y, partials, nslots, s);
  else if (k == 64)
    gram_tiled_launch<T, 64>(n, nb, X, Y, partials, nslots, s);
  else if (k == 8)
    gram_tiled_launch<T, 8>(n, nb, X, Y, partials, nslots, s);
  else if (k < 16)
    gram_launch<T, 1, 1>(n, k, nb, X, Y, partials, nslots, s);
  else if (k <= 32)
    gram_launch<T, 2, 2>(n, k, nb, X, Y, partials, nslots, s);
  else
    gram_launch<T, 4, 4>(n, k, nb, X, Y, partials, nslots, s);
  HZ_LAUNCH_CHECK();
  return nslots;
}

template <class T>
void launch_multi_update(int64_t n, int k, int nb, const BlockTab<T>& X, const cplx_t<T>* H,
                         const cplx_t<T>* Yin, cplx_t<T>* Yout, T sign, cudaStream_t s) {
  ProfScope prof(sizeof(T) == 8 ? "multi_update_c128" : "multi_update_c64",
                 double(nb + (Yin ? 2 : 1)) * n * k * sizeof(cplx_t<T>), s, 8.0 * double(n) * k * k * nb);
  if (k == 32) {
    update_tiled_launch<T, 32>(n, nb, X, H, Yin, Yout, sign, s);
  } else if (k == 16) {
    bool done = false;
    if constexpr (std::is_same<T, double>::value) {
      if (nb >= 1 && nb <= kK8MaxNb && use_dmma() && use_k8()) {
        update16_dispatch<1, double>(nb, n, X, H, Yin, Yout, sign, s);
        done = true;
      }
    }
    if (!done) update_tiled_launch<T, 16>(n, nb, X, H, Yin, Yout, sign, s);
  } else if (k == 64) {
    update_tiled_launch<T, 64>(n, nb, X, H, Yin, Yout, sign, s);
  } else if (k == 8) {
    bool done = false;
    if constexpr (std::is_same<T, double>::value) {
      if (nb >= 1 && nb <= kK8MaxNb && use_dmma() && use_k8()) {
        update8_dispatch<1, double>(nb, n, X, H, Yin, Yout, sign, s);
        done = true;
      }
    }
    if (!done) update_tiled_launch<T, 8>(n, nb, X, H, Yin, Yout, sign, s);
  } else {
    const size_t smem = sizeof(cplx_t<T>) * size_t(k) * k;
    auto kern = multi_update_kernel<T>;
    allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
    kern<<<grid_for(n * k, kBlk), kBlk, smem, s>>>(n, k, nb, X, H, Yin, Yout, sign);
  }
  HZ_LAUNCH_CHECK();
}

void launch_update_lo(int64_t n, int k, int nb, const BlockTab<float>& Z, const double2* H, double2* Y,
                      cudaStream_t s) {
  ProfScope prof("multi_update_lo_c128", double(nb) * n * k * 8.0 + 2.0 * n * k * 16.0, s,
                 8.0 * double(n) * k * k * nb);
  if (nb < 1) return;
  if (k == 8 && nb <= kK8MaxNb && use_dmma() && use_k8()) {
    update8_dispatch<1, float>(nb, n, Z, H, Y, Y, 1.0, s);
  } else if (k == 16 && nb <= kK8MaxNb && use_dmma() && use_k8()) {
    update16_dispatch<1, float>(nb, n, Z, H, Y, Y, 1.0, s);
  } else {
    const size_t smem = sizeof(double2) * size_t(nb) * k * k;
    allow_dyn_smem(reinterpret_cast<const void*>(update_lo_kernel), int(smem));
    update_lo_kernel<<<grid_for(n * k, kBlk), kBlk, smem, s>>>(n, k, nb, Z, H, Y);
  }
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_reduce_partials(int64_t count, int nslots, const cplx_t<T>* partials, cplx_t<T>* out,
                            cudaStream_t s) {
  ProfScope prof("reduce_partials", double(count) * (nslots + 1) * sizeof(cplx_t<T>), s);
  reduce_partials_kernel<T><<<grid_for(count, 32), kBlk, 0, s>>>(count, nslots, partials, out);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_colnorm2_partial(int64_t n, int k, const cplx_t<T>* X, T* partials, int nslots,
                             cudaStream_t s) {
  ProfScope prof("colnorm2", double(n) * k * sizeof(cplx_t<T>), s);
  colnorm2_kernel<T><<<nslots, kBlk, sizeof(T) * kBlk, s>>>(n, k, X, partials, nslots);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_reduce_real(int64_t count, int nslots, const T* partials, T* out, cudaStream_t s) {
  reduce_real_kernel<T><<<grid_for(count, kBlk), kBlk, 0, s>>>(count, nslots, partials, out);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_axpby(int64_t count, cplx_t<T> a, cplx_t<T>* Y, cplx_t<T> b, const cplx_t<T>* X,
                  cudaStream_t s) {
  ProfScope prof("axpby", 3.0 * count * sizeof(cplx_t<T>), s);
  axpby_kernel<T><<<grid_for(count, kBlk), kBlk, 0, s>>>(count, a, Y, b, X);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_bicgstab_update(int64_t count, cplx_t<T> omega, cplx_t<T>* X, const cplx_t<T>* ZS,
                            cplx_t<T>* R, const cplx_t<T>* S, const cplx_t<T>* Tt, cudaStream_t s) {
  bicgstab_update_kernel<T><<<grid_for(count, kBlk), kBlk, 0, s>>>(count, omega, X, ZS, R, S, Tt);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_frob2_partial(int64_t count, const cplx_t<T>* Tt, const cplx_t<T>* S,
                          cplx_t<T>* partials, int nslots, cudaStream_t s) {
  frob2_kernel<T><<<nslots, kBlk, 0, s>>>(count, Tt, S, partials, nslots);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_small_cholesky(int k, const cplx_t<T>* G, cplx_t<T>* R, cplx_t<T>* Rinv, int* flag,
                           T rel_tol, cudaStream_t s) {
  if (k > 64) throw HzError(kValidation, "small_cholesky: k > 64");
  const size_t smem = 2 * sizeof(cplx_t<T>) * size_t(k) * k;
  auto kern = small_cholesky_kernel<T>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  ProfScope prof("small_cholesky", 4.0 * k * k * sizeof(cplx_t<T>), s);
  kern<<<1, 1024, smem, s>>>(k, G, R, Rinv, flag, rel_tol);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_pip_factor(int k, int nb, const cplx_t<T>* Hc, cplx_t<T>* R, cplx_t<T>* Rinv,
                       cplx_t<T>* C, int* flag, T eta2, cudaStream_t s) {
  const size_t base = sizeof(cplx_t<T>) * 2 * size_t(k) * k;
  const size_t full = base + sizeof(cplx_t<T>) * size_t(nb + 1) * k * k;
  const int staged = full <= 200 * 1024 ? 1 : 0;
  const size_t smem = staged ? full : base;
  auto kern = pip_factor_kernel<T>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), 200 * 1024);
  ProfScope prof("pip_factor", double(nb + 2) * k * k * sizeof(cplx_t<T>), s);
  kern<<<1, 1024, smem, s>>>(k, nb, Hc, R, Rinv, C, flag, eta2, staged);
  HZ_LAUNCH_CHECK();
}
template void launch_pip_factor<double>(int, int, const double2*, double2*, double2*, double2*, int*,
                                        double, cudaStream_t);
template void launch_pip_factor<float>(int, int, const float2*, float2*, float2*, float2*, int*, float,
                                       cudaStream_t);

void launch_sensitivity(int64_t n, int k, double w2, const double2* gf, const double2* U,
                        const double2* L, double* g, int accumulate, cudaStream_t s) {
  sensitivity_kernel<<<grid_for(n, kBlk), kBlk, 0, s>>>(n, k, w2, gf, U, L, g, accumulate);
  HZ_LAUNCH_CHECK();
}

#define HZ_INST(T)                                                                                 \
  template int launch_multi_gram<T>(int64_t, int, int, const BlockTab<T>&, const cplx_t<T>*,      \
                                     cplx_t<T>*, int, cudaStream_t);                              \
  template void launch_multi_update<T>(int64_t, int, int, const BlockTab<T>&,                     \
                                       const cplx_t<T>*, const cplx_t<T>*, cplx_t<T>*, T,         \
                                       cudaStream_t);                                             \
  template void launch_reduce_partials<T>(int64_t, int, const cplx_t<T>*, cplx_t<T>*,             \
                                          cudaStream_t);                                          \
  template void launch_colnorm2_partial<T>(int64_t, int, const cplx_t<T>*, T*, int, cudaStream_t); \
  template void launch_reduce_real<T>(int64_t, int, const T*, T*, cudaStream_t);                  \
  template void launch_axpby<T>(int64_t, cplx_t<T>, cplx_t<T>*, cplx_t<T>, const cplx_t<T>*,      \
                                cudaStream_t);                                                    \
  template void launch_bicgstab_update<T>(int64_t, cplx_t<T>, cplx_t<T>*, const cplx_t<T>*,       \
                                          cplx_t<T>*, const cplx_t<T>*, const cplx_t<T>*,         \
                                          cudaStream_t);                                          \
  template void launch_frob2_partial<T>(int64_t, const cplx_t<T>*, const cplx_t<T>*, cplx_t<T>*,  \
                                        int, cudaStream_t);                                       \
  template void launch_small_cholesky<T>(int, const cplx_t<T>*, cplx_t<T>*, cplx_t<T>*, int*, T,  \
                                         cudaStream_t);
HZ_INST(double)
HZ_INST(float)
#undef HZ_INST

namespace {
// 4 independent DMMA accumulator chains per warp, operands in registers
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-9, b = 1.0;
  double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) dmma::mma884(d[c][0], d[c][1], a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = d[0][0] + d[0][1] + d[1][0] + d[1][1] + d[2][0] + d[2][1] +
                                               d[3][0] + d[3][1];
}
}  // namespace

double measure_dmma_tflops() {
  int dev = 0, sms = 0;
  HZ_CUDA(cudaGetDevice(&dev));
  HZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms * 8, threads = 256, iters = 400;
  DevBuf<double> out;
  out.alloc(size_t(blocks) * threads);
  cudaEvent_t e0, e1;
  HZ_CUDA(cudaEventCreate(&e0));
  HZ_CUDA(cudaEventCreate(&e1));
  dmma_peak_kernel<<<blocks, threads>>>(out.get(), 20);  // warm-up / clocks up
  HZ_LAUNCH_CHECK();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    HZ_CUDA(cudaEventRecord(e0));
    dmma_peak_kernel<<<blocks, threads>>>(out.get(), iters);
    HZ_LAUNCH_CHECK();
    HZ_CUDA(cudaEventRecord(e1));
    HZ_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    HZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  HZ_CUDA(cudaEventDestroy(e0));
  HZ_CUDA(cudaEventDestroy(e1));
  // 2 * 8*8*4 flops per mma, 64 mma per iteration per warp
  const double flops = 2.0 * 256 * 64.0 * iters * (double(blocks) * threads / 32);
  return flops / (double(best) * 1e-3) / 1e12;
}

}  // namespace hz
