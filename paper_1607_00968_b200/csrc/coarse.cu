// Coarsest-level direct solve (K5; MgHierarchy::coarse_solve,
// src/multigrid.cpp:114-117 -> BandedLU::solve, src/dense.cpp:39-61).
//
// The reference runs a sequential banded forward/back substitution per
// column on every cycle. On the GPU that is a latency-bound chain of 2*n_c
// dependent steps, so the hierarchy instead forms A_c^{-1} ONCE at setup from
// the same pivoted banded LU factors (one warp per identity column), and every
// cycle applies it as one bandwidth-bound dense pass: n_c^2 complex reads.
#include "block_tiled.cuh"
#include "kernels.hpp"
#include "profile.hpp"

namespace hz {

int split_for_tiles(int tiles);

namespace {

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm (robust against overflow), as libgcc's __divdc3
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

// ab: gbtrf-style band storage, at(i, j) = ab[(kl + ku + i - j) + j * ld]
// (inc/dense.hpp:207-208). One warp solves A x = e_c for column c.
__global__ void __launch_bounds__(128)
banded_inverse_kernel(int64_t n, int64_t kl, int64_t ku, int64_t ld, const double2* __restrict__ ab,
                      const int64_t* __restrict__ piv, double2* __restrict__ ainvT) {
  const int lane = threadIdx.x & 31;
  const int64_t c = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (c >= n) return;
  const int64_t ldx = inv_ld(n);
  double2* x = ainvT + c * ldx;
  for (int64_t i = lane; i < ldx; i += 32) x[i] = make_double2(i == c ? 1.0 : 0.0, 0.0);
  __syncwarp();
  auto at = [&](int64_t i, int64_t j) { return ab[(kl + ku + i - j) + j * ld]; };
  // forward: row interchanges + unit-lower elimination (src/dense.cpp:46-52)
  for (int64_t k = 0; k < n; ++k) {
    const int64_t p = piv[k];
    if (p != k) {
      if (lane == 0) {
        const double2 t = x[k];
        x[k] = x[p];
        x[p] = t;
      }
      __syncwarp();
    }
    const double2 bk = x[k];
    if (bk.x != 0.0 || bk.y != 0.0) {
      const int64_t imax = min(n - 1, k + kl);
      for (int64_t i = k + 1 + lane; i <= imax; i += 32) {
        const double2 l = at(i, k);
        double2 xi = x[i];
        xi.x -= l.x * bk.x - l.y * bk.y;
        xi.y -= l.x * bk.y + l.y * bk.x;
        x[i] = xi;
      }
    }
    __syncwarp();
  }
  // backward: upper solve (src/dense.cpp:53-58)
  for (int64_t k = n - 1; k >= 0; --k) {
    const int64_t jmax = min(n - 1, k + kl + ku);
    double sx = 0.0, sy = 0.0;
    for (int64_t j = k + 1 + lane; j <= jmax; j += 32) {
      const double2 u = at(k, j);
      const double2 xj = x[j];
      sx += u.x * xj.x - u.y * xj.y;
      sy += u.x * xj.y + u.y * xj.x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    if (lane == 0) {
      const double2 v = make_double2(x[k].x - sx, x[k].y - sy);
      x[k] = cdiv(v, at(k, k));
    }
    __syncwarp();
  }
}

// X[i][q] = sum_l ainvT[l][i] B[l][q]. CTA = TI output rows x all k columns;
// ainvT is streamed once (coalesced TI-wide row segments), B chunks come
// from L2.
template <class T, int TI, int TL>
__global__ void __launch_bounds__(256)
coarse_solve_kernel(int64_t n, int k, const cplx_t<T>* __restrict__ ainvT, int64_t ld,
                    const cplx_t<T>* __restrict__ b, cplx_t<T>* x, const cplx_t<T>* c_in, T sign) {
  using V = cplx_t<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* As = reinterpret_cast<V*>(smem_raw);  // [TL][TI]
  V* Bs = As + TL * TI;                    // [TL][k]
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int nout = TI * k;
  constexpr int kMaxPer = 16;  // TI*k <= 256*16
  V acc[kMaxPer];
#pragma unroll
  for (int t = 0; t < kMaxPer; ++t) acc[t] = czero<V>();
  for (int64_t l0 = 0; l0 < n; l0 += TL) {
    const int tl = (n - l0) < TL ? int(n - l0) : TL;
    for (int e = threadIdx.x; e < TL * TI; e += 256) {
      const int l = e / TI, i = e % TI;
      As[e] = (l < tl && i0 + i < n) ? ainvT[(l0 + l) * ld + i0 + i] : czero<V>();
    }
    for (int e = threadIdx.x; e < TL * k; e += 256) {
      const int l = e / k;
      Bs[e] = l < tl ? b[(l0 + l) * k + (e - l * k)] : czero<V>();
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
      const int o = threadIdx.x + t * 256;
      if (o < nout) {
        const int i = o / k, q = o - i * k;
        V a = acc[t];
        for (int l = 0; l < TL; ++l) a = cfma(As[l * TI + i], Bs[l * k + q], a);
        acc[t] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < kMaxPer; ++t) {
    const int o = threadIdx.x + t * 256;
    if (o < nout) {
      const int i = o / k, q = o - i * k;
      if (i0 + i < n) {
        V v = acc[t];
        if (c_in) {
          const V c = c_in[(i0 + i) * k + q];
          v = mk(c.x + sign * v.x, c.y + sign * v.y);
        }
        x[(i0 + i) * k + q] = v;
      }
    }
  }
}

// Register tile of the coarse GEMM: c64 uses 8 rows x TQ columns per thread
// (FP32, ~80% of issued instructions are FFMA), c128 4 rows x TQ (FP64 keeps
// the 3-mult accumulators within the register budget).
template <class T, int K>
struct CoarseTile {
  static constexpr bool F32 = sizeof(T) == 4;
  static constexpr int NQT = K < 16 ? K : ((F32 && K <= 32) ? 8 : 16);  // column threads
  static constexpr int TQ = K / NQT;                        // columns per thread (strided)
  static constexpr int NIT = 256 / NQT;                     // row threads
  static constexpr int TA = F32 ? (K <= 32 ? 8 : 4) : 4;    // rows per thread (strided)
  static constexpr int TI = NIT * TA;                       // rows per CTA
  static constexpr int TL = 16;                             // l per stage
};

// Tiled dense coarse solve for K in {16, 32, 64}: CTA = 64 output rows x K
// columns over one split-K slice of l; A^{-1} rows and B rows are streamed
// through double-buffered cp.async stages; thread tile 4 (i) x K/16 (q),
// both strided so a warp's shared loads are broadcast / contiguous; 3-mult
// complex products. Slices write partials summed in fixed order afterwards.
template <class T, int K>
__global__ void __launch_bounds__(256)
coarse_gemm_kernel(int64_t n, const cplx_t<T>* __restrict__ ainvT, int64_t ld, const cplx_t<T>* __restrict__ b,
                   cplx_t<T>* part, int nsplit, const cplx_t<T>* c_in, T sign) {
  using V = cplx_t<T>;
  using Tile = CoarseTile<T, K>;
  constexpr int TI = Tile::TI, TL = Tile::TL, NQT = Tile::NQT, TQ = Tile::TQ, NIT = Tile::NIT,
                TA = Tile::TA;
  constexpr int AT = TL * TI, BT = TL * K, STAGE = AT + BT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);
  const int tid = threadIdx.x, qt = tid % NQT, it = tid / NQT;
  const int64_t i0 = int64_t(blockIdx.x) * TI;
  const int split = blockIdx.y;
  const int64_t per = (n + nsplit - 1) / nsplit;
  const int64_t l0 = int64_t(split) * per, l1 = (l0 + per) < n ? (l0 + per) : n;
  const int nch = l1 > l0 ? int((l1 - l0 + TL - 1) / TL) : 0;
  const int icount = (n - i0) < TI ? int(n - i0) : TI;
  T t1[TA][TQ], t2[TA][TQ], t3[TA][TQ];
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int q = 0; q < TQ; ++q) t1[a][q] = t2[a][q] = t3[a][q] = T(0);
  constexpr int PER16 = 16 / sizeof(V);
  auto stage = [&](int c, V* dst) {
    const int64_t lc = l0 + int64_t(c) * TL;
    const int lrows = (l1 - lc) < TL ? int(l1 - lc) : TL;
    for (int e = tid; e < TL * (TI / PER16); e += 256) {
      const int l = e / (TI / PER16), ii = (e - l * (TI / PER16)) * PER16;
      V* d = dst + l * TI + ii;
      if (l < lrows && ii < icount)  // icount is a multiple of PER16 unless at the end
        tiled::cp_async16(d, ainvT + (lc + l) * ld + i0 + ii);
      else
        for (int u = 0; u < PER16; ++u) d[u] = czero<V>();
    }
    for (int e = tid; e < TL * (K / PER16); e += 256) {
      const int l = e / (K / PER16), qq = (e - l * (K / PER16)) * PER16;
      V* d = dst + AT + l * K + qq;
      if (l < lrows)
        tiled::cp_async16(d, b + (lc + l) * K + qq);
      else
        for (int u = 0; u < PER16; ++u) d[u] = czero<V>();
    }
  };
  if (nch > 0) stage(0, buf);
  tiled::cp_async_commit();
  for (int c = 0; c < nch; ++c) {
    const int st = c & 1;
    if (c + 1 < nch) stage(c + 1, buf + (st ^ 1) * STAGE);
    tiled::cp_async_commit();
    tiled::cp_async_wait<1>();
    __syncthreads();
    const V* as = buf + st * STAGE;
    const V* bs = as + AT;
#pragma unroll 4
    for (int l = 0; l < TL; ++l) {
      V bv[TQ];
      T bsum[TQ];
#pragma unroll
      for (int q = 0; q < TQ; ++q) {
        bv[q] = bs[l * K + qt + NQT * q];
        bsum[q] = bv[q].x + bv[q].y;
      }
#pragma unroll
      for (int a = 0; a < TA; ++a) {
        const V av = as[l * TI + it + NIT * a];
        const T asum = av.x + av.y;
#pragma unroll
        for (int q = 0; q < TQ; ++q) {
          t1[a][q] = fma(av.x, bv[q].x, t1[a][q]);
          t2[a][q] = fma(av.y, bv[q].y, t2[a][q]);
          t3[a][q] = fma(asum, bsum[q], t3[a][q]);
        }
      }
    }
    __syncthreads();
  }
  tiled::cp_async_wait<0>();
  V* out = part + int64_t(split) * n * K;
#pragma unroll
  for (int a = 0; a < TA; ++a) {
    const int64_t i = i0 + it + NIT * a;
    if (i >= n) continue;
#pragma unroll
    for (int q = 0; q < TQ; ++q) {
      V v;
      v.x = t1[a][q] - t2[a][q];
      v.y = t3[a][q] - t1[a][q] - t2[a][q];
      if (nsplit == 1 && c_in) {  // unsplit: fuse the x = c_in + sign * (A b) epilogue
        const V c = c_in[i * K + qt + NQT * q];
        v = mk(c.x + sign * v.x, c.y + sign * v.y);
      }
      out[i * K + qt + NQT * q] = v;
    }
  }
}

template <class T>
__global__ void __launch_bounds__(256)
split_reduce_kernel(int64_t count, int nsplit, const cplx_t<T>* __restrict__ part, cplx_t<T>* x,
                    const cplx_t<T>* c_in, T sign) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= count) return;
  cplx_t<T> s = part[e];
  for (int t = 1; t < nsplit; ++t) s = cadd(s, part[int64_t(t) * count + e]);
  if (c_in) {
    const cplx_t<T> c = c_in[e];
    s = mk(c.x + sign * s.x, c.y + sign * s.y);
  }
  x[e] = s;
}

template <class T, int K>
void coarse_gemm_launch(int64_t n, const cplx_t<T>* ainvT, int64_t ld, const cplx_t<T>* b, cplx_t<T>* x,
                        const cplx_t<T>* c_in, T sign, cplx_t<T>* part, int nsplit, cudaStream_t s) {
  using V = cplx_t<T>;
  constexpr int TI = CoarseTile<T, K>::TI, TL = CoarseTile<T, K>::TL;
  const size_t smem = sizeof(V) * 2 * (TL * TI + TL * K);
  auto kern = coarse_gemm_kernel<T, K>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
  const int tiles = grid_for(n, TI);
  nsplit = std::min(nsplit, split_for_tiles(tiles));
  if (nsplit > 1 && part == nullptr) nsplit = 1;
  kern<<<dim3(tiles, nsplit), 256, smem, s>>>(n, ainvT, ld, b, nsplit == 1 ? x : part, nsplit, c_in, sign);
  if (nsplit > 1)
    split_reduce_kernel<T><<<grid_for(n * K, 256), 256, 0, s>>>(n * K, nsplit, part, x, c_in, sign);
}

}  // namespace

// Split-K factor: fill a whole number of waves (2 resident CTAs per SM x 148
// SMs) instead of leaving a partial last wave.
int split_for_tiles(int tiles) {
  int sk = (2 * kNumSMs) / tiles;
  return sk < 1 ? 1 : (sk > 32 ? 32 : sk);
}

int coarse_split(int64_t n, int k) {
  if (k != 8 && k != 16 && k != 32 && k != 64) return 0;
  // upper bound over both precisions: the fewest row tiles (256-row c64
  // tiles) give the largest split
  return split_for_tiles(grid_for(n, 256));
}


void launch_banded_inverse(int64_t n, int64_t kl, int64_t ku, int64_t ld, const double2* ab,
                           const int64_t* piv, double2* ainvT, cudaStream_t s) {
  banded_inverse_kernel<<<grid_for(n, 4), 128, 0, s>>>(n, kl, ku, ld, ab, piv, ainvT);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_coarse_gemm(int64_t n, int k, const cplx_t<T>* ainvT, int64_t ld, const cplx_t<T>* b, cplx_t<T>* x,
                        const cplx_t<T>* c_in, T sign, cplx_t<T>* part, cudaStream_t s) {
  using V = cplx_t<T>;
  const int sk = coarse_split(n, k);
  if (sk > 0 && (part != nullptr || sk == 1)) {
    if (k == 32)
      coarse_gemm_launch<T, 32>(n, ainvT, ld, b, x, c_in, sign, part, sk, s);
    else if (k == 16)
      coarse_gemm_launch<T, 16>(n, ainvT, ld, b, x, c_in, sign, part, sk, s);
    else if (k == 8)
      coarse_gemm_launch<T, 8>(n, ainvT, ld, b, x, c_in, sign, part, sk, s);
    else
      coarse_gemm_launch<T, 64>(n, ainvT, ld, b, x, c_in, sign, part, sk, s);
    HZ_LAUNCH_CHECK();
    return;
  }
  constexpr int TL = 32;
  if (k > 256) throw HzError(kValidation, "coarse solve: k > 256 unsupported");
  // TI*k <= 4096 outputs per CTA (16 per thread)
  int ti = 16;
  if (k > 64) ti = 4096 / k >= 16 ? 16 : (4096 / k >= 8 ? 8 : (4096 / k >= 4 ? 4 : 1));
  const size_t smem = sizeof(V) * (TL * 16 + TL * size_t(k));
  const int grid = grid_for(n, ti);
  auto go = [&](auto kern) {
    allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
    kern<<<grid, 256, smem, s>>>(n, k, ainvT, ld, b, x, c_in, sign);
  };
  if (ti == 16)
    go(coarse_solve_kernel<T, 16, TL>);
  else if (ti == 8)
    go(coarse_solve_kernel<T, 8, TL>);
  else if (ti == 4)
    go(coarse_solve_kernel<T, 4, TL>);
  else
    go(coarse_solve_kernel<T, 1, TL>);
  HZ_LAUNCH_CHECK();
}

template <class T>
void launch_coarse_solve(int64_t n, int k, const cplx_t<T>* ainvT, const cplx_t<T>* b,
                         cplx_t<T>* x, cplx_t<T>* part, cudaStream_t s) {
  ProfScope prof(sizeof(T) == 8 ? "coarse_solve_c128" : "coarse_solve_c64",
                 (double(n) * n + 2.0 * n * k) * sizeof(cplx_t<T>), s, 8.0 * double(n) * n * k);
  launch_coarse_gemm<T>(n, k, ainvT, inv_ld(n), b, x, nullptr, T(1), part, s);
}

template void launch_coarse_gemm<double>(int64_t, int, const double2*, int64_t, const double2*, double2*,
                                         const double2*, double, double2*, cudaStream_t);
template void launch_coarse_gemm<float>(int64_t, int, const float2*, int64_t, const float2*, float2*,
                                        const float2*, float, float2*, cudaStream_t);
template void launch_coarse_solve<double>(int64_t, int, const double2*, const double2*, double2*,
                                          double2*, cudaStream_t);
template void launch_coarse_solve<float>(int64_t, int, const float2*, const float2*, float2*,
                                         float2*, cudaStream_t);

}  // namespace hz
