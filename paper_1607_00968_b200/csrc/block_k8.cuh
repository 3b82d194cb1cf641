// Register-direct FP64 tensor-core (DMMA m8n8k4) Gram and block update for
// complex128 blocks of K = 8 columns (included by block.cu).
//
// At K = 8 a node row is 128 bytes, so the m8n8k4 fragments can be loaded
// straight from global memory with no shared-memory staging: for 4
// consecutive rows r0..r0+3 the Gram operands A[g][t] = X[r0+t][g] and
// B[t][g] = Y[r0+t][g] are one 16-byte load per lane (lane = 4g + t) and the
// warp's 32 loads cover exactly the 512 contiguous bytes of those rows. For
// the update, A[g][t] = X[r0+g][q0+t] (q0 = 0, 4) is two loads per lane over
// the 1 KB of 8 rows. One pass reads every block once (the staged kernels of
// block_dmma.cuh re-read Y once per X block and synchronise per 32-row
// chunk); per row the Gram does 3 nb DMMA per 16 (nb + 1) bytes, HBM-bound.
// Complex products use the same 3-multiplication forms as block_dmma.cuh.
#pragma once

#include "block_dmma.cuh"

namespace hz {
namespace k8 {

constexpr int kThreads = 256;
constexpr int kRowsPerStep = 4;  // Gram: rows per DMMA k-step

// row groups in flight per warp and resident CTAs per SM (registers: the
// Gram keeps 12 NB accumulator registers per lane)
#ifndef HZ_GRAM8_U12
#define HZ_GRAM8_U12 2  // row groups in flight per warp for NB <= 2
#endif
template <int NB>
struct Gram8Cfg {
  static constexpr int U = NB <= 2 ? HZ_GRAM8_U12 : (NB <= 3 ? 2 : 1);
  static constexpr int MINB = NB <= 6 ? 2 : 1;
};

// partials[(slot * nb + i) * 64 + p * 8 + q] = sum over the slot's rows of
// conj(X_i[r][p]) Y[r][q]; slot = blockIdx.x owns a contiguous range of
// 4-row groups, its 8 warps take them round robin (fixed order).
template <int NB>
__global__ void __launch_bounds__(kThreads, Gram8Cfg<NB>::MINB)
gram8_kernel(int64_t n, const BlockTab<double> X, const double2* __restrict__ Y, double2* __restrict__ partials) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int slot = blockIdx.x, nslots = gridDim.x;
  const int64_t groups = (n + kRowsPerStep - 1) / kRowsPerStep;
  const int64_t per = (groups + nslots - 1) / nslots;
  const int64_t g0 = int64_t(slot) * per;
  const int64_t g1 = (g0 + per) < groups ? (g0 + per) : groups;
  double acc[NB][3][2];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int m = 0; m < 3; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
  constexpr int kUnroll = Gram8Cfg<NB>::U;
  for (int64_t rg = g0 + warp; rg < g1; rg += 8 * kUnroll) {
    double2 y[kUnroll], x[kUnroll][NB];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t row = (rg + 8 * u) * kRowsPerStep + t;
      const bool ok = rg + 8 * u < g1 && row < n;
      const int64_t e = row * 8 + g;
      y[u] = ok ? __ldg(Y + e) : czero<double2>();
#pragma unroll
      for (int i = 0; i < NB; ++i) x[u][i] = ok ? __ldg(X.p[i] + e) : czero<double2>();
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const double b0 = y[u].x, b1 = y[u].y, b2 = y[u].x - y[u].y;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        dmma::mma884(acc[i][0][0], acc[i][0][1], x[u][i].x, b0);
        dmma::mma884(acc[i][1][0], acc[i][1][1], x[u][i].y, b1);
        dmma::mma884(acc[i][2][0], acc[i][2][1], x[u][i].x + x[u][i].y, b2);
      }
    }
  }
  // fixed-order reduction of the 8 warps: red[i][g][2t + h]
  __shared__ double2 red[NB * 64];
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 v;
          v.x = acc[i][0][h] + acc[i][1][h];
          v.y = acc[i][0][h] - acc[i][1][h] - acc[i][2][h];
          const int e = i * 64 + g * 8 + 2 * t + h;
          red[e] = w == 0 ? v : cadd(red[e], v);
        }
    }
    __syncthreads();
  }
  double2* out = partials + int64_t(slot) * NB * 64;
  for (int e = threadIdx.x; e < NB * 64; e += kThreads) out[e] = red[e];
}

// Yout = Yin + sign * sum_i X_i H_i (Yin may be null = 0; Yout may alias
// Yin). Warps take 8-row tiles round robin over the grid; the H_i tiles are
// staged once per CTA in shared memory (fragment reads are 512 contiguous
// bytes per warp, conflict-free) and the X_i loads are issued in chunks of
// four blocks (8 KB per warp in flight).
template <class XV>
__device__ __forceinline__ double2 ld_widen(const XV* p) {
  const XV v = __ldg(p);
  return make_double2(double(v.x), double(v.y));
}

// TT = float: the X_i are complex64 blocks widened on load (exact)
#ifndef HZ_UPDATE8_MINB
#define HZ_UPDATE8_MINB 2
#endif
template <int NB, class TT = double>
__global__ void __launch_bounds__(kThreads, HZ_UPDATE8_MINB)
update8_kernel(int64_t n, const BlockTab<TT> X, const double2* __restrict__ H, const double2* Yin,
               double2* Yout, double sign) {
  // H_i[4s + t][g] staged at hs[i][s][g][t]: the B fragment of lane 4g + t is
  // hs[i][s][lane], so a warp's fragment load is 512 contiguous bytes
  // (the [p][q] order put lanes t = 0..3 of a quarter-warp on one bank group)
  __shared__ double2 hs[NB * 64];
  for (int e = threadIdx.x; e < NB * 64; e += kThreads) {
    const int i = e >> 6, p = (e >> 3) & 7, q = e & 7;
    hs[i * 64 + (p >> 2) * 32 + q * 4 + (p & 3)] = H[e];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  constexpr int CH = 4;
  const int64_t tiles = (n + 7) / 8;
  for (int64_t tile = int64_t(blockIdx.x) * 8 + warp; tile < tiles; tile += int64_t(gridDim.x) * 8) {
    const int64_t row = tile * 8 + g;
    const bool ok = row < n;
    double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int i0 = 0; i0 < NB; i0 += CH) {
      double2 xa[CH][2];
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (i0 + c < NB) xa[c][s] = ok ? ld_widen(X.p[i0 + c] + row * 8 + 4 * s + t) : czero<double2>();
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (i0 + c < NB) {
            // B[t][g] = H_i[q0 + t][g], q0 = 4 s
            const double2 h = hs[(i0 + c) * 64 + s * 32 + lane];
            const double2 x = xa[c][s];
            dmma::mma884(acc[0][0], acc[0][1], x.x, h.x);
            dmma::mma884(acc[1][0], acc[1][1], x.y, h.y);
            dmma::mma884(acc[2][0], acc[2][1], x.x + x.y, h.x + h.y);
          }
    }
    if (ok) {
      const int64_t base = row * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 y = Yin ? Yin[base + h] : czero<double2>();
        y.x += sign * (acc[0][h] - acc[1][h]);
        y.y += sign * (acc[2][h] - acc[0][h] - acc[1][h]);
        Yout[base + h] = y;
      }
    }
  }
}

}  // namespace k8
}  // namespace hz

namespace hz {
namespace k16 {

// K = 16 register-direct forms. Gram: warp w takes p-half a = w & 1 of every
// 4-row group it visits (row groups go to the 4 warps of its half round
// robin); lane (g, t) loads X[r][8a + g] (one 16-byte load per block) and
// Y[r][8b + g] for both q-halves b, and accumulates the 8 x 8 tiles (a, b).
template <int NB>
struct Gram16Cfg {  // 24 NB accumulator registers per lane
  static constexpr int MINB = NB <= 3 ? 2 : 1;
};

template <int NB>
__global__ void __launch_bounds__(k8::kThreads, Gram16Cfg<NB>::MINB)
gram16_kernel(int64_t n, const BlockTab<double> X, const double2* __restrict__ Y, double2* __restrict__ partials) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int a = warp & 1, wr = warp >> 1;  // p-half, row stream (4 per half)
  const int slot = blockIdx.x, nslots = gridDim.x;
  const int64_t groups = (n + 3) / 4;
  const int64_t per = (groups + nslots - 1) / nslots;
  const int64_t g0 = int64_t(slot) * per;
  const int64_t g1 = (g0 + per) < groups ? (g0 + per) : groups;
  double acc[NB][2][3][2];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[i][b][m][0] = acc[i][b][m][1] = 0.0;
  for (int64_t rg = g0 + wr; rg < g1; rg += 4) {
    const int64_t row = rg * 4 + t;
    const bool ok = row < n;
    const int64_t e = row * 16 + g;
    double2 y[2], x[NB];
#pragma unroll
    for (int b = 0; b < 2; ++b) y[b] = ok ? __ldg(Y + e + 8 * b) : czero<double2>();
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = ok ? __ldg(X.p[i] + e + 8 * a) : czero<double2>();
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double b0 = y[b].x, b1 = y[b].y, b2 = y[b].x - y[b].y;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        dmma::mma884(acc[i][b][0][0], acc[i][b][0][1], x[i].x, b0);
        dmma::mma884(acc[i][b][1][0], acc[i][b][1][1], x[i].y, b1);
        dmma::mma884(acc[i][b][2][0], acc[i][b][2][1], x[i].x + x[i].y, b2);
      }
    }
  }
  // fixed-order reduction over the 4 row streams of each half
  __shared__ double2 red[NB * 256];
  for (int w = 0; w < 4; ++w) {
    if (wr == w) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double2 v;
            v.x = acc[i][b][0][h] + acc[i][b][1][h];
            v.y = acc[i][b][0][h] - acc[i][b][1][h] - acc[i][b][2][h];
            const int e = i * 256 + (8 * a + g) * 16 + 8 * b + 2 * t + h;
            red[e] = w == 0 ? v : cadd(red[e], v);
          }
    }
    __syncthreads();
  }
  double2* out = partials + int64_t(slot) * NB * 256;
  for (int e = threadIdx.x; e < NB * 256; e += k8::kThreads) out[e] = red[e];
}

// Yout = Yin + sign * sum_i X_i H_i, 16 columns; warps take 8-row tiles; per
// block 4 k-steps (q0 = 4 s, A = X[r0+g][q0+t]) x 2 output halves.
template <int NB, class TT = double>
__global__ void __launch_bounds__(k8::kThreads, 2)
update16_kernel(int64_t n, const BlockTab<TT> X, const double2* __restrict__ H, const double2* Yin, double2* Yout,
                double sign) {
  // H_i[4 st + t][8 b + g] staged at hs[i][st][b][g][t] (lane-contiguous fragments)
  __shared__ double2 hs[NB * 256];
  for (int e = threadIdx.x; e < NB * 256; e += k8::kThreads) {
    const int i = e >> 8, p = (e >> 4) & 15, q = e & 15;
    hs[i * 256 + ((p >> 2) * 2 + (q >> 3)) * 32 + (q & 7) * 4 + (p & 3)] = H[e];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t tiles = (n + 7) / 8;
  for (int64_t tile = int64_t(blockIdx.x) * 8 + warp; tile < tiles; tile += int64_t(gridDim.x) * 8) {
    const int64_t row = tile * 8 + g;
    const bool ok = row < n;
    double acc[2][3][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[b][m][0] = acc[b][m][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      double2 xa[4];
#pragma unroll
      for (int st = 0; st < 4; ++st) xa[st] = ok ? k8::ld_widen(X.p[i] + row * 16 + 4 * st + t) : czero<double2>();
#pragma unroll
      for (int st = 0; st < 4; ++st)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const double2 h = hs[i * 256 + (st * 2 + b) * 32 + lane];
          dmma::mma884(acc[b][0][0], acc[b][0][1], xa[st].x, h.x);
          dmma::mma884(acc[b][1][0], acc[b][1][1], xa[st].y, h.y);
          dmma::mma884(acc[b][2][0], acc[b][2][1], xa[st].x + xa[st].y, h.x + h.y);
        }
    }
    if (ok) {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int64_t base = row * 16 + 8 * b + 2 * t;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 y = Yin ? Yin[base + h] : czero<double2>();
          y.x += sign * (acc[b][0][h] - acc[b][1][h]);
          y.y += sign * (acc[b][2][h] - acc[b][0][h] - acc[b][1][h]);
          Yout[base + h] = y;
        }
      }
    }
  }
}

}  // namespace k16
}  // namespace hz
