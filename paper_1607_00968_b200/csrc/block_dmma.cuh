// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) Gram and block-update
// kernels for complex128 blocks with K = 16, 32, 64 columns (included by
// block.cu).
//
// At k >= 16 these tall-skinny products are FP64-bound (8 k^2 flops per
// 32 k bytes per row). B200 has no FP64 tcgen05 kind; its FP64 tensor path
// is DMMA, whose peak (37.1 TF/s measured) equals the DFMA peak (36.5 TF/s,
// scripts/micro/fp64_peak.cu) -- but one DMMA carries 256 FMAs, so the
// kernel is no longer issue-bound the way the FFMA version is. Complex
// products use the 3-multiplication form (3 DMMA per 8x8 complex tile-step):
//   Gram  G = X^H Y : T1 = Xr^T Yr, T2 = Xi^T Yi, T3 = (Xr+Xi)^T (Yr-Yi);
//                     Re = T1 + T2, Im = T1 - T2 - T3
//   Update Y += X C : T1 = Xr Cr, T2 = Xi Ci, T3 = (Xr+Xi)(Cr+Ci);
//                     Re = T1 - T2, Im = T3 - T1 - T2
// m8n8k4 f64 fragments (lane l, g = l >> 2, t = l & 3):
//   A (8x4 row): A[g][t];  B (4x8 col): B[t][g];  C/D: C[g][2t], C[g][2t+1].
#pragma once

#include "block_tiled.cuh"

namespace hz {
namespace dmma {

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- Gram
// CTA = 8 warps = NG row groups x (WP x WQ) warps; warp (group, wp, wq) owns
// the 16 x (8 QT) tile of G at p = 16 wp, q = 8 QT wq for the rows its group
// takes (k-steps of 4 rows, round robin over the staged chunk).
template <int K>
struct GramCfg {
  static constexpr int PT = K >= 16 ? 2 : 1;         // 8-wide p tiles per warp
  static constexpr int WP = K / (8 * PT);            // warps across p
  static constexpr int WQ = K >= 64 ? 2 : (K >= 16 ? K / 16 : 1);  // warps across q
  static constexpr int QT = K / (8 * WQ);            // 8-wide q tiles per warp
  static constexpr int NG = 8 / (WP * WQ);           // row groups
  static constexpr int RC = 32;                      // staged rows per chunk
  // Row stride == 2 (mod 8) complex: a quarter-warp's fragment loads
  // (rows t = 0..3, columns g, g+1) then hit 8 distinct 16-byte bank groups.
  static constexpr int LD = K + 2;
};

template <int K>
__global__ void __launch_bounds__(256)
gram_kernel(int64_t n, const BlockTab<double> X, const double2* __restrict__ Y,
            double2* __restrict__ partials, int nslots) {
  using C = GramCfg<K>;
  constexpr int WP = C::WP, WQ = C::WQ, NG = C::NG, QT = C::QT, RC = C::RC, LD = C::LD;
  constexpr int TILE = RC * LD;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // [2][x|y][RC][K]
  const int i = blockIdx.x, slot = blockIdx.y, nb = gridDim.x;
  const double2* __restrict__ Xi = X.p[i];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp / (WP * WQ), wpq = warp - grp * WP * WQ;
  const int wp = wpq / WQ, wq = wpq - wp * WQ;
  const int g = lane >> 2, t = lane & 3;
  constexpr int PT = C::PT;
  double acc[PT][QT][3][2];
#pragma unroll
  for (int a = 0; a < PT; ++a)
#pragma unroll
    for (int b = 0; b < QT; ++b)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[a][b][m][0] = acc[a][b][m][1] = 0.0;
  const int64_t rows_per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(slot) * rows_per;
  const int64_t r1 = (r0 + rows_per) < n ? (r0 + rows_per) : n;
  const int nchunks = r1 > r0 ? int((r1 - r0 + RC - 1) / RC) : 0;
  auto rows_of = [&](int c) {
    const int64_t c0 = r0 + int64_t(c) * RC;
    return (r1 - c0) < RC ? int(r1 - c0) : RC;
  };
  if (nchunks > 0) {
    tiled::stage_rows<double2, K, RC, LD>(buf, Xi + r0 * K, rows_of(0), tid);
    tiled::stage_rows<double2, K, RC, LD>(buf + TILE, Y + r0 * K, rows_of(0), tid);
  }
  tiled::cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    const int st = c & 1;
    if (c + 1 < nchunks) {
      const int64_t c1 = r0 + int64_t(c + 1) * RC;
      double2* nx = buf + (st ^ 1) * 2 * TILE;
      tiled::stage_rows<double2, K, RC, LD>(nx, Xi + c1 * K, rows_of(c + 1), tid);
      tiled::stage_rows<double2, K, RC, LD>(nx + TILE, Y + c1 * K, rows_of(c + 1), tid);
    }
    tiled::cp_async_commit();
    tiled::cp_async_wait<1>();
    __syncthreads();
    const double2* xs = buf + st * 2 * TILE;
    const double2* ys = xs + TILE;
    // zero-filled tail rows contribute nothing, so every group runs full steps
#pragma unroll 2
    for (int ks = grp; ks < RC / 4; ks += NG) {
      const int r = ks * 4 + t;  // A[g][t] / B[t][g]: row index = t
      double xa[PT][3], yb[QT][3];
#pragma unroll
      for (int a = 0; a < PT; ++a) {
        const double2 x = xs[r * LD + (wp * PT + a) * 8 + g];
        xa[a][0] = x.x;
        xa[a][1] = x.y;
        xa[a][2] = x.x + x.y;
      }
#pragma unroll
      for (int b = 0; b < QT; ++b) {
        const double2 y = ys[r * LD + (wq * QT + b) * 8 + g];
        yb[b][0] = y.x;
        yb[b][1] = y.y;
        yb[b][2] = y.x - y.y;
      }
#pragma unroll
      for (int a = 0; a < PT; ++a)
#pragma unroll
        for (int b = 0; b < QT; ++b)
#pragma unroll
          for (int m = 0; m < 3; ++m) mma884(acc[a][b][m][0], acc[a][b][m][1], xa[a][m], yb[b][m]);
    }
    __syncthreads();
  }
  tiled::cp_async_wait<0>();
  __syncthreads();
  // fixed-order reduction of the row groups through shared memory
  double2* red = buf;  // K*K <= 4*TILE
  for (int gg = 0; gg < NG; ++gg) {
    if (grp == gg) {
#pragma unroll
      for (int a = 0; a < PT; ++a)
#pragma unroll
        for (int b = 0; b < QT; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int p = (wp * PT + a) * 8 + g, q = (wq * QT + b) * 8 + 2 * t + h;
            double2 v;
            v.x = acc[a][b][0][h] + acc[a][b][1][h];
            v.y = acc[a][b][0][h] - acc[a][b][1][h] - acc[a][b][2][h];
            const int e = p * K + q;
            red[e] = gg == 0 ? v : cadd(red[e], v);
          }
    }
    __syncthreads();
  }
  double2* out = partials + (int64_t(slot) * nb + i) * K * K;
  for (int e = tid; e < K * K; e += 256) out[e] = red[e];
}

template <int K>
size_t gram_smem() {
  using C = GramCfg<K>;
  const size_t a = 4 * size_t(C::RC) * C::LD, b = size_t(K) * K;
  return sizeof(double2) * (a > b ? a : b);
}

// ---------------------------------------------------------------- update
// CTA = 8 warps = WR 16-row tiles x WQ column halves; each warp computes a
// 16 x (8 QT) tile over all nb blocks; X_i chunk and C_i are staged
// (double-buffered).
template <int K>
struct UpdateCfg {
  static constexpr int WQ = K >= 32 ? 2 : 1;         // warps across q
  static constexpr int WR = 8 / WQ;                  // 16-row warp tiles
  static constexpr int RC = WR * 16, QT = K / (8 * WQ);
  static constexpr int THREADS = 256;
  // padded strides: A loads (rows g, columns t) want LDX == 4 (mod 8) and
  // B loads (rows t, columns g) want LDH == 2 (mod 8) for conflict-free
  // quarter-warps of 16-byte accesses
  static constexpr int LDX = K + 4;
  static constexpr int LDH = K + 2;
};

template <int K>
__global__ void __launch_bounds__(256)
update_kernel(int64_t n, int nb, const BlockTab<double> X, const double2* __restrict__ H,
              const double2* Yin, double2* Yout, double sign) {
  using C = UpdateCfg<K>;
  constexpr int RC = C::RC, QT = C::QT, LDX = C::LDX, WQ = C::WQ, NT = C::THREADS;
  constexpr int LDH = C::LDH;
  constexpr int XT = RC * LDX, HT = K * LDH, STAGE = XT + HT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr = warp / WQ, wq = warp - wr * WQ;
  const int64_t c0 = int64_t(blockIdx.x) * RC;
  const int rows = (n - c0) < RC ? int(n - c0) : RC;
  double acc[2][QT][3][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < QT; ++b)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[a][b][m][0] = acc[a][b][m][1] = 0.0;
  auto stage = [&](int i, double2* dst) {
    const double2* src = X.p[i] + c0 * K;
    constexpr int CH = K;  // 16-byte chunks per row (c128)
    for (int e = tid; e < RC * CH; e += NT) {
      const int r = e / CH, cc = e - r * CH;
      double2* d = dst + r * LDX + cc;
      if (r < rows)
        tiled::cp_async16(d, src + int64_t(r) * K + cc);
      else
        *d = czero<double2>();
    }
    const double2* hsrc = H + int64_t(i) * K * K;
    for (int e = tid; e < K * K; e += NT) {
      const int p = e / K, q = e - p * K;
      tiled::cp_async16(dst + XT + p * LDH + q, hsrc + e);
    }
  };
  if (nb > 0) stage(0, buf);
  tiled::cp_async_commit();
  for (int i = 0; i < nb; ++i) {
    const int st = i & 1;
    if (i + 1 < nb) stage(i + 1, buf + (st ^ 1) * STAGE);
    tiled::cp_async_commit();
    tiled::cp_async_wait<1>();
    __syncthreads();
    const double2* xs = buf + st * STAGE + wr * 16 * LDX;
    const double2* hs = buf + st * STAGE + XT;
#pragma unroll 2
    for (int p0 = 0; p0 < K; p0 += 4) {
      double xa[2][3], hb[QT][3];
#pragma unroll
      for (int a = 0; a < 2; ++a) {  // A[g][t] = X[row a*8+g][p0+t]
        const double2 x = xs[(a * 8 + g) * LDX + p0 + t];
        xa[a][0] = x.x;
        xa[a][1] = x.y;
        xa[a][2] = x.x + x.y;
      }
#pragma unroll
      for (int b = 0; b < QT; ++b) {  // B[t][g] = C[p0+t][b*8+g]
        const double2 h = hs[(p0 + t) * LDH + (wq * QT + b) * 8 + g];
        hb[b][0] = h.x;
        hb[b][1] = h.y;
        hb[b][2] = h.x + h.y;
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < QT; ++b)
#pragma unroll
          for (int m = 0; m < 3; ++m) mma884(acc[a][b][m][0], acc[a][b][m][1], xa[a][m], hb[b][m]);
    }
    __syncthreads();
  }
  tiled::cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int rl = wr * 16 + a * 8 + g;
    if (rl >= rows) continue;
    const int64_t base = (c0 + rl) * K;
#pragma unroll
    for (int b = 0; b < QT; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = (wq * QT + b) * 8 + 2 * t + h;
        double2 y = Yin ? Yin[base + q] : czero<double2>();
        y.x += sign * (acc[a][b][0][h] - acc[a][b][1][h]);
        y.y += sign * (acc[a][b][2][h] - acc[a][b][0][h] - acc[a][b][1][h]);
        Yout[base + q] = y;
      }
  }
}

template <int K>
size_t update_smem() {
  using C = UpdateCfg<K>;
  return sizeof(double2) * 2 * (size_t(C::RC) * C::LDX + size_t(K) * C::LDH);
}

}  // namespace dmma
}  // namespace hz
