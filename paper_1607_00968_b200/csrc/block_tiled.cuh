// Tiled Gram / block-update kernels for the common block widths K = 16, 32,
// 64 (included by block.cu).
//
// At k >= 16 a complex128 Gram X^H Y or update Y -= X H is FP64-FMA bound,
// not HBM bound (8 k^2 flops per 32 k bytes per row). Both kernels
//  * stream row chunks of the blocks into shared memory with cp.async
//    (LDGSTS), double-buffered so the next chunk's loads overlap this chunk's
//    FMAs;
//  * give each thread a register tile whose columns are STRIDED
//    (q = qt + NQ*b), so a warp's shared loads are contiguous or broadcast
//    (one wavefront); update rows are padded by one element so the
//    row-strided reads of a warp fall in distinct banks;
//  * use the 3-multiplication complex product: 3 FMAs per complex
//    multiply-add instead of 4.
//   Gram  G_pq = sum conj(x_p) y_q : T1 = sum xr yr, T2 = sum xi yi,
//         T3 = sum (xr + xi)(yr - yi);  Re = T1 + T2, Im = T1 - T2 - T3.
//   Update y_q += sum x_p h_pq     : T1 = sum xr hr, T2 = sum xi hi,
//         T3 = sum (xr + xi)(hr + hi); Re = T1 - T2, Im = T3 - T1 - T2.
#pragma once

#include "kernels.hpp"

namespace hz {
namespace tiled {

// 16-byte asynchronous global -> shared copy (sm_80+ LDGSTS)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy `rows` rows of K complex values (contiguous in global) into a padded
// shared tile [RC][LD]; rows >= `rows` are zero-filled with plain stores.
template <class V, int K, int RC, int LD>
__device__ __forceinline__ void stage_rows(V* dst, const V* src, int rows, int tid) {
  constexpr int PER16 = 16 / sizeof(V);  // complex values per 16 bytes (1 c128, 2 c64)
  constexpr int CH = K / PER16;          // 16-byte chunks per row
#pragma unroll 4
  for (int e = tid; e < RC * CH; e += 256) {
    const int r = e / CH, c = (e - r * CH) * PER16;
    V* d = dst + r * LD + c;
    if (r < rows) {
      cp_async16(d, src + int64_t(r) * K + c);
    } else {
#pragma unroll
      for (int u = 0; u < PER16; ++u) d[u] = czero<V>();
    }
  }
}

template <int K>
struct GramShape {
  static constexpr int TP = K == 64 ? 4 : 2;  // p per thread
  static constexpr int TQ = 4;                // q per thread
  static constexpr int NTP = K / TP, NTQ = K / TQ;
  static constexpr int G1 = NTP * NTQ;        // threads per row group
  static constexpr int NG = 256 / G1;         // row groups per CTA
  static constexpr int RC = 32;               // staged rows per chunk
  static constexpr int LD = K;                // a warp reads one row: no padding
};

// CTA (i = blockIdx.x, slot = blockIdx.y) writes the slot's partial of
// X_i^H Y over its row range into partials[slot][i].
template <class T, int K>
__global__ void __launch_bounds__(256)
gram_kernel(int64_t n, const BlockTab<T> X, const cplx_t<T>* __restrict__ Y,
            cplx_t<T>* __restrict__ partials, int nslots) {
  using V = cplx_t<T>;
  using S = GramShape<K>;
  constexpr int TP = S::TP, TQ = S::TQ, NTP = S::NTP, NTQ = S::NTQ, G1 = S::G1, NG = S::NG;
  constexpr int RC = S::RC, LD = S::LD, TILE = RC * LD;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);  // [2 stages][x | y][RC][LD]
  const int i = blockIdx.x, slot = blockIdx.y, nb = gridDim.x;
  const V* __restrict__ Xi = X.p[i];
  const int tid = threadIdx.x, g = tid / G1, t = tid - g * G1;
  const int pt = t / NTQ, qt = t - pt * NTQ;
  T t1[TP][TQ], t2[TP][TQ], t3[TP][TQ];
#pragma unroll
  for (int a = 0; a < TP; ++a)
#pragma unroll
    for (int b = 0; b < TQ; ++b) t1[a][b] = t2[a][b] = t3[a][b] = T(0);
  const int64_t rows_per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(slot) * rows_per;
  const int64_t r1 = (r0 + rows_per) < n ? (r0 + rows_per) : n;
  const int nchunks = r1 > r0 ? int((r1 - r0 + RC - 1) / RC) : 0;
  auto rows_of = [&](int c) {
    const int64_t c0 = r0 + int64_t(c) * RC;
    return (r1 - c0) < RC ? int(r1 - c0) : RC;
  };
  if (nchunks > 0) {
    stage_rows<V, K, RC, LD>(buf, Xi + r0 * K, rows_of(0), tid);
    stage_rows<V, K, RC, LD>(buf + TILE, Y + r0 * K, rows_of(0), tid);
  }
  cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    const int st = c & 1;
    if (c + 1 < nchunks) {  // prefetch the next chunk into the other stage
      const int64_t c1 = r0 + int64_t(c + 1) * RC;
      V* nx = buf + (st ^ 1) * 2 * TILE;
      stage_rows<V, K, RC, LD>(nx, Xi + c1 * K, rows_of(c + 1), tid);
      stage_rows<V, K, RC, LD>(nx + TILE, Y + c1 * K, rows_of(c + 1), tid);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const V* xs = buf + st * 2 * TILE;
    const V* ys = xs + TILE;
    const int rows = rows_of(c);
    if (g < NG) {
      for (int r = g; r < rows; r += NG) {
        V xa[TP], yb[TQ];
#pragma unroll
        for (int a = 0; a < TP; ++a) xa[a] = xs[r * LD + pt + NTP * a];
#pragma unroll
        for (int b = 0; b < TQ; ++b) yb[b] = ys[r * LD + qt + NTQ * b];
        T yd[TQ];
#pragma unroll
        for (int b = 0; b < TQ; ++b) yd[b] = yb[b].x - yb[b].y;
#pragma unroll
        for (int a = 0; a < TP; ++a) {
          const T xsum = xa[a].x + xa[a].y;
#pragma unroll
          for (int b = 0; b < TQ; ++b) {
            t1[a][b] = fma(xa[a].x, yb[b].x, t1[a][b]);
            t2[a][b] = fma(xa[a].y, yb[b].y, t2[a][b]);
            t3[a][b] = fma(xsum, yd[b], t3[a][b]);
          }
        }
      }
    }
    __syncthreads();  // stage st is overwritten by the prefetch two chunks on
  }
  cp_async_wait<0>();
  __syncthreads();
  // fixed-order reduction of the row groups (deterministic)
  V* red = buf;  // K*K <= 4*RC*LD
  for (int gg = 0; gg < NG; ++gg) {
    if (g == gg) {
#pragma unroll
      for (int a = 0; a < TP; ++a)
#pragma unroll
        for (int b = 0; b < TQ; ++b) {
          V v;
          v.x = t1[a][b] + t2[a][b];
          v.y = t1[a][b] - t2[a][b] - t3[a][b];
          const int e = (pt + NTP * a) * K + qt + NTQ * b;
          red[e] = gg == 0 ? v : cadd(red[e], v);
        }
    }
    __syncthreads();
  }
  V* out = partials + (int64_t(slot) * nb + i) * K * K;
  for (int e = tid; e < K * K; e += 256) out[e] = red[e];
}

template <int K>
struct UpdateShape {
  static constexpr int TQ = 4, NQ = K / TQ;   // q per thread (strided by NQ)
  static constexpr int TR = 2;                // rows per thread
  static constexpr int NR = 256 / NQ;         // row tiles
  static constexpr int RC = TR * NR;          // rows per CTA
  static constexpr int LD = K + 2;            // padded (16 B multiple for c64 too)
};

// Yout = (Yin ? Yin : 0) + sign * sum_i X_i H_i over one RC-row chunk; the
// X_i chunk and H_i of block i + 1 are prefetched while block i computes.
template <class T, int K>
__global__ void __launch_bounds__(256)
update_kernel(int64_t n, int nb, const BlockTab<T> X, const cplx_t<T>* __restrict__ H,
              const cplx_t<T>* Yin, cplx_t<T>* Yout, T sign) {
  using V = cplx_t<T>;
  using S = UpdateShape<K>;
  constexpr int TQ = S::TQ, NQ = S::NQ, TR = S::TR, RC = S::RC, LD = S::LD;
  constexpr int XT = RC * LD, HT = K * K, STAGE = XT + HT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);  // [2][X chunk | H]
  const int tid = threadIdx.x, qt = tid % NQ, rt = tid / NQ;
  const int rr = rt * TR;
  const int64_t c0 = int64_t(blockIdx.x) * RC;
  const int rows = (n - c0) < RC ? int(n - c0) : RC;
  T t1[TR][TQ], t2[TR][TQ], t3[TR][TQ];
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TQ; ++b) t1[a][b] = t2[a][b] = t3[a][b] = T(0);
  auto stage = [&](int i, V* dst) {
    stage_rows<V, K, RC, LD>(dst, X.p[i] + c0 * K, rows, tid);
    stage_rows<V, K, K, K>(dst + XT, H + int64_t(i) * K * K, K, tid);
  };
  if (nb > 0) stage(0, buf);
  cp_async_commit();
  for (int i = 0; i < nb; ++i) {
    const int st = i & 1;
    if (i + 1 < nb) stage(i + 1, buf + (st ^ 1) * STAGE);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const V* xs = buf + st * STAGE;
    const V* hs = xs + XT;
#pragma unroll 4
    for (int p = 0; p < K; ++p) {
      V hv[TQ];
      T hvs[TQ];
#pragma unroll
      for (int b = 0; b < TQ; ++b) {
        hv[b] = hs[p * K + qt + NQ * b];
        hvs[b] = hv[b].x + hv[b].y;
      }
#pragma unroll
      for (int a = 0; a < TR; ++a) {
        const V xv = xs[(rr + a) * LD + p];
        const T xsum = xv.x + xv.y;
#pragma unroll
        for (int b = 0; b < TQ; ++b) {
          t1[a][b] = fma(xv.x, hv[b].x, t1[a][b]);
          t2[a][b] = fma(xv.y, hv[b].y, t2[a][b]);
          t3[a][b] = fma(xsum, hvs[b], t3[a][b]);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int a = 0; a < TR; ++a) {
    if (rr + a >= rows) continue;
    const int64_t base = (c0 + rr + a) * K;
#pragma unroll
    for (int b = 0; b < TQ; ++b) {
      const int q = qt + NQ * b;
      V y = Yin ? Yin[base + q] : czero<V>();
      y.x += sign * (t1[a][b] - t2[a][b]);
      y.y += sign * (t3[a][b] - t1[a][b] - t2[a][b]);
      Yout[base + q] = y;
    }
  }
}

template <class T, int K>
size_t gram_smem() {
  using S = GramShape<K>;
  const size_t a = 4 * size_t(S::RC) * S::LD, b = size_t(K) * K;
  return sizeof(cplx_t<T>) * (a > b ? a : b);
}

template <class T, int K>
size_t update_smem() {
  using S = UpdateShape<K>;
  return sizeof(cplx_t<T>) * 2 * (size_t(S::RC) * S::LD + size_t(K) * K);
}

template <int K>
constexpr int update_rows() {
  return UpdateShape<K>::RC;
}

}  // namespace tiled
}  // namespace hz
