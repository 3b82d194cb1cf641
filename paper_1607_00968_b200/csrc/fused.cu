// Fused finest-level smoothing of a V(2,2) visit on a 2D grid: temporal
// blocking of the two pre-smoothing sweeps, the residual and the restriction
// (one kernel) and of the prolongated correction and the two post-smoothing
// sweeps (one kernel), so level 0 streams its right-hand side and iterate a
// few times per cycle instead of once per sweep.
//
// Unfused (src/multigrid.cpp:119-136,162-199, per element of the c64 cycle
// of a c128 block): zero-start sweep 32 B, sweep 24 B, residual 24 B,
// restriction 10 B, prolongation 18 B, sweep 24 B, last sweep 32 B = 164 B.
// Fused: pre reads b (16 B) and writes x (8 B) + the coarse right-hand side
// (2 B); post reads x (8 B), b (16 B), the coarse correction (2 B) and writes
// the result (16 B): 66 B per element.
//
// Mapping. A CTA owns a strip of W fine columns (i), C RHS columns and a
// chunk of rows (j); it streams the rows of its strip in ascending j and
// keeps the last three rows of every intermediate (x1, x2, r; x3, x4) in
// shared-memory rings. Each stage recomputes a halo that shrinks by one node
// per stage (3 for pre, 2 for post), and each CTA re-derives the few rows
// above its chunk. A thread owns one 16-byte unit of a node's columns (2
// complex64 / 1 complex128 values): rings are [row][thread] arrays of
// 16-byte units (conflict-free), and global row accesses are contiguous
// 16-byte runs per node. The next row's global loads are issued before the
// current row's stages (register prefetch).
//
// Every value is computed by exactly the per-element expressions of the
// unfused kernels (stencil.cu: jacobi_zero[_cast], fine MODE 2 / MODE 1 in
// Csr::mul_block order, restrict, prolong-correct, jacobi_out64), so the
// fused cycle is bitwise equal to the unfused one (tested).
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "profile.hpp"
#include "tma.cuh"

namespace hz {

namespace {

// complex values per 16-byte unit
template <class T>
constexpr int cpt() {
  return sizeof(T) == 4 ? 2 : 1;
}

// QU complex values per thread unit (cpt<T>() = one 16-byte vector; 4 for
// complex64 = two vectors, for narrow blocks: twice the columns per thread
// amortise the per-row index math, barriers and per-node coefficients)
template <class T, int QU = cpt<T>()>
struct Unit {
  cplx_t<T> v[QU];
};

// one unit of consecutive columns from global memory (read-only path); In
// may be wider than T (complex128 right-hand side of the c64 cycle)
template <class V, int N>
__device__ __forceinline__ void gload(const V* __restrict__ p, V (&v)[N]) {
  if constexpr (sizeof(V) == 8 && N % 2 == 0) {
#pragma unroll
    for (int h = 0; h < N / 2; ++h) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p) + h);
      v[2 * h] = make_float2(a.x, a.y);
      v[2 * h + 1] = make_float2(a.z, a.w);
    }
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = __ldg(p + c);
  }
}
template <class V, int N>
__device__ __forceinline__ void gstore(V* p, const V (&v)[N]) {
  if constexpr (sizeof(V) == 8 && N % 2 == 0) {
#pragma unroll
    for (int h = 0; h < N / 2; ++h)
      reinterpret_cast<float4*>(p)[h] = make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) p[c] = v[c];
  }
}

// (A u)[centre] of the fine 5-point operator in Csr::mul_block order
// (j-, i-, centre, i+, j+; inc/csr.hpp:43-53); a missing neighbour is
// skipped, as in fine_v4_kernel.
template <class V, class T>
__device__ __forceinline__ V ax_csr(const V& c, T wx, T wy, bool xm, bool xp, bool ym, bool yp, const V& um,
                                    const V& uxm, const V& u0, const V& uxp, const V& up) {
  V acc = czero<V>();
  if (ym) acc = crfma(wy, um, acc);
  if (xm) acc = crfma(wx, uxm, acc);
  acc = cfma(c, u0, acc);
  if (xp) acc = crfma(wx, uxp, acc);
  if (yp) acc = crfma(wy, up, acc);
  return acc;
}

// One stencil row from a ring (rows rm, r0, rp; [thread] units) at thread
// index t (TPN threads per node): MODE 1: o = b - A u; MODE 2:
// o = u + d (b - A u)  (d = wD^{-1}).
template <int TPN, int MODE, class T, int QU>
__device__ __forceinline__ void ring_stencil(const Unit<T, QU>* rm, const Unit<T, QU>* r0, const Unit<T, QU>* rp,
                                             int t, const cplx_t<T>& c, const cplx_t<T>& d, T wx, T wy, bool xm,
                                             bool xp, bool ym, bool yp, const Unit<T, QU>& b, Unit<T, QU>& o) {
  const Unit<T, QU> u0 = r0[t];
  const Unit<T, QU> uxm = xm ? r0[t - TPN] : u0, uxp = xp ? r0[t + TPN] : u0;
  const Unit<T, QU> um = ym ? rm[t] : u0, up = yp ? rp[t] : u0;
#pragma unroll
  for (int q = 0; q < QU; ++q) {
    const auto a = ax_csr(c, wx, wy, xm, xp, ym, yp, um.v[q], uxm.v[q], u0.v[q], uxp.v[q], up.v[q]);
    o.v[q] = MODE == 1 ? csub(b.v[q], a) : cadd(u0.v[q], cmul(d, csub(b.v[q], a)));
  }
}

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem));
}
template <class V>
__device__ __forceinline__ void cpa(V* smem, const V* gmem) {
  if constexpr (sizeof(V) == 8)
    cpa8(smem, gmem);
  else
    cpa16(smem, gmem);
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Shared-memory plan of the streaming kernels. Rings: 3 rows x TH units per
// intermediate. Staging (cp.async, PD rows in flight): per row and thread
// its 16-byte units of each streamed input plus the node's centre and
// wD^{-1} (each thread stages its own copies, so a row is usable after the
// thread's own cp.async.wait -- no barrier).
template <class T, class In, int TPN, int NT, int PD, int QU>
struct PrePlan {
  static constexpr int Q = QU, TH = NT * TPN;
  static constexpr int UIN = int(sizeof(In)) * Q / 16;  // b units per thread
  static constexpr size_t RINGS = size_t(7) * TH * sizeof(Unit<T, QU>);
  static constexpr size_t SLOT = size_t(TH) * (UIN * 16 + 2 * sizeof(cplx_t<T>));
  static constexpr size_t BYTES = RINGS + PD * SLOT;
};
template <class T, class In, int TPN, int NT, int PD, int QU>
struct PostPlan {
  static constexpr int Q = QU, TH = NT * TPN;
  static constexpr int UIN = int(sizeof(In)) * Q / 16;
  static constexpr int XU = int(sizeof(Unit<T, QU>)) / 16;  // 16-byte vectors per unit
  static constexpr int NCN = NT / 2 + 1;  // coarse nodes under a strip
  static constexpr int CS = PD / 2 + 3;   // coarse-row ring slots
  static constexpr size_t RINGS = size_t(6) * TH * sizeof(Unit<T, QU>);
  static constexpr size_t SLOT = size_t(TH) * (XU * 16 + UIN * 16 + 2 * sizeof(cplx_t<T>));
  static constexpr size_t COARSE = size_t(CS) * NCN * TPN * sizeof(Unit<T, QU>);
  static constexpr size_t BYTES = RINGS + PD * SLOT + COARSE;
};

// Pre-smoothing of a zero-start visit: x1 = wD^{-1} b, x2 = x1 + wD^{-1}(b - A x1),
// r = b - A x2, rc = P^T r. Strip: W = NT - 6 fine columns (halo 3 each side),
// coarse columns [CX0, CX0 + W/2); chunk: coarse rows [CY0, CY0 + crows).
template <class T, class In, int TPN, int NT, int PD, int MINB, int QU>
__global__ void __launch_bounds__(NT * TPN, MINB)
fused_pre_kernel(LevelOp<T> op, LevelGeom gc, T wj, const In* __restrict__ b, cplx_t<T>* __restrict__ x2out,
                 cplx_t<T>* __restrict__ rc, int crows) {
  using V = cplx_t<T>;
  using U = Unit<T, QU>;
  using P = PrePlan<T, In, TPN, NT, PD, QU>;
  constexpr int Q = P::Q, TH = P::TH, UIN = P::UIN, W = NT - 6, TC = W / 2;
  extern __shared__ __align__(16) unsigned char smraw[];
  U* x1s = reinterpret_cast<U*>(smraw);  // [3][TH]
  U* x2s = x1s + 3 * TH;                 // [3][TH]
  U* rs = x2s + 3 * TH;                  // [TH]
  uint4* bst = reinterpret_cast<uint4*>(smraw + P::RINGS);     // [PD][UIN][TH]
  V* cds = reinterpret_cast<V*>(bst + size_t(PD) * UIN * TH);  // [PD][2][TH]
  const int n0 = int(op.g.n0), n1 = int(op.g.n1), k = int(op.g.k);
  const int t = threadIdx.x, xs = t / TPN;
  const int CX0 = blockIdx.x * TC, X0 = 2 * CX0;
  const int gx = X0 - 3 + xs;
  const int col = (blockIdx.y * TPN + t % TPN) * Q;
  const int CY0 = blockIdx.z * crows, CY1 = min(CY0 + crows, int(gc.n1));
  const int Y0 = 2 * CY0, Y1 = 2 * CY1;  // fine rows owned: [Y0, min(Y1, n1))
  const bool inx = gx >= 0 && gx < n0;
  const bool xm = gx > 0, xp = gx + 1 < n0;
  const bool own_x = inx && gx >= X0 && gx < X0 + W;
  const T wx = op.w[0], wy = op.w[1];
  // restriction role: coarse column I = CX0 + ci, fine 2I at strip node 2ci + 3
  const int ci = t / TPN, I = CX0 + ci;
  const bool rest = t < TC * TPN && I < int(gc.n0);
  const int rt = (2 * ci + 3) * TPN + t % TPN;
  const bool rxm = 2 * I - 1 >= 0, rxp = 2 * I + 1 < n0;

  // register FIFOs: b, centre and wD^{-1} of rows j-1, j-2
  U b1, b2, acc;
  V c1 = czero<V>(), c2 = czero<V>(), d1 = czero<V>();
#pragma unroll
  for (int q = 0; q < Q; ++q) acc.v[q] = b1.v[q] = b2.v[q] = czero<V>();

  const int jbeg = max(Y0 - 3, 0), jend = min(Y1 + 1, n1 + 1);
  const char* bp = reinterpret_cast<const char*>(b + int64_t(max(gx, 0)) * k + col);
  const int64_t bstride = int64_t(n0) * k * sizeof(In);
  auto issue = [&](int j) {
    if (inx && j < n1 && j <= jend) {
      const int sl = j % PD;
#pragma unroll
      for (int u = 0; u < UIN; ++u) cpa16(bst + (sl * UIN + u) * TH + t, bp + j * bstride + 16 * u);
      const int64_t node = int64_t(gx) + int64_t(n0) * j;
      cpa(cds + (sl * 2) * TH + t, op.center + node);
      cpa(cds + (sl * 2 + 1) * TH + t, op.inv_diag + node);
    }
    cpa_commit();
  };
#pragma unroll
  for (int p = 0; p < PD - 1; ++p) issue(jbeg + p);
  for (int j = jbeg; j <= jend; ++j) {
    issue(j + PD - 1);
    cpa_wait<PD - 1>();
    // (a) x1 row j
    U b0;
    const int sl = j % PD;
    const V c0 = cds[(sl * 2) * TH + t], draw = cds[(sl * 2 + 1) * TH + t];
    const V d0 = mk(wj * draw.x, wj * draw.y);
    if (inx && j < n1) {
      In braw[Q];
      {
        uint4 raw[UIN];
#pragma unroll
        for (int u = 0; u < UIN; ++u) raw[u] = bst[(sl * UIN + u) * TH + t];
        memcpy(braw, raw, sizeof(braw));
      }
      U x1;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        b0.v[q] = ccast<V>(braw[q]);
        x1.v[q] = cmul(d0, b0.v[q]);
      }
      x1s[(j % 3) * TH + t] = x1;
    }
    __syncthreads();
    // (b) x2 row y = j - 1 on strip nodes [1, NT-2]
    {
      const int y = j - 1;
      if (inx && y >= 0 && y >= Y0 - 2 && y < n1 && xs >= 1 && xs <= NT - 2) {
        U o;
        ring_stencil<TPN, 2>(x1s + ((y + 2) % 3) * TH, x1s + (y % 3) * TH, x1s + ((y + 1) % 3) * TH, t, c1, d1,
                             wx, wy, xm, xp, y > 0, y + 1 < n1, b1, o);
        x2s[(y % 3) * TH + t] = o;
        if (own_x && y >= Y0 && y < Y1) gstore(x2out + (int64_t(gx) + int64_t(n0) * y) * k + col, o.v);
      }
    }
    __syncthreads();
    // (c) r row y = j - 2 on strip nodes [2, NT-3]
    const int y = j - 2;
    const bool ry = y >= 0 && y >= Y0 - 1 && y < n1 && y < Y1;
    if (inx && ry && xs >= 2 && xs <= NT - 3) {
      U o;
      ring_stencil<TPN, 1>(x2s + ((y + 2) % 3) * TH, x2s + (y % 3) * TH, x2s + ((y + 1) % 3) * TH, t, c2, d1, wx,
                           wy, xm, xp, y > 0, y + 1 < n1, b2, o);
      rs[t] = o;
    }
    __syncthreads();
    // (d) restriction: fine row y adds to coarse row(s) in ascending fine
    // order (restrict_kernel: ey, then ex ascending; zero weights skipped)
    if (rest && ry) {
      U rv0 = rs[rt], rvm = rv0, rvp = rv0;
      if (rxm) rvm = rs[rt - TPN];
      if (rxp) rvp = rs[rt + TPN];
      const T h = T(0.5), one = T(1);
      if (y & 1) {
        // last row (ey = +1) of coarse row (y-1)/2, first row (ey = -1) of (y+1)/2
        const int J = (y - 1) >> 1;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          V a = acc.v[q];
          if (rxm) a = crfma(h * h, rvm.v[q], a);
          a = crfma(one * h, rv0.v[q], a);
          if (rxp) a = crfma(h * h, rvp.v[q], a);
          acc.v[q] = a;
        }
        if (J >= CY0 && J < CY1) gstore(rc + (int64_t(I) + int64_t(gc.n0) * J) * k + col, acc.v);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          V a = czero<V>();
          if (rxm) a = crfma(h * h, rvm.v[q], a);
          a = crfma(one * h, rv0.v[q], a);
          if (rxp) a = crfma(h * h, rvp.v[q], a);
          acc.v[q] = a;
        }
      } else {
        const int J = y >> 1;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          V a = acc.v[q];
          if (rxm) a = crfma(h * one, rvm.v[q], a);
          a = crfma(one * one, rv0.v[q], a);
          if (rxp) a = crfma(h * one, rvp.v[q], a);
          acc.v[q] = a;
        }
        if (y == n1 - 1 && J >= CY0 && J < CY1) gstore(rc + (int64_t(I) + int64_t(gc.n0) * J) * k + col, acc.v);
      }
    }
    // shift the FIFOs (row j -> j-1 -> j-2)
    b2 = b1;
    b1 = b0;
    c2 = c1;
    c1 = c0;
    d1 = d0;
  }
  cpa_wait<0>();
}

// Post-smoothing: x3 = x2 + P ec, x4 = x3 + wD^{-1}(b - A x3),
// out = (Out)(x4 + wD^{-1}(b - A x4)). Strip: W = NT - 4 fine columns (halo 2);
// chunk: fine rows [Y0, Y0 + frows). The coarse correction rows under the
// strip are staged too (coarse row J with fine row 2J-2, so the barrier of
// that row publishes it before its first use by fine row 2J-1).
template <class T, class In, class Out, int TPN, int NT, int PD, int MINB, int QU>
__global__ void __launch_bounds__(NT * TPN, MINB)
fused_post_kernel(LevelOp<T> op, LevelGeom gc, T wj, const cplx_t<T>* __restrict__ x2,
                  const cplx_t<T>* __restrict__ ec, const In* __restrict__ b, Out* __restrict__ out, int frows) {
  using V = cplx_t<T>;
  using U = Unit<T, QU>;
  using P = PostPlan<T, In, TPN, NT, PD, QU>;
  constexpr int Q = P::Q, TH = P::TH, UIN = P::UIN, W = NT - 4, NCN = P::NCN, CS = P::CS, XU = P::XU;
  extern __shared__ __align__(16) unsigned char smraw[];
  U* x3s = reinterpret_cast<U*>(smraw);  // [3][TH]
  U* x4s = x3s + 3 * TH;                 // [3][TH]
  uint4* xst = reinterpret_cast<uint4*>(smraw + P::RINGS);     // [PD][XU][TH]
  uint4* bst = xst + size_t(PD) * XU * TH;                     // [PD][UIN][TH]
  V* cds = reinterpret_cast<V*>(bst + size_t(PD) * UIN * TH);  // [PD][2][TH]
  U* ecs = reinterpret_cast<U*>(smraw + P::RINGS + PD * P::SLOT);  // [CS][NCN * TPN]
  const int n0 = int(op.g.n0), n1 = int(op.g.n1), k = int(op.g.k);
  const int t = threadIdx.x, xs = t / TPN, cg = t % TPN;
  const int X0 = blockIdx.x * W;
  const int gx = X0 - 2 + xs;
  const int col = (blockIdx.y * TPN + cg) * Q;
  const int Y0 = blockIdx.z * frows, Y1 = min(Y0 + frows, n1);
  const bool inx = gx >= 0 && gx < n0;
  const bool xm = gx > 0, xp = gx + 1 < n0;
  const bool own_x = inx && gx >= X0 && gx < X0 + W;
  const T wx = op.w[0], wy = op.w[1];
  // prolongation parents along i (prolong_v4_kernel), as staged-row indices
  const int cxa = (X0 >> 1) - 1;
  const uint32_t ui = uint32_t(max(gx, 0));
  const int p0 = (int(ui >> 1) - cxa) * TPN + cg, p1 = (int((ui + 1) >> 1) - cxa) * TPN + cg;
  const T wx0 = (ui & 1u) ? T(0.5) : T(1), wx1 = (ui & 1u) ? T(0.5) : T(0);

  U b1, b2;
  V c1 = czero<V>(), c2 = czero<V>(), d1 = czero<V>(), d2 = czero<V>();
#pragma unroll
  for (int q = 0; q < Q; ++q) b1.v[q] = b2.v[q] = czero<V>();

  const int jbeg = max(Y0 - 2, 0), jend = Y1 + 1;
  const int64_t rstride = int64_t(n0) * k;
  const V* xp2 = x2 + int64_t(max(gx, 0)) * k + col;
  const char* bp = reinterpret_cast<const char*>(b + int64_t(max(gx, 0)) * k + col);
  // one coarse row of the strip: NCN nodes x TPN units, one unit per thread
  auto issue_coarse = [&](int J) {
    if (J < int(gc.n1) && t < NCN * TPN) {
      const int cx = cxa + t / TPN;
      if (cx >= 0 && cx < int(gc.n0)) {
        char* dst = reinterpret_cast<char*>(ecs + (J % CS) * (NCN * TPN) + t);
        const char* src =
            reinterpret_cast<const char*>(ec + (int64_t(cx) + int64_t(gc.n0) * J) * k + (blockIdx.y * TPN + t % TPN) * Q);
#pragma unroll
        for (int u = 0; u < XU; ++u) cpa16(dst + 16 * u, src + 16 * u);
      }
    }
  };
  auto issue = [&](int j) {
    if (j <= jend && j < n1) {
      const int sl = j % PD;
      if (inx) {
#pragma unroll
        for (int u = 0; u < XU; ++u)
          cpa16(xst + (sl * XU + u) * TH + t, reinterpret_cast<const char*>(xp2 + j * rstride) + 16 * u);
#pragma unroll
        for (int u = 0; u < UIN; ++u)
          cpa16(bst + (sl * UIN + u) * TH + t, bp + j * rstride * int64_t(sizeof(In)) + 16 * u);
        const int64_t node = int64_t(gx) + int64_t(n0) * j;
        cpa(cds + (sl * 2) * TH + t, op.center + node);
        cpa(cds + (sl * 2 + 1) * TH + t, op.inv_diag + node);
      }
      if (!(j & 1) && (j >> 1) + 1 >= (jbeg >> 1) + 2) issue_coarse((j >> 1) + 1);
    }
    cpa_commit();
  };
  issue_coarse(jbeg >> 1);
  issue_coarse((jbeg >> 1) + 1);
  cpa_commit();
  cpa_wait<0>();
  __syncthreads();
#pragma unroll
  for (int p = 0; p < PD - 1; ++p) issue(jbeg + p);
  for (int j = jbeg; j <= jend; ++j) {
    issue(j + PD - 1);
    cpa_wait<PD - 1>();
    // (a) x3 row j
    U b0;
    const int sl = j % PD;
    const V c0 = cds[(sl * 2) * TH + t], draw = cds[(sl * 2 + 1) * TH + t];
    const V d0 = mk(wj * draw.x, wj * draw.y);
    if (inx && j < n1) {
      const uint32_t uj = uint32_t(j);
      const U* er0 = ecs + int((uj >> 1) % CS) * (NCN * TPN);
      const U* er1 = ecs + int(((uj + 1) >> 1) % CS) * (NCN * TPN);
      const T wy0 = (uj & 1u) ? T(0.5) : T(1), wy1 = (uj & 1u) ? T(0.5) : T(0);
      const T w00 = wx0 * wy0 * T(1), w01 = wx1 * wy0 * T(1), w10 = wx0 * wy1 * T(1), w11 = wx1 * wy1 * T(1);
      const U e00 = er0[p0], e01 = er0[p1], e10 = er1[p0], e11 = er1[p1];
      U xr;
      In braw[Q];
      {
        uint4 a[XU];
#pragma unroll
        for (int u = 0; u < XU; ++u) a[u] = xst[(sl * XU + u) * TH + t];
        memcpy(&xr, a, sizeof(xr));
        uint4 raw[UIN];
#pragma unroll
        for (int u = 0; u < UIN; ++u) raw[u] = bst[(sl * UIN + u) * TH + t];
        memcpy(braw, raw, sizeof(braw));
      }
      U x3;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        // parents in (y, x) ascending order, zero weights skipped
        V corr = czero<V>();
        corr = crfma(w00, e00.v[q], corr);
        if (w01 != T(0)) corr = crfma(w01, e01.v[q], corr);
        if (w10 != T(0)) corr = crfma(w10, e10.v[q], corr);
        if (w11 != T(0)) corr = crfma(w11, e11.v[q], corr);
        x3.v[q] = cadd(xr.v[q], corr);
        b0.v[q] = ccast<V>(braw[q]);
      }
      x3s[(j % 3) * TH + t] = x3;
    }
    __syncthreads();
    // (b) x4 row y = j - 1 on strip nodes [1, NT-2]
    {
      const int y = j - 1;
      if (inx && y >= 0 && y >= Y0 - 1 && y < n1 && y <= Y1 && xs >= 1 && xs <= NT - 2) {
        U o;
        ring_stencil<TPN, 2>(x3s + ((y + 2) % 3) * TH, x3s + (y % 3) * TH, x3s + ((y + 1) % 3) * TH, t, c1, d1,
                             wx, wy, xm, xp, y > 0, y + 1 < n1, b1, o);
        x4s[(y % 3) * TH + t] = o;
      }
    }
    __syncthreads();
    // (c) result row y = j - 2 on the owned nodes
    {
      const int y = j - 2;
      if (own_x && y >= Y0 && y < Y1) {
        U o;
        ring_stencil<TPN, 2>(x4s + ((y + 2) % 3) * TH, x4s + (y % 3) * TH, x4s + ((y + 1) % 3) * TH, t, c2, d2,
                             wx, wy, xm, xp, y > 0, y + 1 < n1, b2, o);
        Out w[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) w[q] = ccast<Out>(o.v[q]);
        gstore(out + (int64_t(gx) + int64_t(n0) * y) * k + col, w);
      }
    }
    b2 = b1;
    b1 = b0;
    c2 = c1;
    c1 = c0;
    d2 = d1;
    d1 = d0;
  }
  cpa_wait<0>();
}


// ---------------------------------------------------------------------------
// k = 8 complex64 variants with bulk-copy (TMA) row staging and one barrier
// per streamed row.
//
// A CTA owns a strip of NT fine nodes (halo 4 per side, so every staged row
// starts 16-byte aligned) and all 8 RHS columns; 4 threads per node, each one
// 16-byte unit (2 complex64 columns). Thread 0 streams each fine row of the
// strip (right-hand side b, the node's (centre, D^{-1}) record, and for the
// post kernel the pre-smoothed iterate and the coarse correction rows) into
// a PD-deep ring of shared-memory slots with cp.async.bulk, completing on one
// mbarrier per slot; the copies of the next rows are in flight while the
// current ones are computed.
//
// The stages of the temporal blocking are skewed by two rows so that every
// stage of step j reads only rows published before the step's single
// __syncthreads (pre: x1 row j, x2 row j-2, r row j-4, restriction of row
// j-5; post: x3 row j, x4 row j-2, result row j-4); rings hold 4 rows (2
// for r). Nodes outside the grid hold exact zeros in every ring, so the
// stencils need no boundary predicates: a skipped neighbour term of the
// unfused kernels and an added w * (+0) give the same bits (the running sum
// starts at +0 and can never be -0), and the fused results stay bitwise
// equal to the unfused sequence.
constexpr int kK8 = 8;

template <class In, int NT, int PD>
struct PreK8Plan {
  static constexpr int TH = NT * 4, W = NT - 8;
  static constexpr size_t BROW = size_t(NT) * kK8 * sizeof(In);   // staged b row
  static constexpr size_t CROW = size_t(NT) * 2 * sizeof(float2);  // staged (centre, D^-1) row
  static constexpr size_t SLOT = BROW + CROW;
  static constexpr size_t RROW = size_t(NT) * kK8 * sizeof(float2);  // one ring row
  static constexpr size_t OFF_SLOTS = 128;  // PD mbarriers first
  static constexpr size_t OFF_X1 = OFF_SLOTS + PD * SLOT;
  static constexpr size_t OFF_X2 = OFF_X1 + 4 * RROW;
  static constexpr size_t OFF_R = OFF_X2 + 4 * RROW;
  static constexpr size_t BYTES = OFF_R + 2 * RROW + 128;  // + slack: edge threads read one unit past a ring row
};

__device__ __forceinline__ float4 u2f4(const Unit<float, 2>& u) { return make_float4(u.v[0].x, u.v[0].y, u.v[1].x, u.v[1].y); }
__device__ __forceinline__ Unit<float, 2> f42u(const float4& a) {
  Unit<float, 2> u;
  u.v[0] = make_float2(a.x, a.y);
  u.v[1] = make_float2(a.z, a.w);
  return u;
}

// (A u)[centre] for one 16-byte unit (2 columns): y-neighbours and centre
// from the thread's registers, x-neighbours from the ring row (units t -+ 4),
// every neighbour present (zero-padded), Csr::mul_block order
__device__ __forceinline__ void ax8r(const float4& um, const float4& u0, const float4& up, const float4* r0, int t,
                                     float2 c, float wx, float wy, float2 (&a)[2]) {
  const float4 uxm = r0[t - 4], uxp = r0[t + 4];
  const float2 ums[2] = {make_float2(um.x, um.y), make_float2(um.z, um.w)};
  const float2 uxms[2] = {make_float2(uxm.x, uxm.y), make_float2(uxm.z, uxm.w)};
  const float2 u0s[2] = {make_float2(u0.x, u0.y), make_float2(u0.z, u0.w)};
  const float2 uxps[2] = {make_float2(uxp.x, uxp.y), make_float2(uxp.z, uxp.w)};
  const float2 ups[2] = {make_float2(up.x, up.y), make_float2(up.z, up.w)};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    float2 acc = czero<float2>();
    acc = crfma(wy, ums[q], acc);
    acc = crfma(wx, uxms[q], acc);
    acc = cfma(c, u0s[q], acc);
    acc = crfma(wx, uxps[q], acc);
    acc = crfma(wy, ups[q], acc);
    a[q] = acc;
  }
}

template <int S>
using Step = std::integral_constant<int, S>;

// restriction of one r row (restrict_kernel order: ey, then ex ascending;
// zero weights skipped), as in fused_pre_kernel
__device__ __forceinline__ void restrict_row(int y, int n1, int CY0, int CY1, int64_t rcbase, int64_t rcstride,
                                             bool rxm, bool rxp, const Unit<float, 2>& rvm,
                                             const Unit<float, 2>& rv0, const Unit<float, 2>& rvp, float2 (&acc)[2],
                                             float2* __restrict__ rc) {
  const float h = 0.5f, one = 1.0f;
  if (y & 1) {
    const int J = (y - 1) >> 1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float2 a = acc[q];
      if (rxm) a = crfma(h * h, rvm.v[q], a);
      a = crfma(one * h, rv0.v[q], a);
      if (rxp) a = crfma(h * h, rvp.v[q], a);
      acc[q] = a;
    }
    if (J >= CY0 && J < CY1) gstore(rc + rcbase + rcstride * J, acc);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float2 a = czero<float2>();
      if (rxm) a = crfma(h * h, rvm.v[q], a);
      a = crfma(one * h, rv0.v[q], a);
      if (rxp) a = crfma(h * h, rvp.v[q], a);
      acc[q] = a;
    }
  } else {
    const int J = y >> 1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float2 a = acc[q];
      if (rxm) a = crfma(h * one, rvm.v[q], a);
      a = crfma(one * one, rv0.v[q], a);
      if (rxp) a = crfma(h * one, rvp.v[q], a);
      acc[q] = a;
    }
    if (y == n1 - 1 && J >= CY0 && J < CY1) gstore(rc + rcbase + rcstride * J, acc);
  }
}

// Steps are unrolled by 4: with rows counted from the first step, every
// ring row, staging slot and register FIFO entry of a step is a compile-time
// constant. A thread keeps its own node's rows of every intermediate in
// registers; the shared-memory rings exist only for the x-neighbours' reads
// of the centre row (shared-memory wavefronts, not DRAM, bound these kernels:
// profiles/r02_k8_fused.txt). Stage order D, C, B, A: stage C reads the b /
// centre FIFO entries of row j-4 before stage A refills them with row j.
template <class In, int NT, int PD, int MINB>
__global__ void __launch_bounds__(NT * 4, MINB)
fused_pre_k8_kernel(LevelOp<float> op, LevelGeom gc, float wj, const In* __restrict__ b, float2* __restrict__ x2out,
                    float2* __restrict__ rc, int crows) {
  static_assert(PD == 2 || PD == 4, "staging depth must divide the 4-step unroll");
  using P = PreK8Plan<In, NT, PD>;
  constexpr int W = P::W, TC = W / 2, TH = P::TH;
  constexpr int RU = NT * 4;  // float4 units per ring row
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  float4* x1s = reinterpret_cast<float4*>(sm + P::OFF_X1);
  float4* x2s = reinterpret_cast<float4*>(sm + P::OFF_X2);
  float4* rs = reinterpret_cast<float4*>(sm + P::OFF_R);
  const int n0 = int(op.g.n0), n1 = int(op.g.n1);
  const int t = threadIdx.x, xs = t >> 2, cg = t & 3;
  const int CX0 = blockIdx.x * TC, X0 = 2 * CX0, gx0 = X0 - 4, gx = gx0 + xs;
  const int CY0 = blockIdx.y * crows, CY1 = min(CY0 + crows, int(gc.n1));
  const int Y0 = 2 * CY0, Y1 = 2 * CY1;
  const int sa = max(0, -gx0), sb = min(NT, n0 - gx0);  // in-grid strip nodes [sa, sb)
  const bool inx = xs >= sa && xs < sb;
  const bool own_x = inx && xs >= 4 && xs < 4 + W;
  const int64_t x2base = int64_t(gx) * kK8 + cg * 2, x2stride = int64_t(n0) * kK8;
  const float wx = op.w[0], wy = op.w[1];
  // restriction units (coarse node ci, column pair rcg): 4 * TC of them,
  // spread evenly over the warps so that no warp carries the stage alone
  constexpr int NW = TH / 32, RPW = (4 * TC + NW - 1) / NW;
  static_assert(RPW <= 32, "one restriction unit per thread");
  const int lane = t & 31, ru = (t >> 5) * RPW + lane;
  const int ci = ru >> 2, rcg = ru & 3, I = CX0 + ci;
  const bool rest = lane < RPW && ru < 4 * TC && I < int(gc.n0);
  const int rt = (2 * ci + 4) * 4 + rcg;
  const bool rxm = 2 * I - 1 >= 0, rxp = 2 * I + 1 < n0;
  const int64_t rcbase = int64_t(I) * kK8 + rcg * 2, rcstride = int64_t(gc.n0) * kK8;

  const int jbeg = Y0 - 3;                                     // first step (x1 row)
  const int jA0 = max(jbeg, 0), jA1 = min(Y1 + 1, n1 - 1);     // x1 rows loaded
  const int yB0 = max(Y0 - 2, 0), yB1 = min(Y1, n1 - 1);       // x2 rows
  const int yC0 = max(Y0 - 1, 0), yC1 = min(Y1 - 1, n1 - 1);   // r rows (and restriction)
  const int nsteps = ((yC1 + 5 - jbeg + 1) + 3) & ~3;

  // zero the rings and the out-of-grid part of every staging slot, init barriers
  for (int i = t; i < int((P::BYTES - P::OFF_X1) / 16); i += TH)
    reinterpret_cast<float4*>(sm + P::OFF_X1)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!inx) {
#pragma unroll
    for (int p = 0; p < PD; ++p) {
      unsigned char* slot = sm + P::OFF_SLOTS + p * P::SLOT;
      float4* bz = reinterpret_cast<float4*>(slot) + t * (sizeof(In) / 8);
#pragma unroll
      for (int v = 0; v < int(sizeof(In) / 8); ++v) bz[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cg == 0) reinterpret_cast<float4*>(slot + P::BROW)[xs] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (t == 0) {
#pragma unroll
    for (int p = 0; p < PD; ++p) tma::mbar_init(&bars[p], 1);
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();
  const uint32_t nb = uint32_t(sb - sa);
  // row r = jbeg + u goes to slot u % PD; rows above the grid only advance
  // the slot's phase, rows past jA1 are never staged (nor waited for)
  auto produce = [&](int r) {
    if (r > jA1) return;
    const int u = r - jbeg, sl = u % PD;
    if (r < jA0) {
      tma::mbar_arrive_expect_tx(&bars[sl], 0);
      return;
    }
    tma::fence_proxy_async();
    unsigned char* slot = sm + P::OFF_SLOTS + sl * P::SLOT;
    const int64_t node0 = int64_t(n0) * r + gx0 + sa;
    tma::mbar_arrive_expect_tx(&bars[sl], nb * uint32_t(kK8 * sizeof(In) + 2 * sizeof(float2)));
    tma::bulk_g2s(slot + size_t(sa) * kK8 * sizeof(In), b + node0 * kK8, nb * uint32_t(kK8 * sizeof(In)), &bars[sl]);
    tma::bulk_g2s(slot + P::BROW + size_t(sa) * 16, op.cd + 2 * node0, nb * 16u, &bars[sl]);
  };
  if (t == 0)
#pragma unroll
    for (int p = 0; p < PD; ++p) produce(jbeg + p);

  // register FIFOs indexed by row mod 4 (relative to jbeg)
  float2 bq[4][2], cq[4], dq[4];
  float4 x1q[4], x2q[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    bq[r][0] = bq[r][1] = czero<float2>();
    cq[r] = dq[r] = czero<float2>();
    x1q[r] = x2q[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float2 acc[2] = {czero<float2>(), czero<float2>()};

  auto step = [&](auto S_, int j, uint32_t parity) {
    constexpr int S = decltype(S_)::value;  // (j - jbeg) mod 4
    constexpr int A = S, B = (S + 2) & 3, C = S, D1 = (S + 3) & 1, SL = S % PD;
    if (t == 0 && j > jbeg) produce(j - 1 + PD);  // the slot of row j-1 was released by the last barrier
    // (D) restriction of r row y = j-5
    {
      const int y = j - 5;
      if (rest && y >= yC0 && y <= yC1) {
        const float4* rr = rs + D1 * RU;
        const Unit<float, 2> rv0 = f42u(rr[rt]);
        const Unit<float, 2> rvm = rxm ? f42u(rr[rt - 4]) : rv0, rvp = rxp ? f42u(rr[rt + 4]) : rv0;
        restrict_row(y, n1, CY0, CY1, rcbase, rcstride, rxm, rxp, rvm, rv0, rvp, acc, rc);
      }
    }
    // (C) r row y = j-4 = b - A x2 (x2 rows j-5, j-4, j-3 in x2q)
    {
      const int y = j - 4;
      if (y >= yC0 && y <= yC1) {
        float2 a[2];
        ax8r(x2q[(S + 3) & 3], x2q[S], x2q[(S + 1) & 3], x2s + S * RU, t, cq[C], wx, wy, a);
        rs[(S & 1) * RU + t] = make_float4(bq[C][0].x - a[0].x, bq[C][0].y - a[0].y, bq[C][1].x - a[1].x,
                                           bq[C][1].y - a[1].y);
      }
    }
    // (B) x2 row y = j-2 = x1 + wD^-1 (b - A x1) (x1 rows j-3, j-2, j-1 in x1q)
    {
      const int y = j - 2;
      float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (y >= yB0 && y <= yB1) {
        float2 a[2];
        ax8r(x1q[(S + 1) & 3], x1q[B], x1q[(S + 3) & 3], x1s + B * RU, t, cq[B], wx, wy, a);
        const Unit<float, 2> x1 = f42u(x1q[B]);
        Unit<float, 2> o;
#pragma unroll
        for (int q = 0; q < 2; ++q) o.v[q] = cadd(x1.v[q], cmul(dq[B], csub(bq[B][q], a[q])));
        // out-of-grid nodes: x1 = 0, wD^-1 = 0 and b = 0 give +0 exactly
        o4 = u2f4(o);
        if (own_x && y >= Y0 && y < Y1) gstore(x2out + x2base + x2stride * y, o.v);
      }
      x2q[B] = o4;
      x2s[B * RU + t] = o4;
    }
    // (A) x1 row j = wD^-1 b (zero for rows / nodes not in the grid)
    {
      float4 x1v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j >= jA0 && j <= jA1) {
        tma::mbar_wait(&bars[SL], parity);
        const unsigned char* slot = sm + P::OFF_SLOTS + SL * P::SLOT;
        const In* bs = reinterpret_cast<const In*>(slot) + 2 * t;
        bq[A][0] = ccast<float2>(bs[0]);
        bq[A][1] = ccast<float2>(bs[1]);
        const float4 cdv = reinterpret_cast<const float4*>(slot + P::BROW)[xs];
        cq[A] = make_float2(cdv.x, cdv.y);
        dq[A] = make_float2(wj * cdv.z, wj * cdv.w);
        Unit<float, 2> x1;
        x1.v[0] = cmul(dq[A], bq[A][0]);
        x1.v[1] = cmul(dq[A], bq[A][1]);
        x1v = u2f4(x1);
      } else {
        bq[A][0] = bq[A][1] = czero<float2>();
        cq[A] = dq[A] = czero<float2>();
      }
      x1q[A] = x1v;
      x1s[A * RU + t] = x1v;
    }
    __syncthreads();
  };
  for (int m = 0; 4 * m < nsteps; ++m) {
    const int j = jbeg + 4 * m;
    // fills of a staging slot alternate parity: slot S % PD is filled for the
    // ((4m + S) / PD)-th time at step 4m + S
    step(Step<0>{}, j, uint32_t(((4 * m + 0) / PD) & 1));
    step(Step<1>{}, j + 1, uint32_t(((4 * m + 1) / PD) & 1));
    step(Step<2>{}, j + 2, uint32_t(((4 * m + 2) / PD) & 1));
    step(Step<3>{}, j + 3, uint32_t(((4 * m + 3) / PD) & 1));
  }
}

template <class In, int NT, int PD>
struct PostK8Plan {
  static constexpr int TH = NT * 4, W = NT - 4, NCN = NT / 2 + 1, CS = 4;
  static constexpr size_t XROW = size_t(NT) * kK8 * sizeof(float2);  // staged x2 row
  static constexpr size_t BROW = size_t(NT) * kK8 * sizeof(In);
  static constexpr size_t CROW = size_t(NT) * 2 * sizeof(float2);
  static constexpr size_t SLOT = XROW + BROW + CROW;
  static constexpr size_t EROW = size_t(NCN) * kK8 * sizeof(float2);  // staged coarse row
  static constexpr size_t RROW = size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t OFF_SLOTS = 128;  // PD + CS mbarriers first
  static constexpr size_t OFF_E = OFF_SLOTS + PD * SLOT;
  static constexpr size_t OFF_X3 = OFF_E + CS * EROW;
  static constexpr size_t OFF_X4 = OFF_X3 + 4 * RROW;
  static constexpr size_t BYTES = OFF_X4 + 4 * RROW + 128;  // + slack: edge threads read one unit past a ring row
};

// Post-smoothing of a zero-start visit, k = 8 complex64: x3 = x2 + P ec,
// x4 = x3 + wD^-1 (b - A x3), out = (Out)(x4 + wD^-1 (b - A x4)). Same step
// structure as fused_pre_k8_kernel (stages C, B, A).
template <class In, class Out, int NT, int PD, int MINB>
__global__ void __launch_bounds__(NT * 4, MINB)
fused_post_k8_kernel(LevelOp<float> op, LevelGeom gc, float wj, const float2* __restrict__ x2,
                     const float2* __restrict__ ec, const In* __restrict__ b, Out* __restrict__ out, int frows) {
  static_assert(PD == 2 || PD == 4, "staging depth must divide the 4-step unroll");
  using P = PostK8Plan<In, NT, PD>;
  constexpr int W = P::W, NCN = P::NCN, CS = P::CS, TH = P::TH;
  constexpr int RU = NT * 4;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);  // [PD] fine rows, [CS] coarse rows
  uint64_t* cbars = bars + PD;
  float4* x3s = reinterpret_cast<float4*>(sm + P::OFF_X3);
  float4* x4s = reinterpret_cast<float4*>(sm + P::OFF_X4);
  const int n0 = int(op.g.n0), n1 = int(op.g.n1), c0n = int(gc.n0), c1n = int(gc.n1);
  const int t = threadIdx.x, xs = t >> 2, cg = t & 3;
  const int X0 = blockIdx.x * W, gx0 = X0 - 2, gx = gx0 + xs;
  const int Y0 = blockIdx.y * frows, Y1 = min(Y0 + frows, n1);
  const int sa = max(0, -gx0), sb = min(NT, n0 - gx0);
  const bool inx = xs >= sa && xs < sb;
  const bool own_x = inx && xs >= 2 && xs < 2 + W;
  const int64_t obase = int64_t(gx) * kK8 + cg * 2, ostride = int64_t(n0) * kK8;
  const int cxa = (X0 >> 1) - 1;  // coarse nodes of the strip: [cxa, cxa + NCN), in grid [ca, cb)
  const int ca = max(0, -cxa), cb = min(NCN, c0n - cxa);
  // prolongation parents along i (prolong_v4_kernel) as strip coarse units
  const int p0 = ((gx >> 1) - cxa) * 4 + cg, p1 = (((gx + 1) >> 1) - cxa) * 4 + cg;
  const float wx0 = (gx & 1) ? 0.5f : 1.0f, wx1 = (gx & 1) ? 0.5f : 0.0f;
  const float wx = op.w[0], wy = op.w[1];

  const int jbeg = Y0 - 2;                                   // first step (x3 row)
  const int jA0 = max(jbeg, 0), jA1 = min(Y1 + 1, n1 - 1);   // x3 rows (staged fine rows)
  const int yB0 = max(Y0 - 1, 0), yB1 = min(Y1, n1 - 1);     // x4 rows
  const int Jc0 = jA0 >> 1, Jc1 = min((jA1 + 1) >> 1, c1n - 1);  // coarse rows
  const int nsteps = ((Y1 + 3 - jbeg + 1) + 3) & ~3;

  for (int i = t; i < int((P::BYTES - P::OFF_X3) / 16); i += TH)
    reinterpret_cast<float4*>(sm + P::OFF_X3)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!inx) {
#pragma unroll
    for (int p = 0; p < PD; ++p) {
      unsigned char* slot = sm + P::OFF_SLOTS + p * P::SLOT;
      reinterpret_cast<float4*>(slot)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      float4* bz = reinterpret_cast<float4*>(slot + P::XROW) + t * (sizeof(In) / 8);
#pragma unroll
      for (int v = 0; v < int(sizeof(In) / 8); ++v) bz[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cg == 0) reinterpret_cast<float4*>(slot + P::XROW + P::BROW)[xs] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  for (int i = t; i < CS * NCN * 4; i += TH) {
    const int cn = (i >> 2) % NCN;
    if (cn < ca || cn >= cb) reinterpret_cast<float4*>(sm + P::OFF_E)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (t == 0) {
#pragma unroll
    for (int p = 0; p < PD + CS; ++p) tma::mbar_init(&bars[p], 1);
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();
  const uint32_t nb = uint32_t(sb - sa), ncb = uint32_t(max(cb - ca, 0));
  int next_c = Jc0;  // next coarse row to stage (thread 0)
  auto issue_coarse = [&](int J) {
    const int u = J - Jc0, sl = u & (CS - 1);
    unsigned char* dst = sm + P::OFF_E + sl * P::EROW + size_t(ca) * kK8 * sizeof(float2);
    tma::mbar_arrive_expect_tx(&cbars[sl], ncb * uint32_t(kK8 * sizeof(float2)));
    tma::bulk_g2s(dst, ec + (int64_t(c0n) * J + cxa + ca) * kK8, ncb * uint32_t(kK8 * sizeof(float2)), &cbars[sl]);
  };
  auto produce = [&](int r) {
    if (r > jA1) return;
    const int u = r - jbeg, sl = u % PD;
    if (r < jA0) {
      tma::mbar_arrive_expect_tx(&bars[sl], 0);
      return;
    }
    tma::fence_proxy_async();
    unsigned char* slot = sm + P::OFF_SLOTS + sl * P::SLOT;
    const int64_t node0 = int64_t(n0) * r + gx0 + sa;
    tma::mbar_arrive_expect_tx(&bars[sl], nb * uint32_t(kK8 * (sizeof(float2) + sizeof(In)) + 2 * sizeof(float2)));
    tma::bulk_g2s(slot + size_t(sa) * kK8 * sizeof(float2), x2 + node0 * kK8, nb * uint32_t(kK8 * sizeof(float2)),
                  &bars[sl]);
    tma::bulk_g2s(slot + P::XROW + size_t(sa) * kK8 * sizeof(In), b + node0 * kK8, nb * uint32_t(kK8 * sizeof(In)),
                  &bars[sl]);
    tma::bulk_g2s(slot + P::XROW + P::BROW + size_t(sa) * 16, op.cd + 2 * node0, nb * 16u, &bars[sl]);
    for (; next_c <= min((r + 1) >> 1, Jc1); ++next_c) issue_coarse(next_c);
  };
  if (t == 0)
#pragma unroll
    for (int p = 0; p < PD; ++p) produce(jbeg + p);

  float2 bq[4][2], cq[4], dq[4];
  float4 x3q[4], x4q[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    bq[r][0] = bq[r][1] = czero<float2>();
    cq[r] = dq[r] = czero<float2>();
    x3q[r] = x4q[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  }

  auto step = [&](auto S_, int j, uint32_t parity) {
    constexpr int S = decltype(S_)::value;  // (j - jbeg) mod 4
    constexpr int A = S, B = (S + 2) & 3, C = S, SL = S % PD;
    if (t == 0 && j > jbeg) produce(j - 1 + PD);
    // (C) result row y = j-4 (x4 rows j-5, j-4, j-3 in x4q)
    {
      const int y = j - 4;
      if (own_x && y >= Y0 && y < Y1) {
        float2 a[2];
        ax8r(x4q[(S + 3) & 3], x4q[S], x4q[(S + 1) & 3], x4s + S * RU, t, cq[C], wx, wy, a);
        const Unit<float, 2> x4 = f42u(x4q[S]);
        Out w[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) w[q] = ccast<Out>(cadd(x4.v[q], cmul(dq[C], csub(bq[C][q], a[q]))));
        gstore(out + obase + ostride * y, w);
      }
    }
    // (B) x4 row y = j-2 (x3 rows j-3, j-2, j-1 in x3q)
    {
      const int y = j - 2;
      float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (y >= yB0 && y <= yB1) {
        float2 a[2];
        ax8r(x3q[(S + 1) & 3], x3q[B], x3q[(S + 3) & 3], x3s + B * RU, t, cq[B], wx, wy, a);
        const Unit<float, 2> x3 = f42u(x3q[B]);
        Unit<float, 2> o;
#pragma unroll
        for (int q = 0; q < 2; ++q) o.v[q] = cadd(x3.v[q], cmul(dq[B], csub(bq[B][q], a[q])));
        o4 = u2f4(o);
      }
      x4q[B] = o4;
      x4s[B * RU + t] = o4;
    }
    // (A) x3 row j = x2 + P ec (zero for rows / nodes not in the grid)
    {
      float4 x3v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j >= jA0 && j <= jA1) {
        tma::mbar_wait(&bars[SL], parity);
        const int J0 = j >> 1, J1 = (j + 1) >> 1;
        tma::mbar_wait(&cbars[(J0 - Jc0) & (CS - 1)], uint32_t(((J0 - Jc0) >> 2) & 1));
        if (J1 != J0) tma::mbar_wait(&cbars[(J1 - Jc0) & (CS - 1)], uint32_t(((J1 - Jc0) >> 2) & 1));
        const unsigned char* slot = sm + P::OFF_SLOTS + SL * P::SLOT;
        const In* bs = reinterpret_cast<const In*>(slot + P::XROW) + 2 * t;
        bq[A][0] = ccast<float2>(bs[0]);
        bq[A][1] = ccast<float2>(bs[1]);
        const float4 cdv = reinterpret_cast<const float4*>(slot + P::XROW + P::BROW)[xs];
        cq[A] = make_float2(cdv.x, cdv.y);
        dq[A] = make_float2(wj * cdv.z, wj * cdv.w);
        const float4* er0 = reinterpret_cast<const float4*>(sm + P::OFF_E + ((J0 - Jc0) & (CS - 1)) * P::EROW);
        const float4* er1 = reinterpret_cast<const float4*>(sm + P::OFF_E + ((J1 - Jc0) & (CS - 1)) * P::EROW);
        const float wy0 = (j & 1) ? 0.5f : 1.0f, wy1 = (j & 1) ? 0.5f : 0.0f;
        const float w00 = wx0 * wy0 * 1.0f, w01 = wx1 * wy0 * 1.0f, w10 = wx0 * wy1 * 1.0f, w11 = wx1 * wy1 * 1.0f;
        const Unit<float, 2> xr = f42u(reinterpret_cast<const float4*>(slot)[t]);
        const Unit<float, 2> e00 = f42u(er0[p0]), e01 = f42u(er0[p1]);
        Unit<float, 2> e10 = e00, e11 = e01;
        if (j & 1) {
          e10 = f42u(er1[p0]);
          e11 = f42u(er1[p1]);
        }
        Unit<float, 2> x3;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          // parents in (y, x) ascending order, zero weights skipped
          float2 corr = czero<float2>();
          corr = crfma(w00, e00.v[q], corr);
          if (w01 != 0.0f) corr = crfma(w01, e01.v[q], corr);
          if (w10 != 0.0f) corr = crfma(w10, e10.v[q], corr);
          if (w11 != 0.0f) corr = crfma(w11, e11.v[q], corr);
          x3.v[q] = cadd(xr.v[q], corr);
        }
        if (inx) x3v = u2f4(x3);
      } else {
        bq[A][0] = bq[A][1] = czero<float2>();
        cq[A] = dq[A] = czero<float2>();
      }
      x3q[A] = x3v;
      x3s[A * RU + t] = x3v;
    }
    __syncthreads();
  };
  for (int m = 0; 4 * m < nsteps; ++m) {
    const int j = jbeg + 4 * m;
    step(Step<0>{}, j, uint32_t(((4 * m + 0) / PD) & 1));
    step(Step<1>{}, j + 1, uint32_t(((4 * m + 1) / PD) & 1));
    step(Step<2>{}, j + 2, uint32_t(((4 * m + 2) / PD) & 1));
    step(Step<3>{}, j + 3, uint32_t(((4 * m + 3) / PD) & 1));
  }
}

// ---------------------------------------------------------------------------
// 2D Galerkin level (9-point planes), k = 8 complex64, one stencil per launch
// (apply / residual / damped Jacobi) with bulk-copy row staging: a CTA owns a
// strip of NT nodes and streams its rows -- x with a one-node halo, the
// 80-byte (9 coefficients, D^-1) records, b -- through a PD-deep ring of
// slots, one mbarrier each; output row j reads the x rows j-1, j, j+1 of three
// slots. 4 threads per node (2 columns each). Rows outside the grid stage a
// row inside it (their coefficients are 0, as in the planes), halo nodes
// outside it hold zeros; sums in ascending plane order, so the results equal
// the stencil_v4 kernels bitwise.
template <int MODE, int NT, int PD>
struct S9Plan {
  static constexpr int TH = NT * 4;
  static constexpr size_t XROW = size_t(NT + 2) * kK8 * sizeof(float2);
  static constexpr size_t CROW = size_t(NT) * 10 * sizeof(float2);
  static constexpr size_t BROW = MODE == 0 ? 0 : size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t SLOT = XROW + CROW + BROW;
  static constexpr size_t OFF_SLOTS = 128;
  static constexpr size_t BYTES = OFF_SLOTS + PD * SLOT;
};

template <int MODE, int NT, int PD, int MINB>
__global__ void __launch_bounds__(NT * 4, MINB)
stencil9_k8_kernel(LevelOp<float> op, float wj, const float2* __restrict__ x, const float2* __restrict__ b,
                   float2* __restrict__ out, int rows) {
  using P = S9Plan<MODE, NT, PD>;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  const int n0 = int(op.g.n0), n1 = int(op.g.n1);
  const int t = threadIdx.x, xs = t >> 2, cg = t & 3;
  const int X0 = blockIdx.x * NT, gx = X0 + xs;
  const int Y0 = blockIdx.y * rows, Y1 = min(Y0 + rows, n1);
  const bool inx = gx < n0;
  // staged x columns [X0 - 1, X0 + NT + 1) clipped to the grid: strip units [xa, xb)
  const int xa = X0 == 0 ? 1 : 0, xb = min(NT + 2, n0 - X0 + 1);
  const int nc = min(NT, n0 - X0);  // owned nodes in the grid
  const int r0 = Y0 - 1, r1 = Y1;   // staged rows (x halo rows included)
  // zero the x halo units outside the grid in every slot (never overwritten)
  for (int p = 0; p < PD; ++p) {
    float4* xr = reinterpret_cast<float4*>(sm + P::OFF_SLOTS + p * P::SLOT);
    for (int u = t; u < (NT + 2) * 4; u += P::TH) {
      const int node = u >> 2;
      if (node < xa || node >= xb) xr[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (t == 0) {
    for (int p = 0; p < PD; ++p) tma::mbar_init(&bars[p], 1);
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();
  auto produce = [&](int r) {
    if (r > r1) return;
    tma::fence_proxy_async();
    const int u = r - r0, sl = u % PD;
    unsigned char* slot = sm + P::OFF_SLOTS + sl * P::SLOT;
    const int rr = min(max(r, 0), n1 - 1);  // rows outside the grid: any finite row (coefficients 0)
    const bool own = r >= Y0 && r < Y1;
    const uint32_t xbytes = uint32_t(xb - xa) * kK8 * sizeof(float2);
    uint32_t tx = xbytes;
    if (own) tx += uint32_t(nc) * (10 * sizeof(float2) + (MODE == 0 ? 0 : kK8 * sizeof(float2)));
    tma::mbar_arrive_expect_tx(&bars[sl], tx);
    tma::bulk_g2s(slot + size_t(xa) * kK8 * sizeof(float2), x + (int64_t(n0) * rr + X0 - 1 + xa) * kK8, xbytes,
                  &bars[sl]);
    if (own) {
      tma::bulk_g2s(slot + P::XROW, op.cd + (int64_t(n0) * r + X0) * 10, uint32_t(nc) * 10 * sizeof(float2),
                    &bars[sl]);
      if (MODE != 0)
        tma::bulk_g2s(slot + P::XROW + P::CROW, b + (int64_t(n0) * r + X0) * kK8,
                      uint32_t(nc) * kK8 * sizeof(float2), &bars[sl]);
    }
  };
  if (t == 0)
    for (int p = 0; p < PD && r0 + p <= r1; ++p) produce(r0 + p);
  auto wait_row = [&](int r) {
    const int u = r - r0;
    tma::mbar_wait(&bars[u % PD], uint32_t((u / PD) & 1));
  };
  wait_row(r0);
  for (int j = Y0; j < Y1; ++j) {
    wait_row(j);
    wait_row(j + 1);
    const unsigned char* sj = sm + P::OFF_SLOTS + ((j - r0) % PD) * P::SLOT;
    const float4* xr[3];
#pragma unroll
    for (int d = 0; d < 3; ++d)
      xr[d] = reinterpret_cast<const float4*>(sm + P::OFF_SLOTS + ((j - 1 + d - r0) % PD) * P::SLOT);
    if (inx) {
      const float2* cf = reinterpret_cast<const float2*>(sj + P::XROW) + xs * 10;
      float2 av[9];
      float4 xv[9];
#pragma unroll
      for (int sdx = 0; sdx < 9; ++sdx) {
        const int dy = sdx / 3 - 1, dx = sdx % 3 - 1;
        av[sdx] = cf[sdx];
        xv[sdx] = xr[dy + 1][(xs + 1 + dx) * 4 + cg];
      }
      float2 acc[2] = {czero<float2>(), czero<float2>()};
#pragma unroll
      for (int sdx = 0; sdx < 9; ++sdx) {
        acc[0] = cfma(av[sdx], make_float2(xv[sdx].x, xv[sdx].y), acc[0]);
        acc[1] = cfma(av[sdx], make_float2(xv[sdx].z, xv[sdx].w), acc[1]);
      }
      float2 o[2];
      if (MODE == 0) {
        o[0] = acc[0];
        o[1] = acc[1];
      } else {
        const float4 bv = reinterpret_cast<const float4*>(sj + P::XROW + P::CROW)[t];
        const float2 bb[2] = {make_float2(bv.x, bv.y), make_float2(bv.z, bv.w)};
        if (MODE == 1) {
          o[0] = csub(bb[0], acc[0]);
          o[1] = csub(bb[1], acc[1]);
        } else {
          const float2 d = cf[9];
          const float2 wd = mk(wj * d.x, wj * d.y);
          const float4 xc = xv[4];
          o[0] = jacobi_upd(make_float2(xc.x, xc.y), wd, bb[0], acc[0]);
          o[1] = jacobi_upd(make_float2(xc.z, xc.w), wd, bb[1], acc[1]);
        }
      }
      gstore(out + (int64_t(n0) * j + gx) * kK8 + cg * 2, o);
    }
    __syncthreads();  // row j-1's slot is free: its last reader was this step
    if (t == 0) produce(j - 1 + PD);
  }
}

#ifndef HZ_S9_NT
#define HZ_S9_NT 64
#endif
#ifndef HZ_S9_PD
#define HZ_S9_PD 4
#endif
int env_int(const char* name, int dflt);

template <int MODE>
void run_stencil9_k8(const LevelOp<float>& op, float wj, const float2* x, const float2* b, float2* out,
                     cudaStream_t s) {
  constexpr int NT = HZ_S9_NT, PD = HZ_S9_PD;
  using P = S9Plan<MODE, NT, PD>;
  constexpr int MINB = int(std::min<size_t>(std::min<size_t>((227 * 1024) / (P::BYTES + 1024), 2048 / P::TH), 8));
  const int strips = int((op.g.n0 + NT - 1) / NT);
  // rows per CTA: enough CTAs for about one resident wave, at least 4 rows
  // (measured at level 1 of config 2: 4 rows 12.7 us, 8 rows 14.5, 16 rows
  // 15.4, the plain kernel 13.3; profiles/r02_stencil9_ab.txt)
  const int slots = kNumSMs * MINB;
  const int chunks = std::max(1, slots / std::max(1, strips));
  const int e = env_int("HZ_S9_ROWS", 0);
  const int rows = e > 0 ? e : std::max(4, int((op.g.n1 + chunks - 1) / chunks));
  const dim3 grid(unsigned(strips), unsigned((op.g.n1 + rows - 1) / rows));
  auto kern = stencil9_k8_kernel<MODE, NT, PD, MINB>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, wj, x, b, out, rows);
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// strip shape: NT nodes x 2 threads per node; c64: 4 columns per CTA
#ifndef HZ_FUSED_PD
#define HZ_FUSED_PD 2  // staged rows in flight: 2 measured 3-4 % faster than 3 with 4 concurrent 8-column groups (less shared memory per CTA; profiles/r01_fused_pd_ab.txt)
#endif
#ifndef HZ_FUSED_MAXB
#define HZ_FUSED_MAXB 8
#endif
constexpr int kTPN = 2, kPD = HZ_FUSED_PD;

template <class T, class In, int NT, int QU>
void run_fused_pre(const LevelOp<T>& op, const LevelGeom& gc, T wj, const In* b, cplx_t<T>* x2, cplx_t<T>* rc,
                   int crows, cudaStream_t s) {
  using P = PrePlan<T, In, kTPN, NT, kPD, QU>;
  constexpr int TC = (NT - 6) / 2, C = kTPN * QU;
  // resident CTAs per SM: by shared memory (228 KB per SM)
  constexpr int MINB = int(std::min<size_t>(HZ_FUSED_MAXB, (227 * 1024) / (P::BYTES + 1024)));
  const dim3 grid(unsigned((gc.n0 + TC - 1) / TC), unsigned(op.g.k / C), unsigned((gc.n1 + crows - 1) / crows));
  auto kern = fused_pre_kernel<T, In, kTPN, NT, kPD, (MINB * P::TH > 2048 ? 2048 / P::TH : MINB), QU>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, gc, wj, b, x2, rc, crows);
}

template <class T, class In, class Out, int NT, int QU>
void run_fused_post(const LevelOp<T>& op, const LevelGeom& gc, T wj, const cplx_t<T>* x2, const cplx_t<T>* ec,
                    const In* b, Out* out, int frows, cudaStream_t s) {
  using P = PostPlan<T, In, kTPN, NT, kPD, QU>;
  constexpr int W = NT - 4, C = kTPN * QU;
  constexpr int MINB = int(std::min<size_t>(HZ_FUSED_MAXB, (227 * 1024) / (P::BYTES + 1024)));
  const dim3 grid(unsigned((op.g.n0 + W - 1) / W), unsigned(op.g.k / C), unsigned((op.g.n1 + frows - 1) / frows));
  auto kern = fused_post_kernel<T, In, Out, kTPN, NT, kPD, (MINB * P::TH > 2048 ? 2048 / P::TH : MINB), QU>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, gc, wj, x2, ec, b, out, frows);
}

// ---- k = 8 complex64 bulk-copy kernels: launch geometry
#ifndef HZ_K8_NT
#define HZ_K8_NT 64  // strip width (fine nodes) of the k = 8 kernels: 4 x NT threads per CTA
#endif
#ifndef HZ_K8_MINB
#define HZ_K8_MINB 2  // resident CTAs per SM the register budget is sized for (3 spills)
#endif
#ifndef HZ_K8_PD
#define HZ_K8_PD 4  // staged rows in flight per CTA (2 or 4)
#endif

template <size_t BYTES, int TH>
constexpr int k8_blocks_per_sm() {
  return int(std::min<size_t>(std::min<size_t>((227 * 1024) / (BYTES + 1024), 2048 / TH), 8));
}

// rows per chunk so that the strips x chunks tiles fill the resident CTA
// slots of the GPU about once (every tile pays a pipeline fill of a few rows)
int k8_chunk_rows(int strips, int rows, int per_sm, const char* env) {
  const int e = env_int(env, 0);
  if (e > 0) return e;
  const int slots = std::max(1, kNumSMs * per_sm);
  const int chunks = std::max(1, slots / std::max(1, strips));
  return std::max(4, (rows + chunks - 1) / chunks);
}

template <class In>
void run_fused_pre_k8(const LevelOp<float>& op, const LevelGeom& gc, float wj, const In* b, float2* x2, float2* rc,
                      cudaStream_t s) {
  constexpr int NT = HZ_K8_NT, PD = HZ_K8_PD;
  using P = PreK8Plan<In, NT, PD>;
  constexpr int MINB = HZ_K8_MINB;
  constexpr int TC = P::W / 2;
  const int strips = int((gc.n0 + TC - 1) / TC);
  const int crows = k8_chunk_rows(strips, int(gc.n1), std::min(MINB, k8_blocks_per_sm<P::BYTES, P::TH>()),
                                  "HZ_K8_PRE_ROWS");
  const dim3 grid(unsigned(strips), unsigned((gc.n1 + crows - 1) / crows));
  auto kern = fused_pre_k8_kernel<In, NT, PD, MINB>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, gc, wj, b, x2, rc, crows);
}

template <class In, class Out>
void run_fused_post_k8(const LevelOp<float>& op, const LevelGeom& gc, float wj, const float2* x2, const float2* ec,
                       const In* b, Out* out, cudaStream_t s) {
  constexpr int NT = HZ_K8_NT, PD = HZ_K8_PD;
  using P = PostK8Plan<In, NT, PD>;
  constexpr int MINB = HZ_K8_MINB;
  const int strips = int((op.g.n0 + P::W - 1) / P::W);
  const int frows = 2 * k8_chunk_rows(strips, int(gc.n1), std::min(MINB, k8_blocks_per_sm<P::BYTES, P::TH>()),
                                      "HZ_K8_POST_CROWS");
  const dim3 grid(unsigned(strips), unsigned((op.g.n1 + frows - 1) / frows));
  auto kern = fused_post_k8_kernel<In, Out, NT, PD, MINB>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, gc, wj, x2, ec, b, out, frows);
}

bool k8_enabled(int k, const void* cd) {
  static const int env = env_int("HZ_FUSED_K8", 1);
  return env != 0 && k == kK8 && cd != nullptr;
}

// strip width in fine nodes: HZ_FUSED_NT = 32, 64 or 128; default 64, and
// 32 when a CTA's 4 columns cover the block in <= 2 CTAs (k <= 8): the
// strips stream their rows sequentially, so narrow blocks need the extra
// (narrower) strips to keep enough row chains in flight
// two 16-byte vectors per thread unit (complex64 only, k % 8 == 0), opt-in
// with HZ_FUSED_WIDE=1: at k = 8 it halves the threads and measured slower
// (post 82 vs 60 us, 1.47 vs 1.31 ms per bench cycle,
// profiles/r01_fused_wide_units.txt) -- these kernels need row chains in
// flight more than per-row amortisation
template <class T>
bool fused_wide(int k) {
  if (sizeof(T) != 4 || k % (kTPN * 2 * cpt<T>()) != 0) return false;
  static const int env = env_int("HZ_FUSED_WIDE", 0);
  return env != 0;
}

int fused_nt(int k, int cols_per_cta) {
  static const int env = env_int("HZ_FUSED_NT", 0);
  if (env == 32 || env == 64 || env == 128) return env;
  return k / cols_per_cta <= 2 ? 32 : 64;
}

}  // namespace

bool launch_stencil9_k8(const LevelOp<float>& op, int mode, float wj, const float2* x, const float2* b, float2* out,
                        cudaStream_t s) {
  static const bool on = env_int("HZ_S9", 1) != 0;
  if (!on || op.kind != kStencil || op.ndim != 2 || op.g.k != kK8 || !op.cd || op.g.z0 != 0 ||
      op.g.z1 != op.g.n1)
    return false;
  if (mode == 0)
    run_stencil9_k8<0>(op, wj, x, b, out, s);
  else if (mode == 1)
    run_stencil9_k8<1>(op, wj, x, b, out, s);
  else
    run_stencil9_k8<2>(op, wj, x, b, out, s);
  return true;
}

// ---------------------------------------------------------------------------
// Two damped-Jacobi sweeps of a 2D Galerkin level in one launch (k = 8,
// complex64): relax(..., 2 sweeps) of src/multigrid.cpp:119-136 with the
// intermediate iterate kept in shared memory. ZERO: the visit starts from
// x = 0, so the first sweep is x1 = wD^-1 b (jacobi_zero) and no iterate is
// read at all.
//
// A CTA owns NT - 2 nodes of a strip of NT (one halo node per side for the
// first sweep) and a chunk of rows; rows stream through a PD-deep ring of
// slots (x with a one-node halo, the 80-byte (9 coefficients, D^-1) records,
// b), one mbarrier each, as in stencil9_k8_kernel. Step j computes the first
// sweep's row j into a 4-row ring and the second sweep's row j - 2 from the
// ring rows j - 3 .. j - 1 published by earlier barriers: one __syncthreads
// per step. Same per-column operations in the same order as two
// stencil9_k8 / stencil_v4 launches (ascending plane order, jacobi_upd), and
// couplings that leave the grid are exact zeros in the records, so the
// results are bitwise equal.
template <bool ZERO, int NT, int PD>
struct S9PairPlan {
  static constexpr int TH = NT * 4;
  static constexpr size_t XROW = ZERO ? 0 : size_t(NT + 2) * kK8 * sizeof(float2);
  static constexpr size_t CROW = size_t(NT) * 10 * sizeof(float2);
  static constexpr size_t BROW = size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t SLOT = XROW + CROW + BROW;
  static constexpr size_t RROW = size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t OFF_SLOTS = 128;
  static constexpr size_t OFF_RING = OFF_SLOTS + PD * SLOT;
  static constexpr size_t BYTES = OFF_RING + 4 * RROW;
};

template <bool ZERO, int NT, int PD, int MINB>
__global__ void __launch_bounds__(NT * 4, MINB)
stencil9_pair_k8_kernel(LevelOp<float> op, float wj, const float2* __restrict__ x, const float2* __restrict__ b,
                        float2* __restrict__ out, int rows) {
  using P = S9PairPlan<ZERO, NT, PD>;
  static_assert(PD >= 5, "rows j-2 .. j+1 are live in a step");
  constexpr int RU = NT * 4;  // float4 units per ring row
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  float4* ring = reinterpret_cast<float4*>(sm + P::OFF_RING);
  const int n0 = int(op.g.n0), n1 = int(op.g.n1);
  const int t = threadIdx.x, xs = t >> 2, cg = t & 3;
  const int X0 = blockIdx.x * (NT - 2), gx = X0 - 1 + xs;  // strip nodes [X0 - 1, X0 + NT - 1)
  const int Y0 = blockIdx.y * rows, Y1 = min(Y0 + rows, n1);
  const bool inx = gx >= 0 && gx < n0;
  const bool own_x = inx && xs >= 1 && xs < NT - 1;
  const int rA0 = max(Y0 - 1, 0), rA1 = min(Y1, n1 - 1);  // first-sweep rows (inclusive)
  const int r0 = Y0 - 2, r1 = Y1 + 1;                     // streamed rows
  // in-grid parts of a staged row: records / b over strip nodes [sa, sb), x over units [xa, xb) of
  // nodes [X0 - 2, X0 + NT)
  const int sa = max(0, 1 - X0), sb = min(NT, n0 - X0 + 1);
  const int xa = max(0, 2 - X0), xb = min(NT + 2, n0 - X0 + 2);
  for (int i = t; i < int((P::BYTES - P::OFF_SLOTS) / 16); i += P::TH)
    reinterpret_cast<float4*>(sm + P::OFF_SLOTS)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t == 0) {
    for (int p = 0; p < PD; ++p) tma::mbar_init(&bars[p], 1);
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();
  auto produce = [&](int r) {
    if (r > r1) return;
    tma::fence_proxy_async();
    const int sl = (r - r0) % PD;
    unsigned char* slot = sm + P::OFF_SLOTS + sl * P::SLOT;
    const bool recs = r >= rA0 && r <= rA1;
    const int rr = min(max(r, 0), n1 - 1);  // x rows outside the grid: any finite row (their couplings are 0)
    const uint32_t xbytes = ZERO ? 0u : uint32_t(xb - xa) * kK8 * sizeof(float2);
    const uint32_t nrec = uint32_t(sb - sa);
    tma::mbar_arrive_expect_tx(&bars[sl], xbytes + (recs ? nrec * uint32_t((10 + kK8) * sizeof(float2)) : 0u));
    if (!ZERO)
      tma::bulk_g2s(slot + size_t(xa) * kK8 * sizeof(float2), x + (int64_t(n0) * rr + X0 - 2 + xa) * kK8, xbytes,
                    &bars[sl]);
    if (recs) {
      const int64_t node0 = int64_t(n0) * r + X0 - 1 + sa;
      tma::bulk_g2s(slot + P::XROW + size_t(sa) * 10 * sizeof(float2), op.cd + node0 * 10,
                    nrec * uint32_t(10 * sizeof(float2)), &bars[sl]);
      tma::bulk_g2s(slot + P::XROW + P::CROW + size_t(sa) * kK8 * sizeof(float2), b + node0 * kK8,
                    nrec * uint32_t(kK8 * sizeof(float2)), &bars[sl]);
    }
  };
  if (t == 0)
    for (int p = 0; p < PD; ++p) produce(r0 + p);
  auto wait_row = [&](int r) {
    const int u = r - r0;
    tma::mbar_wait(&bars[u % PD], uint32_t((u / PD) & 1));
  };
  auto slot_of = [&](int r) { return sm + P::OFF_SLOTS + ((r - r0) % PD) * P::SLOT; };
  // one sweep's output for this thread's 2 columns of row r: xr = the three x rows (units of 4 per
  // node, unit 0 = node `base` - 1), own value xc
  auto sweep = [&](const unsigned char* srow, const float4* xm1, const float4* x00, const float4* xp1, int base,
                   float2 (&o)[2]) {
    const float2* cf = reinterpret_cast<const float2*>(srow + P::XROW) + xs * 10;
    const float4* xr[3] = {xm1, x00, xp1};
    float2 av[9];
    float4 xv[9];
#pragma unroll
    for (int sdx = 0; sdx < 9; ++sdx) {
      const int dy = sdx / 3 - 1, dx = sdx % 3 - 1;
      av[sdx] = cf[sdx];
      xv[sdx] = xr[dy + 1][(base + dx) * 4 + cg];
    }
    float2 acc[2] = {czero<float2>(), czero<float2>()};
#pragma unroll
    for (int sdx = 0; sdx < 9; ++sdx) {
      acc[0] = cfma(av[sdx], make_float2(xv[sdx].x, xv[sdx].y), acc[0]);
      acc[1] = cfma(av[sdx], make_float2(xv[sdx].z, xv[sdx].w), acc[1]);
    }
    const float4 bv = reinterpret_cast<const float4*>(srow + P::XROW + P::CROW)[t];
    const float2 d = cf[9];
    const float2 wd = mk(wj * d.x, wj * d.y);
    const float4 xc = xv[4];
    o[0] = jacobi_upd(make_float2(xc.x, xc.y), wd, make_float2(bv.x, bv.y), acc[0]);
    o[1] = jacobi_upd(make_float2(xc.z, xc.w), wd, make_float2(bv.z, bv.w), acc[1]);
  };
  for (int j = Y0 - 1; j <= Y1 + 1; ++j) {
    // (2) second sweep, row y = j - 2, from the ring rows y - 1, y, y + 1
    const int y = j - 2;
    if (own_x && y >= Y0 && y < Y1) {
      float2 o[2];
      sweep(slot_of(y), ring + ((y + 3) & 3) * RU, ring + (y & 3) * RU, ring + ((y + 1) & 3) * RU, xs, o);
      gstore(out + (int64_t(n0) * y + gx) * kK8 + cg * 2, o);
    }
    // (1) first sweep, row j, into the ring
    float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j >= rA0 && j <= rA1) {
      if (ZERO) {
        wait_row(j);
        if (inx) {
          const unsigned char* srow = slot_of(j);
          const float2 d = (reinterpret_cast<const float2*>(srow + P::XROW) + xs * 10)[9];
          const float2 wd = mk(wj * d.x, wj * d.y);
          const float4 bv = reinterpret_cast<const float4*>(srow + P::XROW + P::CROW)[t];
          const float2 a = cmul(wd, make_float2(bv.x, bv.y)), c = cmul(wd, make_float2(bv.z, bv.w));
          x1 = make_float4(a.x, a.y, c.x, c.y);
        }
      } else {
        wait_row(j - 1);
        wait_row(j);
        wait_row(j + 1);
        if (inx) {
          float2 o[2];
          sweep(slot_of(j), reinterpret_cast<const float4*>(slot_of(j - 1)), reinterpret_cast<const float4*>(slot_of(j)),
                reinterpret_cast<const float4*>(slot_of(j + 1)), xs + 1, o);
          x1 = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
        }
      }
    }
    ring[(j & 3) * RU + t] = x1;
    __syncthreads();  // row j - 2's slot is free: its last readers were this step's sweeps
    if (t == 0 && j - 2 >= r0) produce(j - 2 + PD);
  }
}

template <bool ZERO>
void run_stencil9_pair_k8(const LevelOp<float>& op, float wj, const float2* x, const float2* b, float2* out,
                          cudaStream_t s) {
  constexpr int NT = 64, PD = 6;
  using P = S9PairPlan<ZERO, NT, PD>;
  constexpr int MINB = int(std::min<size_t>(std::min<size_t>((227 * 1024) / (P::BYTES + 1024), 2048 / P::TH), 8));
  const int strips = int((op.g.n0 + NT - 3) / (NT - 2));
  // rows per CTA: about one resident wave of CTAs, at least 8 rows (3 extra rows are staged and 2 extra
  // first-sweep rows computed per chunk); HZ_S9P_ROWS forces
  const int chunks = std::max(1, kNumSMs * MINB / std::max(1, strips));
  const int e = env_int("HZ_S9P_ROWS", 0);
  const int rows = e > 0 ? e : std::max(8, int((op.g.n1 + chunks - 1) / chunks));
  const dim3 grid(unsigned(strips), unsigned((op.g.n1 + rows - 1) / rows));
  auto kern = stencil9_pair_k8_kernel<ZERO, NT, PD, MINB>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, wj, x, b, out, rows);
}

bool launch_stencil9_pair_k8(const LevelOp<float>& op, float wj, const float2* x, const float2* b, float2* out,
                             cudaStream_t s) {
  static const bool on = env_int("HZ_S9_PAIR", 1) != 0;
  static const int64_t min_nodes = env_int("HZ_S9_PAIR_MIN_NODES", 100000);
  if (!on || op.kind != kStencil || op.ndim != 2 || op.g.k != kK8 || !op.cd || op.g.z0 != 0 ||
      op.g.z1 != op.g.n1 || int64_t(op.g.nodes) < min_nodes || op.g.n1 < 4)
    return false;
  const double n = double(op.g.nodes);
  ProfScope prof(x ? "jacobi2_stencil_c64_L1" : "jacobi2_zero_stencil_c64_L1",
                 n * (kK8 * 8.0 * (x ? 3.0 : 2.0) + 80.0), s);
  if (x)
    run_stencil9_pair_k8<false>(op, wj, x, b, out, s);
  else
    run_stencil9_pair_k8<true>(op, wj, x, b, out, s);
  HZ_LAUNCH_CHECK();
  return true;
}

// ---------------------------------------------------------------------------
// Zero-start pre-smoothing visit of a 2D Galerkin level in one launch (k = 8,
// complex64): x1 = wD^-1 b, x2 = x1 + wD^-1 (b - A x1), r = b - A x2 and the
// restriction rc = P^T r (cycle_rec, src/multigrid.cpp:162-178), with x1 and r
// never written to memory. The geometry is fused_pre_k8_kernel's (strip of NT
// nodes = 2 * TC + 8, halo 4 per side, chunks of coarse rows, restriction
// units spread over the warps, restrict_row); the operator is the 9-point
// stencil read from the level's 80-byte records, so all three rows of every
// stage come from shared-memory rings (4 rows of x1, 4 of x2, 2 of r), and the
// record / b rows stay in their slots until the stage that needs them last
// (row j - 4) has run. Stages of step j: restriction of r row j - 5, r row
// j - 4, x2 row j - 2, x1 row j; each reads only ring rows published by an
// earlier step's barrier. Same operations in the same order as the unfused
// kernels: bitwise equal.
template <int NT, int PD>
struct S9PrePlan {
  static constexpr int TH = NT * 4, W = NT - 8, TC = W / 2;
  static constexpr size_t CROW = size_t(NT) * 10 * sizeof(float2);
  static constexpr size_t BROW = size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t SLOT = CROW + BROW;
  static constexpr size_t RROW = size_t(NT) * kK8 * sizeof(float2);
  static constexpr size_t OFF_SLOTS = 128;
  static constexpr size_t OFF_X1 = OFF_SLOTS + PD * SLOT;
  static constexpr size_t OFF_X2 = OFF_X1 + 4 * RROW;
  static constexpr size_t OFF_R = OFF_X2 + 4 * RROW;
  static constexpr size_t BYTES = OFF_R + 2 * RROW;
};

template <int NT, int PD, int MINB>
__global__ void __launch_bounds__(NT * 4, MINB)
stencil9_pre_k8_kernel(LevelOp<float> op, LevelGeom gc, float wj, const float2* __restrict__ b,
                       float2* __restrict__ x2out, float2* __restrict__ rc, int crows) {
  using P = S9PrePlan<NT, PD>;
  static_assert(PD >= 6, "rows j-4 .. j are live in a step");
  constexpr int W = P::W, TC = P::TC, TH = P::TH, RU = NT * 4;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  float4* x1s = reinterpret_cast<float4*>(sm + P::OFF_X1);
  float4* x2s = reinterpret_cast<float4*>(sm + P::OFF_X2);
  float4* rs = reinterpret_cast<float4*>(sm + P::OFF_R);
  const int n0 = int(op.g.n0), n1 = int(op.g.n1);
  const int t = threadIdx.x, xs = t >> 2, cg = t & 3;
  const int CX0 = blockIdx.x * TC, X0 = 2 * CX0, gx0 = X0 - 4, gx = gx0 + xs;
  const int CY0 = blockIdx.y * crows, CY1 = min(CY0 + crows, int(gc.n1));
  const int Y0 = 2 * CY0, Y1 = 2 * CY1;
  const int sa = max(0, -gx0), sb = min(NT, n0 - gx0);  // in-grid strip nodes [sa, sb)
  const bool inx = xs >= sa && xs < sb;
  const bool own_x = inx && xs >= 4 && xs < 4 + W;
  // restriction units (coarse node ci, column pair rcg), spread evenly over the warps
  constexpr int NW = TH / 32, RPW = (4 * TC + NW - 1) / NW;
  static_assert(RPW <= 32, "one restriction unit per thread");
  const int lane = t & 31, ru = (t >> 5) * RPW + lane;
  const int ci = ru >> 2, rcg = ru & 3, I = CX0 + ci;
  const bool rest = lane < RPW && ru < 4 * TC && I < int(gc.n0);
  const int rt = (2 * ci + 4) * 4 + rcg;
  const bool rxm = 2 * I - 1 >= 0, rxp = 2 * I + 1 < n0;
  const int64_t rcbase = int64_t(I) * kK8 + rcg * 2, rcstride = int64_t(gc.n0) * kK8;

  const int jbeg = Y0 - 3;                                    // first step (x1 row)
  const int jA0 = max(jbeg, 0), jA1 = min(Y1 + 1, n1 - 1);    // x1 rows = staged rows
  const int yB0 = max(Y0 - 2, 0), yB1 = min(Y1, n1 - 1);      // x2 rows
  const int yC0 = max(Y0 - 1, 0), yC1 = min(Y1 - 1, n1 - 1);  // r rows (and restriction)
  const int jend = yC1 + 5;                                   // last step (restriction of row yC1)

  for (int i = t; i < int((P::BYTES - P::OFF_SLOTS) / 16); i += TH)
    reinterpret_cast<float4*>(sm + P::OFF_SLOTS)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (t == 0) {
    for (int p = 0; p < PD; ++p) tma::mbar_init(&bars[p], 1);
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();
  const uint32_t nb = uint32_t(sb - sa);
  // staged row r (in [jA0, jA1]) goes to slot (r - jA0) % PD
  auto produce = [&](int r) {
    if (r < jA0 || r > jA1) return;
    tma::fence_proxy_async();
    const int sl = (r - jA0) % PD;
    unsigned char* slot = sm + P::OFF_SLOTS + sl * P::SLOT;
    const int64_t node0 = int64_t(n0) * r + gx0 + sa;
    tma::mbar_arrive_expect_tx(&bars[sl], nb * uint32_t((10 + kK8) * sizeof(float2)));
    tma::bulk_g2s(slot + size_t(sa) * 10 * sizeof(float2), op.cd + node0 * 10, nb * uint32_t(10 * sizeof(float2)),
                  &bars[sl]);
    tma::bulk_g2s(slot + P::CROW + size_t(sa) * kK8 * sizeof(float2), b + node0 * kK8,
                  nb * uint32_t(kK8 * sizeof(float2)), &bars[sl]);
  };
  if (t == 0)
    for (int p = 0; p < PD; ++p) produce(jA0 + p);
  auto slot_of = [&](int r) { return sm + P::OFF_SLOTS + ((r - jA0) % PD) * P::SLOT; };
  // (A u)[this thread's 2 columns] of row y from three ring rows, coefficients from the row's records
  auto ax9 = [&](const unsigned char* srow, const float4* rm, const float4* r0, const float4* rp, float2 (&acc)[2],
                 float4& centre) {
    const float2* cf = reinterpret_cast<const float2*>(srow) + xs * 10;
    const float4* xr[3] = {rm, r0, rp};
    float2 av[9];
    float4 xv[9];
#pragma unroll
    for (int sdx = 0; sdx < 9; ++sdx) {
      const int dy = sdx / 3 - 1, dx = sdx % 3 - 1;
      av[sdx] = cf[sdx];
      xv[sdx] = xr[dy + 1][(xs + dx) * 4 + cg];
    }
    acc[0] = acc[1] = czero<float2>();
#pragma unroll
    for (int sdx = 0; sdx < 9; ++sdx) {
      acc[0] = cfma(av[sdx], make_float2(xv[sdx].x, xv[sdx].y), acc[0]);
      acc[1] = cfma(av[sdx], make_float2(xv[sdx].z, xv[sdx].w), acc[1]);
    }
    centre = xv[4];
  };
  float2 racc[2] = {czero<float2>(), czero<float2>()};
  for (int j = jbeg; j <= jend; ++j) {
    // (D) restriction of r row y = j - 5
    {
      const int y = j - 5;
      if (rest && y >= yC0 && y <= yC1) {
        const float4* rr = rs + (y & 1) * RU;
        const Unit<float, 2> rv0 = f42u(rr[rt]);
        const Unit<float, 2> rvm = rxm ? f42u(rr[rt - 4]) : rv0, rvp = rxp ? f42u(rr[rt + 4]) : rv0;
        restrict_row(y, n1, CY0, CY1, rcbase, rcstride, rxm, rxp, rvm, rv0, rvp, racc, rc);
      }
    }
    // (C) r row y = j - 4 = b - A x2
    {
      const int y = j - 4;
      float4 rv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inx && xs >= 2 && xs < NT - 2 && y >= yC0 && y <= yC1) {
        const unsigned char* srow = slot_of(y);
        float2 a[2];
        float4 c4;
        ax9(srow, x2s + ((y + 3) & 3) * RU, x2s + (y & 3) * RU, x2s + ((y + 1) & 3) * RU, a, c4);
        const float4 bv = reinterpret_cast<const float4*>(srow + P::CROW)[t];
        const float2 r0 = csub(make_float2(bv.x, bv.y), a[0]), r1 = csub(make_float2(bv.z, bv.w), a[1]);
        rv = make_float4(r0.x, r0.y, r1.x, r1.y);
      }
      rs[(y & 1) * RU + t] = rv;
    }
    // (B) x2 row y = j - 2 = x1 + wD^-1 (b - A x1)
    {
      const int y = j - 2;
      float4 o4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (inx && xs >= 1 && xs < NT - 1 && y >= yB0 && y <= yB1) {
        const unsigned char* srow = slot_of(y);
        float2 a[2];
        float4 c4;
        ax9(srow, x1s + ((y + 3) & 3) * RU, x1s + (y & 3) * RU, x1s + ((y + 1) & 3) * RU, a, c4);
        const float4 bv = reinterpret_cast<const float4*>(srow + P::CROW)[t];
        const float2 d = (reinterpret_cast<const float2*>(srow) + xs * 10)[9];
        const float2 wd = mk(wj * d.x, wj * d.y);
        float2 o[2];
        o[0] = jacobi_upd(make_float2(c4.x, c4.y), wd, make_float2(bv.x, bv.y), a[0]);
        o[1] = jacobi_upd(make_float2(c4.z, c4.w), wd, make_float2(bv.z, bv.w), a[1]);
        o4 = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
        if (own_x && y >= Y0 && y < Y1) gstore(x2out + (int64_t(n0) * y + gx) * kK8 + cg * 2, o);
      }
      x2s[(y & 3) * RU + t] = o4;
    }
    // (A) x1 row j = wD^-1 b
    {
      float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j >= jA0 && j <= jA1) {
        const int u = j - jA0;
        tma::mbar_wait(&bars[u % PD], uint32_t((u / PD) & 1));
        if (inx) {
          const unsigned char* srow = slot_of(j);
          const float2 d = (reinterpret_cast<const float2*>(srow) + xs * 10)[9];
          const float2 wd = mk(wj * d.x, wj * d.y);
          const float4 bv = reinterpret_cast<const float4*>(srow + P::CROW)[t];
          const float2 a = cmul(wd, make_float2(bv.x, bv.y)), c = cmul(wd, make_float2(bv.z, bv.w));
          x1 = make_float4(a.x, a.y, c.x, c.y);
        }
      }
      x1s[(j & 3) * RU + t] = x1;
    }
    __syncthreads();  // row j - 4's slot is free: the r stage was its last reader
    if (t == 0 && j - 4 >= jA0) produce(j - 4 + PD);
  }
}

void run_stencil9_pre_k8(const LevelOp<float>& op, const LevelGeom& gc, float wj, const float2* b, float2* x2,
                         float2* rc, cudaStream_t s) {
  constexpr int NT = 64, PD = 7;
  using P = S9PrePlan<NT, PD>;
  constexpr int MINB = int(std::min<size_t>(std::min<size_t>((227 * 1024) / (P::BYTES + 1024), 2048 / P::TH), 8));
  const int strips = int((gc.n0 + P::TC - 1) / P::TC);
  // coarse rows per CTA: about one resident wave, at least 4 (5 extra fine rows are staged per chunk)
  const int chunks = std::max(1, kNumSMs * MINB / std::max(1, strips));
  const int e = env_int("HZ_S9PRE_ROWS", 0);
  const int crows = e > 0 ? e : std::max(4, int((gc.n1 + chunks - 1) / chunks));
  const dim3 grid(unsigned(strips), unsigned((gc.n1 + crows - 1) / crows));
  auto kern = stencil9_pre_k8_kernel<NT, PD, MINB>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), int(P::BYTES));
  kern<<<grid, P::TH, P::BYTES, s>>>(op, gc, wj, b, x2, rc, crows);
}

bool launch_stencil9_pre_k8(const LevelOp<float>& op, const LevelGeom& gc, float wj, const float2* b, float2* x2,
                            float2* rc, cudaStream_t s) {
  // opt-in (HZ_S9_PRE=1): measured neutral to slightly slower on the bench (73.0 vs 73.6 RHS/s in interleaved
  // repetitions, profiles/r02_s9_pre_ab.txt) although it replaces 37.5 us of kernels by 26.7 us -- with four
  // groups in flight its 104 KB of shared memory per CTA displaces the other groups' kernels
  static const bool on = env_int("HZ_S9_PRE", 0) != 0;
  static const int64_t min_nodes = env_int("HZ_S9_PRE_MIN_NODES", 100000);
  if (!on || op.kind != kStencil || op.ndim != 2 || op.g.k != kK8 || !op.cd || op.g.z0 != 0 ||
      op.g.z1 != op.g.n1 || int64_t(op.g.nodes) < min_nodes || op.g.n1 < 5)
    return false;
  const double n = double(op.g.nodes), nc = double(gc.nodes);
  ProfScope prof("fused_pre_stencil_c64_L1", n * (kK8 * 8.0 * 2.0 + 80.0) + nc * kK8 * 8.0, s);
  run_stencil9_pre_k8(op, gc, wj, b, x2, rc, s);
  HZ_LAUNCH_CHECK();
  return true;
}

bool fused_vcycle_enabled() {
  static const bool on = env_int("HZ_FUSED_VCYCLE", 1) != 0;
  return on;
}

template <class T>
bool fused_fine_vcycle_ok(const LevelOp<T>& op) {
  return fused_vcycle_enabled() && op.kind == kFine && op.ndim == 2 && op.g.n2 == 1 &&
         op.g.k % (kTPN * cpt<T>()) == 0 && op.g.z0 == 0 && op.g.z1 == op.g.n1;
}

template <class T, class In>
void launch_fused_pre(const LevelOp<T>& op, const LevelGeom& gc, T wj, const In* b, cplx_t<T>* x2,
                      cplx_t<T>* rc, cudaStream_t s) {
  static const int crows = std::max(1, env_int("HZ_FUSED_PRE_ROWS", 16));
  const double n = double(op.g.nodes), nc = double(gc.nodes), k = op.g.k, s_ = sizeof(cplx_t<T>);
  ProfScope prof(sizeof(T) == 8 ? "fused_pre_fine_c128" : "fused_pre_fine_c64",
                 n * (k * (sizeof(In) + s_) + 2.0 * s_) + nc * k * s_, s);
  if constexpr (std::is_same<T, float>::value) {
    if (k8_enabled(int(op.g.k), op.cd)) {
      run_fused_pre_k8<In>(op, gc, wj, b, x2, rc, s);
      HZ_LAUNCH_CHECK();
      return;
    }
  }
  if (fused_wide<T>(int(op.g.k))) {
    constexpr int QW = 2 * cpt<T>();
    const int nt = fused_nt(int(op.g.k), kTPN * QW);
    if (nt == 32)
      run_fused_pre<T, In, 32, QW>(op, gc, wj, b, x2, rc, crows, s);
    else
      run_fused_pre<T, In, 64, QW>(op, gc, wj, b, x2, rc, crows, s);
  } else {
    const int nt = fused_nt(int(op.g.k), kTPN * cpt<T>());
    if (nt == 32)
      run_fused_pre<T, In, 32, cpt<T>()>(op, gc, wj, b, x2, rc, crows, s);
    else if (nt == 64)
      run_fused_pre<T, In, 64, cpt<T>()>(op, gc, wj, b, x2, rc, crows, s);
    else
      run_fused_pre<T, In, 128, cpt<T>()>(op, gc, wj, b, x2, rc, crows, s);
  }
  HZ_LAUNCH_CHECK();
}

template <class T, class In, class Out>
void launch_fused_post(const LevelOp<T>& op, const LevelGeom& gc, T wj, const cplx_t<T>* x2,
                       const cplx_t<T>* ec, const In* b, Out* out, cudaStream_t s) {
  static const int frows = std::max(1, env_int("HZ_FUSED_POST_ROWS", 32));
  const double n = double(op.g.nodes), nc = double(gc.nodes), k = op.g.k, s_ = sizeof(cplx_t<T>);
  ProfScope prof(sizeof(T) == 8 ? "fused_post_fine_c128" : "fused_post_fine_c64",
                 n * (k * (s_ + sizeof(In) + sizeof(Out)) + 2.0 * s_) + nc * k * s_, s);
  if constexpr (std::is_same<T, float>::value) {
    if (k8_enabled(int(op.g.k), op.cd)) {
      run_fused_post_k8<In, Out>(op, gc, wj, x2, ec, b, out, s);
      HZ_LAUNCH_CHECK();
      return;
    }
  }
  if (fused_wide<T>(int(op.g.k))) {
    constexpr int QW = 2 * cpt<T>();
    const int nt = fused_nt(int(op.g.k), kTPN * QW);
    if (nt == 32)
      run_fused_post<T, In, Out, 32, QW>(op, gc, wj, x2, ec, b, out, frows, s);
    else
      run_fused_post<T, In, Out, 64, QW>(op, gc, wj, x2, ec, b, out, frows, s);
  } else {
    const int nt = fused_nt(int(op.g.k), kTPN * cpt<T>());
    if (nt == 32)
      run_fused_post<T, In, Out, 32, cpt<T>()>(op, gc, wj, x2, ec, b, out, frows, s);
    else if (nt == 64)
      run_fused_post<T, In, Out, 64, cpt<T>()>(op, gc, wj, x2, ec, b, out, frows, s);
    else
      run_fused_post<T, In, Out, 128, cpt<T>()>(op, gc, wj, x2, ec, b, out, frows, s);
  }
  HZ_LAUNCH_CHECK();
}

template bool fused_fine_vcycle_ok<float>(const LevelOp<float>&);
template bool fused_fine_vcycle_ok<double>(const LevelOp<double>&);
template void launch_fused_pre<float, double2>(const LevelOp<float>&, const LevelGeom&, float, const double2*,
                                               float2*, float2*, cudaStream_t);
template void launch_fused_pre<float, float2>(const LevelOp<float>&, const LevelGeom&, float, const float2*,
                                              float2*, float2*, cudaStream_t);
template void launch_fused_pre<double, double2>(const LevelOp<double>&, const LevelGeom&, double, const double2*,
                                                double2*, double2*, cudaStream_t);
template void launch_fused_post<float, double2, double2>(const LevelOp<float>&, const LevelGeom&, float,
                                                         const float2*, const float2*, const double2*, double2*,
                                                         cudaStream_t);
template void launch_fused_post<float, double2, float2>(const LevelOp<float>&, const LevelGeom&, float,
                                                        const float2*, const float2*, const double2*, float2*,
                                                        cudaStream_t);
template void launch_fused_post<float, float2, float2>(const LevelOp<float>&, const LevelGeom&, float,
                                                       const float2*, const float2*, const float2*, float2*,
                                                       cudaStream_t);
template void launch_fused_post<double, double2, double2>(const LevelOp<double>&, const LevelGeom&, double,
                                                          const double2*, const double2*, const double2*,
                                                          double2*, cudaStream_t);

}  // namespace hz
