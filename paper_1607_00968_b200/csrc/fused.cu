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
