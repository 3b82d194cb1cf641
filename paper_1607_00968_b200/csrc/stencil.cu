// Grid kernels of the shifted-Laplacian multigrid and the Helmholtz operator
// over node-major RHS-interleaved blocks x[node][k] (inc/block.hpp:13-27).
//
// Thread mapping: one thread per (node, column) element, consecutive threads
// on consecutive elements, so every warp-wide load of a neighbour plane is a
// contiguous, fully coalesced 512 B (c128) / 256 B (c64) transaction and each
// per-node coefficient is fetched once per warp and broadcast across the k
// columns that share it. x-neighbours hit L1; y/z neighbour planes were
// fetched moments earlier by neighbouring CTAs and hit the 126 MB L2, so HBM
// sees (close to) one read per input and one write per output: these kernels
// are HBM-bandwidth bound.
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "profile.hpp"
#include "block_k8.cuh"

namespace hz {

namespace {

constexpr int kBlock = 256;

template <class T>
struct Elem {
  uint32_t node, col, i, j, kz;
};

template <class T>
__device__ __forceinline__ bool decode(const LevelGeom& g, uint32_t e, Elem<T>& el) {
  if (e >= g.e_end()) return false;
  g.div_k.divmod(e, el.node, el.col);
  g.unpack(el.node, el.i, el.j, el.kz);
  return true;
}

// (A x)[e] for the fine 5/7-point operator.
// CSR=false: HelmholtzProblem::apply_block order -- centre first, then
//            x-, x+, y-, y+, z-, z+ (src/helmholtz.cpp:85-98).
// CSR=true : Csr::mul_block order over the sorted row -- z-, y-, x-, centre,
//            x+, y+, z+ (inc/csr.hpp:43-53), used by the multigrid levels.
// widening load: XV = the level's complex type, or complex64 read into complex128
template <class V, class XV>
__device__ __forceinline__ V ldw(const XV* p) {
  if constexpr (std::is_same<V, XV>::value) {
    return __ldg(p);
  } else {
    const XV v = __ldg(p);
    return mk(double(v.x), double(v.y));
  }
}

template <class T, int NDIM, bool CSR, class XV = cplx_t<T>>
__device__ __forceinline__ cplx_t<T> fine_ax(const LevelOp<T>& op, const XV* __restrict__ x,
                                             uint32_t e, const Elem<T>& el) {
  using V = cplx_t<T>;
  const LevelGeom& g = op.g;
  const uint32_t sx = g.k, sy = g.n0 * g.k, sz = g.n0 * g.n1 * g.k;
  // All loads are issued before any arithmetic (out-of-range neighbours read
  // the centre element and are dropped by a select, not a branch), so each
  // thread has its 5-7 independent loads in flight at once instead of a
  // chain of dependent round trips.
  const bool xm = el.i > 0, xp = el.i + 1 < g.n0, ym = el.j > 0, yp = el.j + 1 < g.n1;
  const bool zm = NDIM == 3 && el.kz > 0, zp = NDIM == 3 && el.kz + 1 < g.n2;
  const V c = __ldg(&op.center[el.node]);
  const V u0 = ldw<V>(&x[e]);
  const V uxm = ldw<V>(&x[xm ? e - sx : e]), uxp = ldw<V>(&x[xp ? e + sx : e]);
  const V uym = ldw<V>(&x[ym ? e - sy : e]), uyp = ldw<V>(&x[yp ? e + sy : e]);
  V uzm = u0, uzp = u0;
  if (NDIM == 3) {
    uzm = ldw<V>(&x[zm ? e - sz : e]);
    uzp = ldw<V>(&x[zp ? e + sz : e]);
  }
  const T wx = op.w[0], wy = op.w[1], wz = op.w[2];
  V acc;
  if (!CSR) {
    acc = cmul(c, u0);
    if (xm) acc = crfma(wx, uxm, acc);
    if (xp) acc = crfma(wx, uxp, acc);
    if (ym) acc = crfma(wy, uym, acc);
    if (yp) acc = crfma(wy, uyp, acc);
    if (zm) acc = crfma(wz, uzm, acc);
    if (zp) acc = crfma(wz, uzp, acc);
  } else {
    acc = czero<V>();
    if (zm) acc = crfma(wz, uzm, acc);
    if (ym) acc = crfma(wy, uym, acc);
    if (xm) acc = crfma(wx, uxm, acc);
    acc = cfma(c, u0, acc);
    if (xp) acc = crfma(wx, uxp, acc);
    if (yp) acc = crfma(wy, uyp, acc);
    if (zp) acc = crfma(wz, uzp, acc);
  }
  return acc;
}

// (A x)[e] for a Galerkin 9/27-point stencil, ascending CSR column order.
template <class T, int NDIM>
__device__ __forceinline__ cplx_t<T> stencil_ax(const LevelOp<T>& op,
                                                const cplx_t<T>* __restrict__ x, uint32_t e,
                                                const Elem<T>& el) {
  using V = cplx_t<T>;
  const LevelGeom& g = op.g;
  const int64_t sx = g.k, sy = int64_t(g.n0) * g.k, sz = int64_t(g.n0) * g.n1 * g.k;
  const V* __restrict__ cf = op.coef + el.node;
  constexpr int S = NDIM == 3 ? 27 : 9;
  // Issue every coefficient and neighbour load first (out-of-range
  // neighbours read the centre and are masked), then accumulate in the
  // ascending-column order of the reference's CSR row.
  V av[S], xv[S];
  bool ok[S];
  const int zlo = NDIM == 3 ? -1 : 0, zhi = NDIM == 3 ? 1 : 0;
#pragma unroll
  for (int dz = zlo; dz <= zhi; ++dz) {
    const bool okz = NDIM == 2 || (dz < 0 ? el.kz > 0 : (dz > 0 ? el.kz + 1 < g.n2 : true));
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const bool oky = dy < 0 ? el.j > 0 : (dy > 0 ? el.j + 1 < g.n1 : true);
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const bool okx = dx < 0 ? el.i > 0 : (dx > 0 ? el.i + 1 < g.n0 : true);
        const int s = (NDIM == 3 ? (dz + 1) * 9 : 0) + (dy + 1) * 3 + (dx + 1);
        ok[s] = okz && oky && okx;
        av[s] = __ldg(&cf[int64_t(s) * g.nodes]);
        xv[s] = __ldg(&x[ok[s] ? int64_t(e) + dz * sz + dy * sy + dx * sx : int64_t(e)]);
      }
    }
  }
  V acc = czero<V>();
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (ok[s]) acc = cfma(av[s], xv[s], acc);
  return acc;
}

template <class T, int NDIM, int KIND, bool CSR>
__device__ __forceinline__ cplx_t<T> level_ax(const LevelOp<T>& op, const cplx_t<T>* x, uint32_t e,
                                              const Elem<T>& el) {
  if constexpr (KIND == kFine)
    return fine_ax<T, NDIM, CSR>(op, x, e, el);
  else
    return stencil_ax<T, NDIM>(op, x, e, el);
}

// MODE 0: out = A x ; 1: out = b - A x ; 2: out = x + (wj dinv)(b - A x)
// MODE 3: out = b - A x with A x in apply_block order (the fused form of
// apply + axpby(-1, r, 1, b): bitwise the same values)
template <class T, int NDIM, int KIND, int MODE>
__global__ void __launch_bounds__(kBlock)
level_kernel(LevelOp<T> op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b,
             cplx_t<T>* __restrict__ out, T wj) {
  using V = cplx_t<T>;
  const uint32_t e = op.g.e_begin() + blockIdx.x * kBlock + threadIdx.x;
  Elem<T> el;
  if (!decode(op.g, e, el)) return;
  const V ax = level_ax<T, NDIM, KIND, MODE == 1 || MODE == 2>(op, x, e, el);
  if (MODE == 0) {
    out[e] = ax;
  } else if (MODE == 1 || MODE == 3) {
    out[e] = csub(__ldg(&b[e]), ax);
  } else {
    const V d = __ldg(&op.inv_diag[el.node]);
    const V wd = mk(wj * d.x, wj * d.y);
    out[e] = KIND == kFine ? cadd(__ldg(&x[e]), cmul(wd, csub(__ldg(&b[e]), ax)))
                           : jacobi_upd(__ldg(&x[e]), wd, __ldg(&b[e]), ax);
  }
}

// out = A x for the complex128 fine operator with x a complex64 block
// (widened on load, exact): the apply_block arithmetic of level_kernel
// MODE 0 on the same values, reading half the bytes of x.
template <int NDIM>
__global__ void __launch_bounds__(kBlock)
apply_lo_kernel(LevelOp<double> op, const float2* __restrict__ x, double2* __restrict__ out) {
  const uint32_t e = op.g.e_begin() + blockIdx.x * kBlock + threadIdx.x;
  Elem<double> el;
  if (!decode(op.g, e, el)) return;
  out[e] = fine_ax<double, NDIM, false, float2>(op, x, e, el);
}

// the same for two consecutive columns per thread (k even): 16-byte loads of
// the complex64 block, 32 bytes stored; per column the operations of fine_ax
// in the same order (apply_block: centre, x-, x+, y-, y+, z-, z+)
template <int NDIM>
__global__ void __launch_bounds__(kBlock)
apply_lo2_kernel(LevelOp<double> op, const float2* __restrict__ x, double2* __restrict__ out) {
  const LevelGeom& g = op.g;
  const uint32_t e = g.e_begin() + (blockIdx.x * kBlock + threadIdx.x) * 2;
  if (e >= g.e_end()) return;
  uint32_t node, col, i, j, kz;
  g.div_k.divmod(e, node, col);
  g.unpack(node, i, j, kz);
  const uint32_t sx = g.k, sy = g.n0 * g.k, sz = g.n0 * g.n1 * g.k;
  const bool xm = i > 0, xp = i + 1 < g.n0, ym = j > 0, yp = j + 1 < g.n1;
  const bool zm = NDIM == 3 && kz > 0, zp = NDIM == 3 && kz + 1 < g.n2;
  auto ld = [&](uint32_t at) { return __ldg(reinterpret_cast<const float4*>(x + at)); };
  const double2 c = __ldg(&op.center[node]);
  const float4 u0 = ld(e), uxm = ld(xm ? e - sx : e), uxp = ld(xp ? e + sx : e), uym = ld(ym ? e - sy : e),
               uyp = ld(yp ? e + sy : e);
  float4 uzm = u0, uzp = u0;
  if (NDIM == 3) {
    uzm = ld(zm ? e - sz : e);
    uzp = ld(zp ? e + sz : e);
  }
  const double wx = op.w[0], wy = op.w[1], wz = op.w[2];
  auto col_of = [](const float4& v, int q) { return q == 0 ? mk(double(v.x), double(v.y)) : mk(double(v.z), double(v.w)); };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    double2 acc = cmul(c, col_of(u0, q));
    if (xm) acc = crfma(wx, col_of(uxm, q), acc);
    if (xp) acc = crfma(wx, col_of(uxp, q), acc);
    if (ym) acc = crfma(wy, col_of(uym, q), acc);
    if (yp) acc = crfma(wy, col_of(uyp, q), acc);
    if (zm) acc = crfma(wz, col_of(uzm, q), acc);
    if (zp) acc = crfma(wz, col_of(uzp, q), acc);
    out[e + q] = acc;
  }
}

// W = A Z (complex128 fine operator, Z complex64 widened on load, K = 8)
// fused with the Gram [X_0..X_{NB-2}, W]^H W of the Arnoldi step: the
// register-direct k8::gram8_kernel with its Y = X_{NB-1} operand computed in
// the kernel (apply_lo_kernel's expression on the same values) and stored as
// W, so W is written once and never re-read for the Gram. Rows go to warps
// and slots exactly as in gram8_kernel: the partials are bitwise those of
// apply_lo + gram8.
template <int NB, int NDIM>
__global__ void __launch_bounds__(k8::kThreads, k8::Gram8Cfg<NB>::MINB)
gram8_apply_kernel(LevelOp<double> op, const float2* __restrict__ Z, double2* __restrict__ W,
                   const BlockTab<double> X, double2* __restrict__ partials) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int slot = blockIdx.x, nslots = gridDim.x;
  const int64_t n = op.g.nodes;
  const int64_t groups = (n + k8::kRowsPerStep - 1) / k8::kRowsPerStep;
  const int64_t per = (groups + nslots - 1) / nslots;
  const int64_t g0 = int64_t(slot) * per;
  const int64_t g1 = (g0 + per) < groups ? (g0 + per) : groups;
  double acc[NB][3][2];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int m = 0; m < 3; ++m) acc[i][m][0] = acc[i][m][1] = 0.0;
  constexpr int kUnroll = k8::Gram8Cfg<NB>::U;
  for (int64_t rg = g0 + warp; rg < g1; rg += 8 * kUnroll) {
    double2 y[kUnroll], x[kUnroll][NB];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t row = (rg + 8 * u) * k8::kRowsPerStep + t;
      const bool ok = rg + 8 * u < g1 && row < n;
      const uint32_t e = uint32_t(row * 8 + g);
      y[u] = czero<double2>();
      if (ok) {
        Elem<double> el;
        el.node = uint32_t(row);
        el.col = uint32_t(g);
        op.g.unpack(el.node, el.i, el.j, el.kz);
        y[u] = fine_ax<double, NDIM, false, float2>(op, Z, e, el);
        W[e] = y[u];
      }
#pragma unroll
      for (int i = 0; i < NB - 1; ++i) x[u][i] = ok ? __ldg(X.p[i] + e) : czero<double2>();
      x[u][NB - 1] = y[u];
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
  for (int e = threadIdx.x; e < NB * 64; e += k8::kThreads) out[e] = red[e];
}

template <int NB>
void gram8_apply_dispatch(int nb, const LevelOp<double>& op, const float2* Z, double2* W, const BlockTab<double>& X,
                          double2* partials, int nslots, cudaStream_t s) {
  if constexpr (NB <= 12) {
    if (nb == NB) {
      if (op.ndim == 3)
        gram8_apply_kernel<NB, 3><<<nslots, k8::kThreads, 0, s>>>(op, Z, W, X, partials);
      else
        gram8_apply_kernel<NB, 2><<<nslots, k8::kThreads, 0, s>>>(op, Z, W, X, partials);
      return;
    }
    gram8_apply_dispatch<NB + 1>(nb, op, Z, W, X, partials, nslots, s);
  }
}

// Galerkin 9/27-point level kernel, CPT consecutive columns per thread: the
// neighbour index math and the coefficient loads (shared by all k columns of
// a node) are amortised over CPT outputs -- the one-column-per-thread form
// is instruction-issue bound at 27 neighbours. Branch-free: out-of-range
// neighbours have exactly zero Galerkin coefficients and read the centre.
template <class T, int NDIM, int MODE, int CPT>
__global__ void __launch_bounds__(kBlock)
stencil_mc_kernel(LevelOp<T> op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b,
                  cplx_t<T>* __restrict__ out, T wj) {
  using V = cplx_t<T>;
  const LevelGeom& g = op.g;
  const uint32_t t = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t e0 = g.e_begin() + t * CPT;
  if (e0 >= g.e_end()) return;
  uint32_t node, col, i, j, kz;
  g.div_k.divmod(e0, node, col);
  g.unpack(node, i, j, kz);
  const int64_t sx = g.k, sy = int64_t(g.n0) * g.k, sz = int64_t(g.n0) * g.n1 * g.k;
  const V* __restrict__ cf = op.coef + node;
  V acc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) acc[c] = czero<V>();
  const int zlo = NDIM == 3 ? -1 : 0, zhi = NDIM == 3 ? 1 : 0;
#pragma unroll
  for (int dz = zlo; dz <= zhi; ++dz) {
    const bool okz = NDIM == 2 || (dz < 0 ? kz > 0 : (dz > 0 ? kz + 1 < g.n2 : true));
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const bool oky = dy < 0 ? j > 0 : (dy > 0 ? j + 1 < g.n1 : true);
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const bool okx = dx < 0 ? i > 0 : (dx > 0 ? i + 1 < g.n0 : true);
        const int s = (NDIM == 3 ? (dz + 1) * 9 : 0) + (dy + 1) * 3 + (dx + 1);
        const int64_t off = (okz && oky && okx) ? dz * sz + dy * sy + dx * sx : 0;
        const V a = __ldg(&cf[int64_t(s) * g.nodes]);
        const V* xp = x + int64_t(e0) + off;
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[c] = cfma(a, __ldg(&xp[c]), acc[c]);
      }
    }
  }
  if (MODE == 0) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) out[e0 + c] = acc[c];
  } else if (MODE == 1) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) out[e0 + c] = csub(__ldg(&b[e0 + c]), acc[c]);
  } else {
    const V d = __ldg(&op.inv_diag[node]);
    const V wd = mk(wj * d.x, wj * d.y);
#pragma unroll
    for (int c = 0; c < CPT; ++c)
      out[e0 + c] = jacobi_upd(__ldg(&x[e0 + c]), wd, __ldg(&b[e0 + c]), acc[c]);
  }
}

// CPT = 4 consecutive columns of one node with 16-byte loads / stores
__device__ __forceinline__ void ld4(const float2* __restrict__ p, float2 (&v)[4]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = make_float2(a.x, a.y);
  v[1] = make_float2(a.z, a.w);
  v[2] = make_float2(b.x, b.y);
  v[3] = make_float2(b.z, b.w);
}
__device__ __forceinline__ void ld4(const double2* __restrict__ p, double2 (&v)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = __ldg(p + c);
}
__device__ __forceinline__ void st4(float2* p, const float2 (&v)[4]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
}
__device__ __forceinline__ void st4(double2* p, const double2 (&v)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) p[c] = v[c];
}
// CG = true: coherent (L1-bypassing) loads, for data written earlier in the
// same (persistent) kernel -- the read-only path may hold stale lines
template <bool CG>
__device__ __forceinline__ void ld4v(const float2* __restrict__ p, float2 (&v)[4]) {
  if constexpr (CG) {
    const float4 a = __ldcg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldcg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = make_float2(a.x, a.y);
    v[1] = make_float2(a.z, a.w);
    v[2] = make_float2(b.x, b.y);
    v[3] = make_float2(b.z, b.w);
  } else {
    ld4(p, v);
  }
}
template <bool CG>
__device__ __forceinline__ void ld4v(const double2* __restrict__ p, double2 (&v)[4]) {
  if constexpr (CG) {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __ldcg(p + c);
  } else {
    ld4(p, v);
  }
}

// Galerkin level kernel, 4 columns per thread, with every load of a group of
// G neighbours (G = 9: a whole plane; G = 3: one row) issued before its FMAs
// and 16-byte vector loads: the one-load-then-FMA form leaves the kernel
// latency bound (~1.7 TB/s at level 1 of config 2). Same
// accumulation order as stencil_mc_kernel, so the results are bitwise equal.
template <class T, int NDIM, int MODE, int G, bool CG = false>
__device__ __forceinline__ void stencil_v4_item(const LevelOp<T>& op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b, cplx_t<T>* __restrict__ out, T wj, uint32_t t) {
  using V = cplx_t<T>;
  constexpr int CPT = 4;
  const LevelGeom& g = op.g;
  const uint32_t e0 = g.e_begin() + t * CPT;
  if (e0 >= g.e_end()) return;
  uint32_t node, col, i, j, kz;
  g.div_k.divmod(e0, node, col);
  g.unpack(node, i, j, kz);
  const int64_t sx = g.k, sy = int64_t(g.n0) * g.k, sz = int64_t(g.n0) * g.n1 * g.k;
  const V* __restrict__ cf = op.coef + node;
  V acc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) acc[c] = czero<V>();
  constexpr int S = NDIM == 3 ? 27 : 9;
#pragma unroll
  for (int s0 = 0; s0 < S; s0 += G) {
    V av[G], xv[G][CPT];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int s = s0 + q;
      const int dz = NDIM == 3 ? s / 9 - 1 : 0, dy = (s / 3) % 3 - 1, dx = s % 3 - 1;
      const bool okz = NDIM == 2 || (dz < 0 ? kz > 0 : (dz > 0 ? kz + 1 < g.n2 : true));
      const bool oky = dy < 0 ? j > 0 : (dy > 0 ? j + 1 < g.n1 : true);
      const bool okx = dx < 0 ? i > 0 : (dx > 0 ? i + 1 < g.n0 : true);
      const int64_t off = (okz && oky && okx) ? dz * sz + dy * sy + dx * sx : 0;
      av[q] = __ldg(&cf[int64_t(s) * g.nodes]);
      ld4v<CG>(x + int64_t(e0) + off, xv[q]);
    }
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c] = cfma(av[q], xv[q][c], acc[c]);
  }
  V o[CPT];
  if (MODE == 0) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = acc[c];
  } else if (MODE == 1) {
    V bv[CPT];
    ld4v<CG>(b + e0, bv);
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = csub(bv[c], acc[c]);
  } else {
    V bv[CPT], xc[CPT];
    ld4v<CG>(b + e0, bv);
    ld4v<CG>(x + e0, xc);
    const V d = __ldg(&op.inv_diag[node]);
    const V wd = mk(wj * d.x, wj * d.y);
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = jacobi_upd(xc[c], wd, bv[c], acc[c]);
  }
  st4(out + e0, o);
}

// resident CTAs per SM the Galerkin level kernel is compiled for (register
// cap 65536 / (kBlock * HZ_STENCIL_MINB)); 1 = compiler's choice
#ifndef HZ_STENCIL_MINB
#define HZ_STENCIL_MINB 1
#endif
template <class T, int NDIM, int MODE, int G>
__global__ void __launch_bounds__(kBlock, HZ_STENCIL_MINB)
stencil_v4_kernel(LevelOp<T> op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b,
                  cplx_t<T>* __restrict__ out, T wj) {
  stencil_v4_item<T, NDIM, MODE, G>(op, x, b, out, wj, blockIdx.x * kBlock + threadIdx.x);
}

// Compact 27-point fine level (kFine27): the couplings lap[q] + mu[q] (M_i +
// M_j)/2 are formed on the fly from the per-node mass (1 complex per node
// read instead of 27 coefficient planes; each M_j is reused by 27 rows through
// L1), in the same order and arithmetic as build27_kernel, and summed in
// ascending plane order like stencil_v4_item. CPT columns per thread
// (4: 16-byte loads; 1: any k).
template <class T, int MODE, int CPT>
__device__ __forceinline__ void fine27_item(const LevelOp<T>& op, const cplx_t<T>* __restrict__ x,
                                            const cplx_t<T>* __restrict__ b, cplx_t<T>* __restrict__ out, T wj,
                                            uint32_t t) {
  using V = cplx_t<T>;
  const LevelGeom& g = op.g;
  const uint32_t e0 = g.e_begin() + t * CPT;
  if (e0 >= g.e_end()) return;
  uint32_t node, col, i, j, kz;
  g.div_k.divmod(e0, node, col);
  g.unpack(node, i, j, kz);
  const int64_t sx = g.k, sy = int64_t(g.n0) * g.k, sz = int64_t(g.n0) * g.n1 * g.k;
  const int64_t nx = 1, ny = g.n0, nz = int64_t(g.n0) * g.n1;
  const V Mi = __ldg(&op.center[node]);
  const T half = T(0.5);
  V acc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) acc[c] = czero<V>();
  // loads of a group of G neighbours issued before its FMAs: a plane for
  // complex64, a row for complex128 (register budget)
  constexpr int G = sizeof(T) == 8 && CPT == 4 ? 3 : 9;
#pragma unroll
  for (int s0 = 0; s0 < 27; s0 += G) {
    V av[G], xv[G][CPT];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int s = s0 + q;
      const int dz = s / 9 - 1, dy = (s / 3) % 3 - 1, dx = s % 3 - 1;
      const int cls = (dx != 0) + (dy != 0) + (dz != 0);
      const bool okz = dz < 0 ? kz > 0 : (dz > 0 ? kz + 1 < g.n2 : true);
      const bool oky = dy < 0 ? j > 0 : (dy > 0 ? j + 1 < g.n1 : true);
      const bool okx = dx < 0 ? i > 0 : (dx > 0 ? i + 1 < g.n0 : true);
      const bool ok = okz && oky && okx;
      const int64_t off = ok ? dz * sz + dy * sy + dx * sx : 0;
      if (cls == 0) {
        av[q] = mk(op.w27[0] + op.w27[4] * Mi.x, op.w27[4] * Mi.y);
      } else {
        const V Mj = __ldg(&op.center[int64_t(node) + (ok ? dz * nz + dy * ny + dx * nx : 0)]);
        const T avr = half * (Mi.x + Mj.x), avi = half * (Mi.y + Mj.y);
        av[q] = ok ? mk(op.w27[cls] + op.w27[4 + cls] * avr, op.w27[4 + cls] * avi) : czero<V>();
      }
      if constexpr (CPT == 4) {
        ld4(x + int64_t(e0) + off, xv[q]);
      } else {
#pragma unroll
        for (int c = 0; c < CPT; ++c) xv[q][c] = __ldg(x + int64_t(e0) + off + c);
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c] = cfma(av[q], xv[q][c], acc[c]);
  }
  V o[CPT];
  if (MODE == 0) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = acc[c];
  } else if (MODE == 1) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = csub(__ldg(b + e0 + c), acc[c]);
  } else {
    const V d = __ldg(&op.inv_diag[node]);
    const V wd = mk(wj * d.x, wj * d.y);
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[c] = jacobi_upd(__ldg(x + e0 + c), wd, __ldg(b + e0 + c), acc[c]);
  }
  if constexpr (CPT == 4) {
    st4(out + e0, o);
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) out[e0 + c] = o[c];
  }
}

template <class T, int MODE, int CPT>
__global__ void __launch_bounds__(kBlock)
fine27_kernel(LevelOp<T> op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b,
              cplx_t<T>* __restrict__ out, T wj) {
  fine27_item<T, MODE, CPT>(op, x, b, out, wj, blockIdx.x * kBlock + threadIdx.x);
}

// Fine 5/7-point level kernel, 4 columns per thread with 16-byte loads (all
// loads issued first); same per-column arithmetic and order as fine_ax.
template <class T, int NDIM, int MODE, class Out = cplx_t<T>>
__global__ void __launch_bounds__(kBlock)
fine_v4_kernel(LevelOp<T> op, const cplx_t<T>* __restrict__ x, const cplx_t<T>* __restrict__ b,
               Out* __restrict__ out, T wj) {
  using V = cplx_t<T>;
  constexpr int CPT = 4;
  constexpr bool CSR = MODE == 1 || MODE == 2;
  const LevelGeom& g = op.g;
  const uint32_t t = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t e0 = g.e_begin() + t * CPT;
  if (e0 >= g.e_end()) return;
  uint32_t node, col, i, j, kz;
  g.div_k.divmod(e0, node, col);
  g.unpack(node, i, j, kz);
  const uint32_t sx = g.k, sy = g.n0 * g.k, sz = g.n0 * g.n1 * g.k;
  const bool xm = i > 0, xp = i + 1 < g.n0, ym = j > 0, yp = j + 1 < g.n1;
  const bool zm = NDIM == 3 && kz > 0, zp = NDIM == 3 && kz + 1 < g.n2;
  const V c = __ldg(&op.center[node]);
  V u0[CPT], uxm[CPT], uxp[CPT], uym[CPT], uyp[CPT], uzm[CPT], uzp[CPT];
  ld4(x + e0, u0);
  ld4(x + (xm ? e0 - sx : e0), uxm);
  ld4(x + (xp ? e0 + sx : e0), uxp);
  ld4(x + (ym ? e0 - sy : e0), uym);
  ld4(x + (yp ? e0 + sy : e0), uyp);
  if (NDIM == 3) {
    ld4(x + (zm ? e0 - sz : e0), uzm);
    ld4(x + (zp ? e0 + sz : e0), uzp);
  }
  V bv[CPT];
  if (MODE != 0) ld4(b + e0, bv);
  V dv = czero<V>();
  if (MODE == 2) dv = __ldg(&op.inv_diag[node]);
  const T wx = op.w[0], wy = op.w[1], wz = op.w[2];
  V o[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    V acc;
    if (!CSR) {
      acc = cmul(c, u0[q]);
      if (xm) acc = crfma(wx, uxm[q], acc);
      if (xp) acc = crfma(wx, uxp[q], acc);
      if (ym) acc = crfma(wy, uym[q], acc);
      if (yp) acc = crfma(wy, uyp[q], acc);
      if (zm) acc = crfma(wz, uzm[q], acc);
      if (zp) acc = crfma(wz, uzp[q], acc);
    } else {
      acc = czero<V>();
      if (zm) acc = crfma(wz, uzm[q], acc);
      if (ym) acc = crfma(wy, uym[q], acc);
      if (xm) acc = crfma(wx, uxm[q], acc);
      acc = cfma(c, u0[q], acc);
      if (xp) acc = crfma(wx, uxp[q], acc);
      if (yp) acc = crfma(wy, uyp[q], acc);
      if (zp) acc = crfma(wz, uzp[q], acc);
    }
    if (MODE == 0) {
      o[q] = acc;
    } else if (MODE == 1 || MODE == 3) {
      o[q] = csub(bv[q], acc);
    } else {
      const V wd = mk(wj * dv.x, wj * dv.y);
      o[q] = cadd(u0[q], cmul(wd, csub(bv[q], acc)));
    }
  }
  if constexpr (std::is_same<Out, cplx_t<T>>::value) {
    st4(out + e0, o);
  } else {
    Out w[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) w[q] = ccast<Out>(o[q]);
    st4(out + e0, w);
  }
}

// Zero-start sweep fused with the c128 -> c64 cast of the right-hand side
// (complex64 preconditioner): b32 = (c64) b64, x1 = wD^{-1} b32; 4 columns
// per thread, the same per-column operations as cast + jacobi_zero.
__global__ void __launch_bounds__(kBlock)
jacobi_zero_cast_kernel(LevelGeom g, const float2* __restrict__ inv_diag, float wj, const double2* __restrict__ b64,
                        float2* __restrict__ b32, float2* __restrict__ out) {
  const uint32_t e0 = g.e_begin() + (blockIdx.x * kBlock + threadIdx.x) * 4;
  if (e0 >= g.e_end()) return;
  const uint32_t node = g.div_k.div(e0);
  const float2 d = __ldg(&inv_diag[node]);
  const float2 wd = mk(wj * d.x, wj * d.y);
  double2 bb[4];
  ld4(b64 + e0, bb);
  float2 bv[4], o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    bv[q] = ccast<float2>(bb[q]);
    o[q] = cmul(wd, bv[q]);
  }
  st4(b32 + e0, bv);
  st4(out + e0, o);
}

template <class T, class In>
__global__ void __launch_bounds__(kBlock)
jacobi_zero_kernel(LevelGeom g, const cplx_t<T>* __restrict__ inv_diag, T wj,
                   const In* __restrict__ b, cplx_t<T>* __restrict__ out) {
  using V = cplx_t<T>;
  const uint32_t e = g.e_begin() + blockIdx.x * kBlock + threadIdx.x;
  if (e >= g.e_end()) return;
  const uint32_t node = g.div_k.div(e);
  const V d = __ldg(&inv_diag[node]);
  const V wd = mk(wj * d.x, wj * d.y);
  out[e] = cmul(wd, ccast<V>(__ldg(&b[e])));
}

// rc[C] = sum_{f in 3^d box around 2C} w_f r[f], f ascending (the CSR of
// R = P^T visits fine rows in order, inc/csr.hpp:110-127).
template <class T, int NDIM>
__global__ void __launch_bounds__(kBlock)
restrict_kernel(LevelGeom gf, LevelGeom gc, const cplx_t<T>* __restrict__ r,
                cplx_t<T>* __restrict__ bc) {
  using V = cplx_t<T>;
  const uint32_t e = gc.e_begin() + blockIdx.x * kBlock + threadIdx.x;
  Elem<T> el;
  if (!decode(gc, e, el)) return;
  const int64_t k = gf.k;
  constexpr int S = NDIM == 3 ? 27 : 9;
  // loads first (masked, see fine_ax), then the ascending-f accumulation
  V rv[S];
  T wv[S];
  const int64_t fc = (2 * int64_t(el.i) + int64_t(gf.n0) * (2 * int64_t(el.j) + int64_t(gf.n1) * 2 * el.kz)) * k +
                     el.col;
  const int zlo = NDIM == 3 ? -1 : 0, zhi = NDIM == 3 ? 1 : 0;
#pragma unroll
  for (int ez = zlo; ez <= zhi; ++ez) {
    const int64_t fz = 2 * int64_t(el.kz) + ez;
    const bool okz = fz >= 0 && fz < gf.n2;
#pragma unroll
    for (int ey = -1; ey <= 1; ++ey) {
      const int64_t fy = 2 * int64_t(el.j) + ey;
      const bool oky = fy >= 0 && fy < gf.n1;
#pragma unroll
      for (int ex = -1; ex <= 1; ++ex) {
        const int64_t fx = 2 * int64_t(el.i) + ex;
        const bool ok = okz && oky && fx >= 0 && fx < gf.n0;
        const int s = (NDIM == 3 ? (ez + 1) * 9 : 0) + (ey + 1) * 3 + (ex + 1);
        wv[s] = ok ? (ex == 0 ? T(1) : T(0.5)) * (ey == 0 ? T(1) : T(0.5)) * (ez == 0 ? T(1) : T(0.5)) : T(0);
        const int64_t off = (int64_t(ex) + int64_t(gf.n0) * (ey + int64_t(gf.n1) * ez)) * k;
        rv[s] = __ldg(&r[ok ? fc + off : fc]);
      }
    }
  }
  V acc = czero<V>();
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (wv[s] != T(0)) acc = crfma(wv[s], rv[s], acc);
  bc[e] = acc;
}

// x[f] += sum_{C parents of f} w ec[C]  (corr summed first, then added:
// axpby(x, 1, corr, 1), src/multigrid.cpp:195-197)
template <class T, int NDIM>
__global__ void __launch_bounds__(kBlock)
prolong_correct_kernel(LevelGeom gf, LevelGeom gc, const cplx_t<T>* __restrict__ ec,
                       cplx_t<T>* __restrict__ x) {
  using V = cplx_t<T>;
  const uint32_t e = gf.e_begin() + blockIdx.x * kBlock + threadIdx.x;
  Elem<T> el;
  if (!decode(gf, e, el)) return;
  const int64_t k = gf.k;
  // parents per axis: even f -> (f/2, weight 1); odd f -> (f-1)/2, (f+1)/2
  // with 1/2 each. Always gather 2 per axis (the second of an even f has
  // weight 0 and is skipped in the sum), all loads issued up front.
  const uint32_t cx0 = el.i >> 1, cx1 = (el.i + 1) >> 1;
  const uint32_t cy0 = el.j >> 1, cy1 = (el.j + 1) >> 1;
  const uint32_t cz0 = NDIM == 3 ? (el.kz >> 1) : 0, cz1 = NDIM == 3 ? ((el.kz + 1) >> 1) : 0;
  const T wx0 = (el.i & 1u) ? T(0.5) : T(1), wx1 = (el.i & 1u) ? T(0.5) : T(0);
  const T wy0 = (el.j & 1u) ? T(0.5) : T(1), wy1 = (el.j & 1u) ? T(0.5) : T(0);
  const T wz0 = NDIM == 3 && (el.kz & 1u) ? T(0.5) : T(1), wz1 = NDIM == 3 && (el.kz & 1u) ? T(0.5) : T(0);
  constexpr int NZ = NDIM == 3 ? 2 : 1;
  V ev[NZ][2][2];
  T wv[NZ][2][2];
#pragma unroll
  for (int c = 0; c < NZ; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int64_t C = (a ? cx1 : cx0) + int64_t(gc.n0) * ((b ? cy1 : cy0) + int64_t(gc.n1) * (c ? cz1 : cz0));
        ev[c][b][a] = __ldg(&ec[C * k + el.col]);
        wv[c][b][a] = (a ? wx1 : wx0) * (b ? wy1 : wy0) * (c ? wz1 : wz0);
      }
  const V xe = x[e];
  V corr = czero<V>();
#pragma unroll
  for (int c = 0; c < NZ; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a)
        if (wv[c][b][a] != T(0)) corr = crfma(wv[c][b][a], ev[c][b][a], corr);
  x[e] = cadd(xe, corr);
}

// ---- 4-columns-per-thread forms of the transfers and the zero-start sweep
// (16-byte loads, complex64 with k % 4 == 0); per-column arithmetic and
// order exactly as the one-column kernels above.
template <class T, int NDIM, bool CG = false>
__device__ __forceinline__ void restrict_v4_item(const LevelGeom& gf, const LevelGeom& gc, const cplx_t<T>* __restrict__ r, cplx_t<T>* __restrict__ bc, uint32_t t) {
  using V = cplx_t<T>;
  const uint32_t e0 = gc.e_begin() + t * 4;
  if (e0 >= gc.e_end()) return;
  uint32_t node, col, I, J, K;
  gc.div_k.divmod(e0, node, col);
  gc.unpack(node, I, J, K);
  const int64_t k = gf.k;
  constexpr int S = NDIM == 3 ? 27 : 9;
  V rv[S][4];
  T wv[S];
  const int64_t fc = (2 * int64_t(I) + int64_t(gf.n0) * (2 * int64_t(J) + int64_t(gf.n1) * 2 * K)) * k + col;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int ez = NDIM == 3 ? s / 9 - 1 : 0, ey = (s / 3) % 3 - 1, ex = s % 3 - 1;
    const int64_t fz = 2 * int64_t(K) + ez, fy = 2 * int64_t(J) + ey, fx = 2 * int64_t(I) + ex;
    const bool ok = fz >= 0 && fz < gf.n2 && fy >= 0 && fy < gf.n1 && fx >= 0 && fx < gf.n0;
    wv[s] = ok ? (ex == 0 ? T(1) : T(0.5)) * (ey == 0 ? T(1) : T(0.5)) * (ez == 0 ? T(1) : T(0.5)) : T(0);
    const int64_t off = (int64_t(ex) + int64_t(gf.n0) * (ey + int64_t(gf.n1) * ez)) * k;
    ld4v<CG>(r + (ok ? fc + off : fc), rv[s]);
  }
  V o[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    V acc = czero<V>();
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (wv[s] != T(0)) acc = crfma(wv[s], rv[s][c], acc);
    o[c] = acc;
  }
  st4(bc + e0, o);
}

template <class T, int NDIM>
__global__ void __launch_bounds__(kBlock)
restrict_v4_kernel(LevelGeom gf, LevelGeom gc, const cplx_t<T>* __restrict__ r, cplx_t<T>* __restrict__ bc) {
  restrict_v4_item<T, NDIM>(gf, gc, r, bc, blockIdx.x * kBlock + threadIdx.x);
}

template <class T, int NDIM, bool CG = false>
__device__ __forceinline__ void prolong_v4_item(const LevelGeom& gf, const LevelGeom& gc, const cplx_t<T>* __restrict__ ec, cplx_t<T>* __restrict__ x, uint32_t t) {
  using V = cplx_t<T>;
  const uint32_t e0 = gf.e_begin() + t * 4;
  if (e0 >= gf.e_end()) return;
  uint32_t node, col, i, j, kz;
  gf.div_k.divmod(e0, node, col);
  gf.unpack(node, i, j, kz);
  const int64_t k = gf.k;
  const uint32_t cx0 = i >> 1, cx1 = (i + 1) >> 1, cy0 = j >> 1, cy1 = (j + 1) >> 1;
  const uint32_t cz0 = NDIM == 3 ? (kz >> 1) : 0, cz1 = NDIM == 3 ? ((kz + 1) >> 1) : 0;
  const T wx0 = (i & 1u) ? T(0.5) : T(1), wx1 = (i & 1u) ? T(0.5) : T(0);
  const T wy0 = (j & 1u) ? T(0.5) : T(1), wy1 = (j & 1u) ? T(0.5) : T(0);
  const T wz0 = NDIM == 3 && (kz & 1u) ? T(0.5) : T(1), wz1 = NDIM == 3 && (kz & 1u) ? T(0.5) : T(0);
  constexpr int NZ = NDIM == 3 ? 2 : 1;
  V ev[NZ][2][2][4];
  T wv[NZ][2][2];
#pragma unroll
  for (int c = 0; c < NZ; ++c)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int64_t C = (a ? cx1 : cx0) + int64_t(gc.n0) * ((b ? cy1 : cy0) + int64_t(gc.n1) * (c ? cz1 : cz0));
        ld4v<CG>(ec + C * k + col, ev[c][b][a]);
        wv[c][b][a] = (a ? wx1 : wx0) * (b ? wy1 : wy0) * (c ? wz1 : wz0);
      }
  V xe[4], o[4];
  ld4v<CG>(x + e0, xe);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    V corr = czero<V>();
#pragma unroll
    for (int c = 0; c < NZ; ++c)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int a = 0; a < 2; ++a)
          if (wv[c][b][a] != T(0)) corr = crfma(wv[c][b][a], ev[c][b][a][q], corr);
    o[q] = cadd(xe[q], corr);
  }
  st4(x + e0, o);
}

template <class T, int NDIM>
__global__ void __launch_bounds__(kBlock)
prolong_v4_kernel(LevelGeom gf, LevelGeom gc, const cplx_t<T>* __restrict__ ec, cplx_t<T>* __restrict__ x) {
  prolong_v4_item<T, NDIM>(gf, gc, ec, x, blockIdx.x * kBlock + threadIdx.x);
}

template <class T, bool CG = false>
__device__ __forceinline__ void jacobi_zero_v4_item(const LevelGeom& g, const cplx_t<T>* __restrict__ inv_diag, T wj, const cplx_t<T>* __restrict__ b, cplx_t<T>* __restrict__ out, uint32_t t) {
  using V = cplx_t<T>;
  const uint32_t e0 = g.e_begin() + t * 4;
  if (e0 >= g.e_end()) return;
  const uint32_t node = g.div_k.div(e0);
  const V d = __ldg(&inv_diag[node]);
  const V wd = mk(wj * d.x, wj * d.y);
  V bv[4], o[4];
  ld4v<CG>(b + e0, bv);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = cmul(wd, bv[q]);
  st4(out + e0, o);
}

template <class T>
__global__ void __launch_bounds__(kBlock)
jacobi_zero_v4_kernel(LevelGeom g, const cplx_t<T>* __restrict__ inv_diag, T wj, const cplx_t<T>* __restrict__ b,
                      cplx_t<T>* __restrict__ out) {
  jacobi_zero_v4_item<T>(g, inv_diag, wj, b, out, blockIdx.x * kBlock + threadIdx.x);
}

// ---------------------------------------------------------------- Galerkin
// Fine-operator entry A[f][f+o], o in {-1,0,1}^3 (0 if absent).
template <int NDIM, int KIND>
__device__ __forceinline__ double2 fine_entry(const LevelOp<double>& op, int64_t f, int ox, int oy,
                                              int oz) {
  if constexpr (KIND == kFine) {
    const int nz = (ox != 0) + (oy != 0) + (oz != 0);
    if (nz == 0) return op.center[f];
    if (nz > 1) return make_double2(0.0, 0.0);
    const int a = ox != 0 ? 0 : (oy != 0 ? 1 : 2);
    return make_double2(op.w[a], 0.0);
  } else {
    const int s = (NDIM == 3 ? (oz + 1) * 9 : 0) + (oy + 1) * 3 + (ox + 1);
    return op.coef[int64_t(s) * op.g.nodes + f];
  }
}

// One thread per coarse node C. Follows the reference's two Gustavson
// products: AP = A P (row f, g ascending, then P-row targets ascending),
// then (R AP)[C] over f ascending (inc/csr.hpp:130-160). All weights are
// powers of two, so each product is exact and the sums run in the reference
// order.
template <int NDIM, int KIND>
__global__ void __launch_bounds__(128)
galerkin_kernel(LevelOp<double> fine, LevelGeom gc, double2* __restrict__ coef_c) {
  const uint32_t C = blockIdx.x * 128 + threadIdx.x;
  if (C >= gc.nodes) return;
  const LevelGeom& gf = fine.g;
  uint32_t I, J, K;
  gc.unpack(C, I, J, K);
  constexpr int S = NDIM == 3 ? 27 : 9;
  double2 acc[S];
#pragma unroll
  for (int s = 0; s < S; ++s) acc[s] = make_double2(0.0, 0.0);
  const int zlo = NDIM == 3 ? -1 : 0, zhi = NDIM == 3 ? 1 : 0;
  for (int ez = zlo; ez <= zhi; ++ez) {
    const int64_t fz = 2 * int64_t(K) + ez;
    if (fz < 0 || fz >= gf.n2) continue;
    for (int ey = -1; ey <= 1; ++ey) {
      const int64_t fy = 2 * int64_t(J) + ey;
      if (fy < 0 || fy >= gf.n1) continue;
      for (int ex = -1; ex <= 1; ++ex) {
        const int64_t fx = 2 * int64_t(I) + ex;
        if (fx < 0 || fx >= gf.n0) continue;
        const double wf = (ex ? 0.5 : 1.0) * (ey ? 0.5 : 1.0) * (ez ? 0.5 : 1.0);
        const int64_t f = fx + int64_t(gf.n0) * (fy + int64_t(gf.n1) * fz);
        double2 ap[S];
#pragma unroll
        for (int s = 0; s < S; ++s) ap[s] = make_double2(0.0, 0.0);
        // A row f, ascending column: oz, oy, ox
        for (int oz = zlo; oz <= zhi; ++oz) {
          const int64_t gz = fz + oz;
          if (gz < 0 || gz >= gf.n2) continue;
          for (int oy = -1; oy <= 1; ++oy) {
            const int64_t gy = fy + oy;
            if (gy < 0 || gy >= gf.n1) continue;
            for (int ox = -1; ox <= 1; ++ox) {
              const int64_t gx = fx + ox;
              if (gx < 0 || gx >= gf.n0) continue;
              if (KIND == kFine && ((ox != 0) + (oy != 0) + (oz != 0)) > 1) continue;
              const double2 a = fine_entry<NDIM, KIND>(fine, f, ox, oy, oz);
              if (KIND == kStencil && a.x == 0.0 && a.y == 0.0) continue;
              // P row g: parents ascending (z, y, x)
              int64_t pz[2], py[2], px[2];
              double wz[2], wy[2], wx[2];
              int nzp, nyp, nxp;
              auto par = [](int64_t gcoord, int64_t* p, double* w) -> int {
                if ((gcoord & 1) == 0) {
                  p[0] = gcoord / 2;
                  w[0] = 1.0;
                  return 1;
                }
                p[0] = (gcoord - 1) / 2;
                p[1] = (gcoord + 1) / 2;
                w[0] = w[1] = 0.5;
                return 2;
              };
              nxp = par(gx, px, wx);
              nyp = par(gy, py, wy);
              if (NDIM == 3) {
                nzp = par(gz, pz, wz);
              } else {
                nzp = 1;
                pz[0] = 0;
                wz[0] = 1.0;
              }
              for (int c = 0; c < nzp; ++c)
                for (int b = 0; b < nyp; ++b)
                  for (int q = 0; q < nxp; ++q) {
                    const int dx = int(px[q] - I), dy = int(py[b] - J),
                              dz = NDIM == 3 ? int(pz[c] - K) : 0;
                    const int s = (NDIM == 3 ? (dz + 1) * 9 : 0) + (dy + 1) * 3 + (dx + 1);
                    const double p = wx[q] * wy[b] * wz[c];
                    ap[s].x += a.x * p;
                    ap[s].y += a.y * p;
                  }
            }
          }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          acc[s].x += wf * ap[s].x;
          acc[s].y += wf * ap[s].y;
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) coef_c[int64_t(s) * gc.nodes + C] = acc[s];
}

template <class Dst, class Src>
__global__ void __launch_bounds__(kBlock) cast_kernel(int64_t count, const Src* __restrict__ in,
                                                      Dst* __restrict__ out) {
  const int64_t e = int64_t(blockIdx.x) * kBlock + threadIdx.x;
  if (e < count) out[e] = ccast<Dst>(in[e]);
}

template <class T>
constexpr const char* prec_tag() {
  return sizeof(T) == 8 ? "c128" : "c64";
}

// algorithmic bytes of one level_kernel launch: vectors read /
// written once per element, coefficients once per node
template <class T>
double level_bytes(const LevelOp<T>& op, int mode) {
  const double s = sizeof(cplx_t<T>), n = double(op.g.owned_nodes()), k = op.g.k;
  const double coef = op.kind != kStencil ? 1.0 : (op.ndim == 3 ? 27.0 : 9.0);
  const double vec = mode == 0 ? 2.0 : 3.0;
  const double diag = mode == 2 ? 1.0 : 0.0;
  return n * (vec * k * s + (coef + diag) * s);
}

template <class T, int MODE>
const char* level_name(int kind, int level) {
  static const char* names[3][3][2] = {
      {{"apply_fine_c128", "apply_fine_c64"}, {"residual_fine_c128", "residual_fine_c64"},
       {"jacobi_fine_c128", "jacobi_fine_c64"}},
      {{"apply_stencil_c128", "apply_stencil_c64"}, {"residual_stencil_c128", "residual_stencil_c64"},
       {"jacobi_stencil_c128", "jacobi_stencil_c64"}},
      {{"apply_fine27_c128", "apply_fine27_c64"}, {"residual_fine27_c128", "residual_fine27_c64"},
       {"jacobi_fine27_c128", "jacobi_fine27_c64"}}};
  const char* base = names[kind][MODE][sizeof(T) == 8 ? 0 : 1];
  if (kind != kStencil) return base;
  // Galerkin levels by level index: level 1 streams from HBM, deeper levels
  // are L2-resident and launch/latency bound, so they are reported apart
  return profile_name_level(base, level);
}

// Below this many (node, column) elements a Galerkin level is latency bound
// and one column per thread (4x the threads in flight) beats the 4-column
// form (HZ_V4_MIN_ELEMS overrides).
int64_t stencil_v4_min_elems() {
  static const int64_t v = [] {
    const char* e = std::getenv("HZ_V4_MIN_ELEMS");
    return e ? int64_t(std::atoll(e)) : int64_t(0);
  }();
  return v;
}

// the bulk-copy 2D Galerkin kernel for levels of at least HZ_S9_MIN_NODES
// nodes (default 100,000: level 1 of config 2, 131k nodes, 12.7 vs 13.3 us;
// level 2, 33k nodes, 9.4 vs 8.6 us -- smaller levels are latency bound and the
// plain kernel starts faster)
template <class T, int MODE>
bool stencil9_bulk(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* out, T wj,
                   cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value) {
    static const int64_t min_nodes = [] {
      const char* e = std::getenv("HZ_S9_MIN_NODES");
      return e ? int64_t(std::atoll(e)) : int64_t(100000);
    }();
    if (int64_t(op.g.nodes) < min_nodes) return false;
    return launch_stencil9_k8(op, MODE, wj, x, b, out, s);
  } else {
    return false;
  }
}

template <class T, int MODE>
bool galerkin3d_stream(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* out, T wj,
                       cudaStream_t s) {
  if constexpr (std::is_same<T, float>::value) {
    if (op.ndim != 3 || !op.cd) return false;
    return launch_galerkin3d(op, MODE, wj, x, b, out, s);
  } else {
    return false;
  }
}

template <class T, int MODE>
void dispatch_level(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* out,
                    T wj, cudaStream_t s) {
  const int64_t total = op.g.owned_elems();
  const int grid = grid_for(total, kBlock);
  ProfScope prof(level_name<T, MODE>(op.kind, op.level), level_bytes(op, MODE), s);
  static const bool fine_v4 = [] {
    const char* e = std::getenv("HZ_FINE_V4");
    return !(e && e[0] == '0');
  }();
  // c64 only: for c128 the 4-column form needs 7 x 64 B per thread in
  // registers and runs slower than one column per thread
  if (launch_stream3d<T, cplx_t<T>>(op, MODE, wj, x, b, out, s)) {
    return;  // 3D fine level, k = 8: plane-streaming kernels (stream3d.cu)
  } else if (op.kind == kFine27) {
    if (op.g.k % 4 == 0)
      fine27_kernel<T, MODE, 4><<<grid_for(total / 4, kBlock), kBlock, 0, s>>>(op, x, b, out, wj);
    else
      fine27_kernel<T, MODE, 1><<<grid, kBlock, 0, s>>>(op, x, b, out, wj);
  } else if (op.kind == kFine && fine_v4 && sizeof(T) == 4 && op.g.k % 4 == 0) {
    const int g4 = grid_for(total / 4, kBlock);
    if (op.ndim == 3)
      fine_v4_kernel<T, 3, MODE><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
    else
      fine_v4_kernel<T, 2, MODE><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
  } else if (op.kind == kFine) {
    if (op.ndim == 3)
      level_kernel<T, 3, kFine, MODE><<<grid, kBlock, 0, s>>>(op, x, b, out, wj);
    else
      level_kernel<T, 2, kFine, MODE><<<grid, kBlock, 0, s>>>(op, x, b, out, wj);
  } else if (galerkin3d_stream<T, MODE>(op, x, b, out, wj, s)) {
    // complex64 3D Galerkin level, k = 8: plane streaming (galerkin3d.cu)
  } else if (stencil9_bulk<T, MODE>(op, x, b, out, wj, s)) {
    // complex64 2D Galerkin level, k = 8: bulk-copy row staging (fused.cu)
  } else if (op.g.k % 4 == 0 && total >= stencil_v4_min_elems()) {
    const int g4 = grid_for(total / 4, kBlock);
    static const int variant = [] {
      const char* e = std::getenv("HZ_STENCIL_VARIANT");
      return e ? std::atoi(e) : 1;
    }();
    if (variant == 0) {
      if (op.ndim == 3)
        stencil_mc_kernel<T, 3, MODE, 4><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
      else
        stencil_mc_kernel<T, 2, MODE, 4><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
    } else if (variant == 2 || (sizeof(T) == 8 && variant != 3)) {
      if (op.ndim == 3)
        stencil_v4_kernel<T, 3, MODE, 3><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
      else
        stencil_v4_kernel<T, 2, MODE, 3><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
    } else {
      if (op.ndim == 3)
        stencil_v4_kernel<T, 3, MODE, 9><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
      else
        stencil_v4_kernel<T, 2, MODE, 9><<<g4, kBlock, 0, s>>>(op, x, b, out, wj);
    }
  } else {
    if (op.ndim == 3)
      level_kernel<T, 3, kStencil, MODE><<<grid, kBlock, 0, s>>>(op, x, b, out, wj);
    else
      level_kernel<T, 2, kStencil, MODE><<<grid, kBlock, 0, s>>>(op, x, b, out, wj);
  }
  HZ_LAUNCH_CHECK();
}

}  // namespace

template <class T>
void launch_apply(const LevelOp<T>& op, const cplx_t<T>* u, cplx_t<T>* out, cudaStream_t s) {
  dispatch_level<T, 0>(op, u, nullptr, out, T(0), s);
}
void launch_apply_lo(const LevelOp<double>& op, const float2* u, double2* out, cudaStream_t s) {
  const double n = double(op.g.owned_nodes()), k = op.g.k;
  ProfScope prof(op.kind == kFine27 ? "apply_fine27_c128" : "apply_fine_c128", n * (k * (8.0 + 16.0) + 16.0), s);
  if (launch_stream3d_lo(op, u, out, s)) return;
  if (op.kind != kFine) throw HzError(kState, "apply_lo: 5/7-point operator, or 8-column blocks of the 27-point one");
  static const bool two = [] {  // HZ_APPLY_LO2=0: one column per thread
    const char* e = std::getenv("HZ_APPLY_LO2");
    return !(e && e[0] == '0');
  }();
  if (two && op.g.k % 2 == 0) {
    const int grid2 = grid_for(op.g.owned_elems() / 2, kBlock);
    if (op.ndim == 3)
      apply_lo2_kernel<3><<<grid2, kBlock, 0, s>>>(op, u, out);
    else
      apply_lo2_kernel<2><<<grid2, kBlock, 0, s>>>(op, u, out);
    HZ_LAUNCH_CHECK();
    return;
  }
  const int grid = grid_for(op.g.owned_elems(), kBlock);
  if (op.ndim == 3)
    apply_lo_kernel<3><<<grid, kBlock, 0, s>>>(op, u, out);
  else
    apply_lo_kernel<2><<<grid, kBlock, 0, s>>>(op, u, out);
  HZ_LAUNCH_CHECK();
}

int launch_gram8_apply(const LevelOp<double>& op, int nb, const BlockTab<double>& X, const float2* Z, double2* W,
                       double2* partials, int max_slots, cudaStream_t s) {
  if (op.kind != kFine || op.g.k != 8 || nb < 1 || nb > 12 || op.g.z0 != 0 || op.g.z1 != (op.ndim == 3 ? op.g.n2 : op.g.n1))
    throw HzError(kState, "gram8_apply: 8-column whole-grid fine operator, nb in [1, 12]");
  const double n = double(op.g.nodes);
  ProfScope prof("apply_gram_c128", n * 8.0 * (8.0 + 16.0 + 16.0 * (nb - 1)) + n * 16.0, s, 8.0 * n * 64.0 * nb);
  const int64_t want = std::min<int64_t>(2 * kNumSMs, (int64_t(op.g.nodes) + 31) / 32);
  const int nslots = int(std::max<int64_t>(1, std::min<int64_t>(want, max_slots)));
  gram8_apply_dispatch<1>(nb, op, Z, W, X, partials, nslots, s);
  HZ_LAUNCH_CHECK();
  return nslots;
}

template <class T>
void launch_residual(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* r,
                     cudaStream_t s) {
  dispatch_level<T, 1>(op, x, b, r, T(0), s);
}
template <class T>
void launch_apply_residual(const LevelOp<T>& op, const cplx_t<T>* x, const cplx_t<T>* b, cplx_t<T>* r,
                           cudaStream_t s) {
  if (op.kind != kFine) {  // compact 27-point fine operator: the stencil residual
    dispatch_level<T, 1>(op, x, b, r, T(0), s);
    return;
  }
  const int64_t total = op.g.owned_elems();
  ProfScope prof(sizeof(T) == 8 ? "apply_residual_fine_c128" : "apply_residual_fine_c64", level_bytes(op, 1), s);
  if (launch_stream3d<T, cplx_t<T>>(op, 3, T(0), x, b, r, s)) return;
  if (sizeof(T) == 4 && op.g.k % 4 == 0) {
    const int g4 = grid_for(total / 4, kBlock);
    if (op.ndim == 3)
      fine_v4_kernel<T, 3, 3><<<g4, kBlock, 0, s>>>(op, x, b, r, T(0));
    else
      fine_v4_kernel<T, 2, 3><<<g4, kBlock, 0, s>>>(op, x, b, r, T(0));
  } else if (op.ndim == 3) {
    level_kernel<T, 3, kFine, 3><<<grid_for(total, kBlock), kBlock, 0, s>>>(op, x, b, r, T(0));
  } else {
    level_kernel<T, 2, kFine, 3><<<grid_for(total, kBlock), kBlock, 0, s>>>(op, x, b, r, T(0));
  }
  HZ_LAUNCH_CHECK();
}
template <class T>
void launch_jacobi(const LevelOp<T>& op, T wj, const cplx_t<T>* x, const cplx_t<T>* b,
                   cplx_t<T>* xout, cudaStream_t s) {
  dispatch_level<T, 2>(op, x, b, xout, wj, s);
}
template <class T, class In>
void launch_jacobi_zero(const LevelOp<T>& op, T wj, const In* b, cplx_t<T>* xout, cudaStream_t s) {
  const int64_t total = op.g.owned_elems();
  ProfScope prof(sizeof(T) == 8 ? "jacobi_zero_c128" : "jacobi_zero_c64",
                 double(op.g.owned_nodes()) * ((double(sizeof(In)) + sizeof(cplx_t<T>)) * op.g.k + sizeof(cplx_t<T>)), s);
  if constexpr (std::is_same<In, cplx_t<T>>::value && sizeof(T) == 4) {
    if (op.g.k % 4 == 0) {
      jacobi_zero_v4_kernel<T><<<grid_for(total / 4, kBlock), kBlock, 0, s>>>(op.g, op.inv_diag, wj, b, xout);
      HZ_LAUNCH_CHECK();
      return;
    }
  }
  jacobi_zero_kernel<T, In><<<grid_for(total, kBlock), kBlock, 0, s>>>(op.g, op.inv_diag, wj, b, xout);
  HZ_LAUNCH_CHECK();
}
template <class T>
void launch_restrict(const LevelGeom& gf, const LevelGeom& gc, int ndim, const cplx_t<T>* r,
                     cplx_t<T>* bc, cudaStream_t s) {
  const int grid = grid_for(gc.owned_elems(), kBlock);
  ProfScope prof(sizeof(T) == 8 ? "restrict_c128" : "restrict_c64",
                 (double(gf.nodes) * gc.owned_nodes() / gc.nodes + gc.owned_nodes()) * gf.k * sizeof(cplx_t<T>), s);
  if (sizeof(T) == 4 && gf.k % 4 == 0) {
    const int g4 = grid_for(gc.owned_elems() / 4, kBlock);
    if (ndim == 3)
      restrict_v4_kernel<T, 3><<<g4, kBlock, 0, s>>>(gf, gc, r, bc);
    else
      restrict_v4_kernel<T, 2><<<g4, kBlock, 0, s>>>(gf, gc, r, bc);
  } else if (ndim == 3) {
    restrict_kernel<T, 3><<<grid, kBlock, 0, s>>>(gf, gc, r, bc);
  } else {
    restrict_kernel<T, 2><<<grid, kBlock, 0, s>>>(gf, gc, r, bc);
  }
  HZ_LAUNCH_CHECK();
}
template <class T>
void launch_prolong_correct(const LevelGeom& gf, const LevelGeom& gc, int ndim,
                            const cplx_t<T>* ec, cplx_t<T>* x, cudaStream_t s) {
  const int grid = grid_for(gf.owned_elems(), kBlock);
  ProfScope prof(sizeof(T) == 8 ? "prolong_correct_c128" : "prolong_correct_c64",
                 (2.0 * gf.owned_nodes() + gc.nodes * double(gf.owned_nodes()) / gf.nodes) * gf.k * sizeof(cplx_t<T>), s);
  if (sizeof(T) == 4 && gf.k % 4 == 0) {
    const int g4 = grid_for(gf.owned_elems() / 4, kBlock);
    if (ndim == 3)
      prolong_v4_kernel<T, 3><<<g4, kBlock, 0, s>>>(gf, gc, ec, x);
    else
      prolong_v4_kernel<T, 2><<<g4, kBlock, 0, s>>>(gf, gc, ec, x);
  } else if (ndim == 3) {
    prolong_correct_kernel<T, 3><<<grid, kBlock, 0, s>>>(gf, gc, ec, x);
  } else {
    prolong_correct_kernel<T, 2><<<grid, kBlock, 0, s>>>(gf, gc, ec, x);
  }
  HZ_LAUNCH_CHECK();
}

bool fused_fine_ok(const LevelOp<float>& op) {
  return (op.kind == kFine && op.g.k % 4 == 0) || (op.kind == kFine27 && stream3d_ok(op));
}
bool cast_zero_ok(const LevelOp<float>& op) { return op.g.k % 4 == 0; }

void launch_jacobi_zero_cast(const LevelOp<float>& op, float wj, const double2* b64, float2* b32, float2* x1,
                             cudaStream_t s) {
  const int64_t total = op.g.owned_elems();
  const double n = double(op.g.owned_nodes()), k = op.g.k;
  ProfScope prof("jacobi_zero_cast_c64", n * (k * (16.0 + 8.0 + 8.0) + 8.0), s);
  jacobi_zero_cast_kernel<<<grid_for(total / 4, kBlock), kBlock, 0, s>>>(op.g, op.inv_diag, wj, b64, b32, x1);
  HZ_LAUNCH_CHECK();
}

void launch_jacobi_out64(const LevelOp<float>& op, float wj, const float2* x, const float2* b, double2* out,
                         cudaStream_t s) {
  const int64_t total = op.g.owned_elems();
  const double n = double(op.g.owned_nodes()), k = op.g.k;
  ProfScope prof("jacobi_out64_fine_c64", n * (k * (8.0 + 8.0 + 16.0) + 8.0 + 8.0), s);
  if (launch_stream3d<float, double2>(op, 2, wj, x, b, out, s)) return;
  if (op.kind != kFine) throw HzError(kState, "jacobi_out64: 5/7-point operator, or 8-column blocks of the 27-point one");
  if (op.ndim == 3)
    fine_v4_kernel<float, 3, 2, double2><<<grid_for(total / 4, kBlock), kBlock, 0, s>>>(op, x, b, out, wj);
  else
    fine_v4_kernel<float, 2, 2, double2><<<grid_for(total / 4, kBlock), kBlock, 0, s>>>(op, x, b, out, wj);
  HZ_LAUNCH_CHECK();
}

void launch_galerkin(const LevelOp<double>& fine, const LevelGeom& gc, double2* coef_c,
                     cudaStream_t s) {
  const int grid = grid_for(gc.nodes, 128);
  if (fine.kind == kFine) {
    if (fine.ndim == 3)
      galerkin_kernel<3, kFine><<<grid, 128, 0, s>>>(fine, gc, coef_c);
    else
      galerkin_kernel<2, kFine><<<grid, 128, 0, s>>>(fine, gc, coef_c);
  } else {
    if (fine.ndim == 3)
      galerkin_kernel<3, kStencil><<<grid, 128, 0, s>>>(fine, gc, coef_c);
    else
      galerkin_kernel<2, kStencil><<<grid, 128, 0, s>>>(fine, gc, coef_c);
  }
  HZ_LAUNCH_CHECK();
}

template <class Dst, class Src>
void launch_cast(int64_t count, const Src* in, Dst* out, cudaStream_t s) {
  ProfScope prof("cast", double(count) * (sizeof(Src) + sizeof(Dst)), s);
  cast_kernel<Dst, Src><<<grid_for(count, kBlock), kBlock, 0, s>>>(count, in, out);
  HZ_LAUNCH_CHECK();
}

#define HZ_INST(T)                                                                                 \
  template void launch_apply<T>(const LevelOp<T>&, const cplx_t<T>*, cplx_t<T>*, cudaStream_t);   \
  template void launch_residual<T>(const LevelOp<T>&, const cplx_t<T>*, const cplx_t<T>*,         \
                                   cplx_t<T>*, cudaStream_t);                                     \
  template void launch_apply_residual<T>(const LevelOp<T>&, const cplx_t<T>*, const cplx_t<T>*,   \
                                         cplx_t<T>*, cudaStream_t);                               \
  template void launch_jacobi<T>(const LevelOp<T>&, T, const cplx_t<T>*, const cplx_t<T>*,        \
                                 cplx_t<T>*, cudaStream_t);                                       \
  template void launch_restrict<T>(const LevelGeom&, const LevelGeom&, int, const cplx_t<T>*,     \
                                   cplx_t<T>*, cudaStream_t);                                     \
  template void launch_prolong_correct<T>(const LevelGeom&, const LevelGeom&, int,                \
                                          const cplx_t<T>*, cplx_t<T>*, cudaStream_t);
HZ_INST(double)
HZ_INST(float)
#undef HZ_INST
template void launch_jacobi_zero<double, double2>(const LevelOp<double>&, double, const double2*,
                                                  double2*, cudaStream_t);
template void launch_jacobi_zero<float, float2>(const LevelOp<float>&, float, const float2*,
                                                float2*, cudaStream_t);
template void launch_jacobi_zero<float, double2>(const LevelOp<float>&, float, const double2*,
                                                 float2*, cudaStream_t);
template void launch_cast<float2, double2>(int64_t, const double2*, float2*, cudaStream_t);
template void launch_cast<double2, float2>(int64_t, const float2*, double2*, cudaStream_t);
template void launch_cast<double2, double2>(int64_t, const double2*, double2*, cudaStream_t);

namespace {
struct W27 {
  double lap[4], mu[4];
};
__global__ void __launch_bounds__(128)
build27_kernel(LevelGeom g, W27 w, const double2* __restrict__ mass, const double* __restrict__ m, double shift_w2,
               double2* __restrict__ planes) {
  const int64_t i = int64_t(blockIdx.x) * 128 + threadIdx.x;
  if (i >= g.nodes) return;
  uint32_t x, y, z;
  g.unpack(uint32_t(i), x, y, z);
  const double2 Mi = make_double2(mass[i].x, mass[i].y - shift_w2 * m[i]);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int sidx = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
        const int q = abs(dx) + abs(dy) + abs(dz);
        const int64_t xx = int64_t(x) + dx, yy = int64_t(y) + dy, zz = int64_t(z) + dz;
        double2 c = make_double2(0.0, 0.0);
        if (q == 0) {
          c = make_double2(w.lap[0] + w.mu[0] * Mi.x, w.mu[0] * Mi.y);
        } else if (xx >= 0 && xx < g.n0 && yy >= 0 && yy < g.n1 && zz >= 0 && zz < g.n2) {
          const int64_t j = xx + int64_t(g.n0) * (yy + int64_t(g.n1) * zz);
          const double2 Mj = make_double2(mass[j].x, mass[j].y - shift_w2 * m[j]);
          const double avr = 0.5 * (Mi.x + Mj.x), avi = 0.5 * (Mi.y + Mj.y);
          c = make_double2(w.lap[q] + w.mu[q] * avr, w.mu[q] * avi);
        }
        planes[int64_t(sidx) * g.nodes + i] = c;
      }
}
__global__ void inv_plane_kernel(int64_t n, const double2* __restrict__ c, double2* __restrict__ inv) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (i >= n) return;
  // 1 / (a + ib) = (a - ib) / (a^2 + b^2)
  const double2 a = c[i];
  const double d = a.x * a.x + a.y * a.y;
  inv[i] = make_double2(a.x / d, -a.y / d);
}
}  // namespace

void launch_build27(const LevelGeom& g, const double* lap, const double* mu, const double2* mass, const double* m,
                    double shift_w2, double2* planes, cudaStream_t s) {
  W27 w;
  for (int q = 0; q < 4; ++q) {
    w.lap[q] = lap[q];
    w.mu[q] = mu[q];
  }
  build27_kernel<<<grid_for(g.nodes, 128), 128, 0, s>>>(g, w, mass, m, shift_w2, planes);
  HZ_LAUNCH_CHECK();
}

void launch_inv_plane(int64_t n, const double2* centre, double2* inv, cudaStream_t s) {
  inv_plane_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, centre, inv);
  HZ_LAUNCH_CHECK();
}

namespace {
__global__ void shift_mass_kernel(int64_t n, const double2* __restrict__ mass, const double* __restrict__ m,
                                  double shift_w2, double2* __restrict__ ms) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (i < n) ms[i] = make_double2(mass[i].x, mass[i].y - shift_w2 * m[i]);  // as build27_kernel's M_i
}
__global__ void inv_centre27_kernel(int64_t n, double lap0, double mu0, const double2* __restrict__ ms,
                                    double2* __restrict__ inv) {
  const int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (i >= n) return;
  const double2 a = make_double2(lap0 + mu0 * ms[i].x, mu0 * ms[i].y);
  const double d = a.x * a.x + a.y * a.y;
  inv[i] = make_double2(a.x / d, -a.y / d);
}
}  // namespace

void launch_shift_mass(int64_t n, const double2* mass, const double* m, double shift_w2, double2* ms, cudaStream_t s) {
  shift_mass_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, mass, m, shift_w2, ms);
  HZ_LAUNCH_CHECK();
}

void launch_inv_centre27(int64_t n, double lap0, double mu0, const double2* ms, double2* inv, cudaStream_t s) {
  inv_centre27_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, lap0, mu0, ms, inv);
  HZ_LAUNCH_CHECK();
}

}  // namespace hz
