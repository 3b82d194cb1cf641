// Block-tridiagonal (plane) direct solver for large 3D coarsest levels.
//
// The reference factors the coarsest Galerkin operator with a banded LU
// whose band is one full plane (src/dense.cpp:9-61). For the 3-level
// hierarchies that converge in 3D (coarsest 33x33x17 = 18,513 nodes, band
// 1,123) that factor costs minutes on the host, and its substitution is a
// chain of 2 n_c dependent steps. Ordered plane by plane the same operator
// is block tridiagonal, A = tridiag(L_j, D_j, U_j) with m = n0*n1 unknowns
// per plane, so the solve becomes 2 (n2 - 1) + 1 dense m x m block products:
//   setup:   S_0 = D_0;  E_j = S_j^{-1};  F_j = E_j U_j;
//            S_{j+1} = D_{j+1} - L_{j+1} F_j
//   forward: y_0 = E_0 b_0;  y_j = E_j (b_j - L_j y_{j-1})
//   back:    x_{last} = y_{last};  x_j = y_j - F_j x_{j+1}
// E_j and F_j are dense, stored row-major (row = output node of the plane) for
// planes up to 2 x 148 x 8 nodes and transposed for the coarse GEMM above;
// L_j, U_j are read straight from the Galerkin stencil planes. Block LU
// without inter-plane pivoting on the shifted (complex, absorbing) operator;
// each S_j is inverted by Gauss-Jordan with partial pivoting. Agreement with
// the reference's banded LU is to cond(A_c) * eps (tested).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "block_tiled.cuh"
#include "devbuf.hpp"
#include "kernels.hpp"
#include "profile.hpp"
#include "tma.cuh"

namespace hz {

namespace {

__device__ __forceinline__ double2 cdivd(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

__device__ __forceinline__ int plane_s(int dx, int dy, int dz) { return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1); }

// S[r][c] = coupling of plane j row r to plane j+dz column c (dense m x m,
// row-major), from the 27 Galerkin planes.
__global__ void build_block_kernel(LevelGeom g, const double2* __restrict__ coef, int j, int dz,
                                   double2* __restrict__ S) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  const int ri = int(r % g.n0), rj = int(r / g.n0), ci = int(c % g.n0), cj = int(c / g.n0);
  const int dx = ci - ri, dy = cj - rj;
  double2 v = make_double2(0.0, 0.0);
  if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && j + dz >= 0 && j + dz < int(g.n2))
    v = coef[int64_t(plane_s(dx, dy, dz)) * g.nodes + int64_t(j) * m + r];
  S[e] = v;
}

// Gauss-Jordan, step p: pivot search over rows p..m-1 of column p (1 CTA)
__global__ void gj_pivot_kernel(int64_t m, const double2* __restrict__ S, int p, int* piv) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int arg = p;
  for (int64_t r = p + threadIdx.x; r < m; r += blockDim.x) {
    const double2 a = S[r * m + p];
    const double v = a.x * a.x + a.y * a.y;
    if (v > best) {
      best = v;
      arg = int(r);
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = bv[threadIdx.x + o];
      const int i2 = bi[threadIdx.x + o];
      if (v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < bi[threadIdx.x])) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) piv[p] = bv[0] > 0.0 ? bi[0] : -1;
}

// swap rows p <-> piv[p]; save column p (tmp) and the scaled pivot row (row)
__global__ void gj_prepare_kernel(int64_t m, double2* __restrict__ S, int p, const int* __restrict__ piv,
                                  double2* __restrict__ col, double2* __restrict__ row) {
  const int q = piv[p];
  if (q < 0) return;
  const int64_t c = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (c >= m) return;
  if (q != p) {
    const double2 a = S[int64_t(p) * m + c], b = S[int64_t(q) * m + c];
    S[int64_t(p) * m + c] = b;
    S[int64_t(q) * m + c] = a;
  }
  __threadfence();
}

__global__ void gj_scale_kernel(int64_t m, double2* __restrict__ S, int p, const int* __restrict__ piv,
                                double2* __restrict__ col, double2* __restrict__ row) {
  if (piv[p] < 0) return;
  const int64_t c = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (c >= m) return;
  const double2 pv = S[int64_t(p) * m + p];
  // in-place inversion: the pivot entry becomes 1 before scaling
  const double2 a = c == p ? make_double2(1.0, 0.0) : S[int64_t(p) * m + c];
  row[c] = cdivd(a, pv);
  col[c] = S[c * m + p];  // column p of every row (pivot row's value unused)
}

// rank-1 elimination of column p from every other row (in-place inverse)
__global__ void gj_eliminate_kernel(int64_t m, double2* __restrict__ S, int p, const int* __restrict__ piv,
                                    const double2* __restrict__ col, const double2* __restrict__ row) {
  if (piv[p] < 0) return;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  if (r == p) {
    S[e] = row[c];
    return;
  }
  const double2 f = col[r];
  const double2 base = c == p ? make_double2(0.0, 0.0) : S[e];
  const double2 rc = row[c];
  S[e] = make_double2(base.x - (f.x * rc.x - f.y * rc.y), base.y - (f.x * rc.y + f.y * rc.x));
}

// undo the row interchanges as column interchanges (reverse order)
__global__ void gj_unswap_kernel(int64_t m, double2* __restrict__ S, int p, const int* __restrict__ piv) {
  const int q = piv[p];
  if (q < 0 || q == p) return;
  const int64_t r = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (r >= m) return;
  const double2 a = S[r * m + p], b = S[r * m + q];
  S[r * m + p] = b;
  S[r * m + q] = a;
}

// F[r][c] = sum_l E[r][l] U[l][c], U = plane j -> j+dir coupling (9 per column)
__global__ void mul_eu_kernel(LevelGeom g, const double2* __restrict__ coef, int j, int dir,
                              const double2* __restrict__ E, double2* __restrict__ F) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  const int ci = int(c % g.n0), cj = int(c / g.n0);
  double2 s = make_double2(0.0, 0.0);
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int li = ci - dx, lj = cj - dy;  // l + (dx, dy, dir) = c
      if (li < 0 || li >= int(g.n0) || lj < 0 || lj >= int(g.n1)) continue;
      const int64_t l = li + int64_t(g.n0) * lj;
      const double2 u = coef[int64_t(plane_s(dx, dy, dir)) * g.nodes + int64_t(j) * m + l];
      s = cfma(E[r * m + l], u, s);
    }
  F[e] = s;
}

// S[r][c] -= sum_l L[r][l] F[l][c], L = plane j1 -> j1-dir coupling (F of plane j1-dir)
__global__ void schur_kernel(LevelGeom g, const double2* __restrict__ coef, int j1, int dir,
                             const double2* __restrict__ F, double2* __restrict__ S) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  const int ri = int(r % g.n0), rj = int(r / g.n0);
  double2 s = S[e];
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int li = ri + dx, lj = rj + dy;
      if (li < 0 || li >= int(g.n0) || lj < 0 || lj >= int(g.n1)) continue;
      const int64_t l = li + int64_t(g.n0) * lj;
      const double2 a = coef[int64_t(plane_s(dx, dy, -dir)) * g.nodes + int64_t(j1) * m + r];
      s = csub(s, cmul(a, F[l * m + c]));
    }
  S[e] = s;
}

// Programmatic dependent launch for the plane-step chain (HZ_BT_PDL=1, default off:
// measured 6 % slower per cycle on config 3, neutral on config 4): a step's
// kernel is launched while its predecessor still runs, does everything that
// does not depend on the data (operator loads, the next block's L2 prefetch)
// and only then waits for the predecessor's results (griddepcontrol.wait: the
// whole prerequisite grid complete and visible). Every global write comes after
// the wait, so the scratch blocks are never overwritten under a running reader.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

bool bt_pdl() {  // read per launch: the tests switch it within one process
  const char* e = std::getenv("HZ_BT_PDL");
  return e && e[0] == '1';
}

template <class... KA, class... A>
void launch_chain_smem(void (*kern)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = bt_pdl() ? 1 : 0;
  HZ_CUDA(cudaLaunchKernelEx(&cfg, kern, KA(args)...));
}
template <class... KA, class... A>
void launch_chain(void (*kern)(KA...), dim3 grid, dim3 block, cudaStream_t s, A... args) {
  launch_chain_smem(kern, grid, block, 0, s, args...);
}

// r = b_j - L_j y_{j-dir} for one plane, all k columns (L = plane j -> j-dir
// coupling; b may be r itself: the middle plane of the twisted sweep
// subtracts both neighbours in two passes)
template <class T>
__global__ void couple_kernel(LevelGeom g, const cplx_t<T>* __restrict__ coef, int j, int dir, const cplx_t<T>* b,
                              const cplx_t<T>* yprev, cplx_t<T>* r, int k) {
  using V = cplx_t<T>;
  const int n0 = int(g.n0), n1 = int(g.n1);
  const int m = n0 * n1;
  const int e = int(blockIdx.x) * 256 + threadIdx.x;
  pdl_launch_dependents();
  if (e >= m * k) return;
  const int row = e / k;
  const int q = e - row * k;
  const int rj = row / n0, ri = row - rj * n0;
  // the 9 couplings and neighbours are loaded first (masked), then summed in
  // the fixed (dy, dx) order
  V av[9], yv[9];
  bool ok[9];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const int s9 = (dy + 1) * 3 + dx + 1;
      av[s9] = __ldg(&coef[int64_t(plane_s(dx, dy, -dir)) * g.nodes + int64_t(j) * m + row]);
    }
  pdl_wait();  // yprev (and b, when it is r itself) come from the preceding step
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const int s9 = (dy + 1) * 3 + dx + 1;
      const int li = ri + dx, lj = rj + dy;
      ok[s9] = li >= 0 && li < n0 && lj >= 0 && lj < n1;
      yv[s9] = yprev[ok[s9] ? (li + n0 * lj) * k + q : e];
    }
  V s = b[e];
#pragma unroll
  for (int s9 = 0; s9 < 9; ++s9)
    if (ok[s9]) s = csub(s, cmul(av[s9], yv[s9]));
  r[e] = s;
}

// dst[c][r] = src[r][c] with row stride ld (transposed copy for the GEMM)
__global__ void transpose_kernel(int64_t m, const double2* __restrict__ src, double2* __restrict__ dst, int64_t ld) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  dst[c * ld + r] = src[e];
}

// dst[r][c] = src[r][c] with row stride ld
__global__ void strided_copy_kernel(int64_t m, const double2* __restrict__ src, double2* __restrict__ dst,
                                    int64_t ld) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  dst[r * ld + c] = src[e];
}

template <class V>
__device__ __forceinline__ void cp_async_elem(V* smem, const V* gmem) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (sizeof(V) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem));
}

// One plane step out = c_in + sign * (P r) with P = E_j or F_j (m x m,
// row-major, row stride ld) and r an m x k block, for KG of its columns
// (blockIdx.y = column group); used for small planes (bt_rowmajor), where
// the split-K GEMM + reduce pair is launch/latency bound. Each warp owns one
// plane row (two above 2 x 148 x 8 rows) and the whole reduction over l:
// lanes stride l, the row of P streams from HBM coalesced (next chunk's loads
// issued before the current chunk's math), the chunk of r (LC nodes x KG
// columns, column-major in shared memory) is staged once per CTA by cp.async
// (double-buffered) and read conflict-free by all 8 warps; lane partial sums
// meet in an xor butterfly, so no split-K partials and no second launch.
// Deterministic: fixed per-lane order, fixed butterfly.
template <class T, int RW, int KG, int LC, int PF, int NW>
__global__ void __launch_bounds__(32 * NW)
bt_rows_kernel(int m, int k, const cplx_t<T>* __restrict__ P, int ld, const cplx_t<T>* __restrict__ r,
               cplx_t<T>* out, const cplx_t<T>* c_in, T sign, const cplx_t<T>* __restrict__ Pnext) {
  using V = cplx_t<T>;
  constexpr int U = LC / 32;
  // The factor blocks do not depend on the data: the rows this CTA will own
  // in the chain's next plane step are brought into L2 now (one bulk prefetch
  // per row), while this latency-bound step leaves the HBM mostly idle.
  if (Pnext != nullptr && blockIdx.y == 0 && threadIdx.x < NW * RW) {
    const int row = int(blockIdx.x) * (NW * RW) + int(threadIdx.x);
    if (row < m)
      tma::prefetch_l2(Pnext + int64_t(row) * ld, uint32_t((size_t(m) * sizeof(V) + 15) / 16 * 16));
  }
  pdl_launch_dependents();
  // chunk of r in its natural [l][q] order, rows padded to KG + 1 values: the
  // staging writes and the per-lane reads (lane = l) are both conflict free
  constexpr int RS = KG + 1;
  __shared__ __align__(16) V rs[2][LC * RS];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int i0 = int(blockIdx.x) * (NW * RW);
  const int q0 = blockIdx.y * KG;
  const int nch = (m + LC - 1) / LC;
  // rows past the end are clamped (computed, not stored): no predicates in the loop
  const V* prow[RW];
  bool live[RW];
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int row = i0 + w + NW * t;
    live[t] = row < m;
    prow[t] = P + int64_t(min(row, m - 1)) * ld + lane;
  }
  const V* rq = r + q0;
  auto stage = [&](int c, V* dst) {
    const int l0 = c * LC;
#pragma unroll
    for (int e = tid; e < LC * KG; e += 32 * NW) {
      const int l = e / KG, q = e % KG;
      if (l0 + l < m)
        cp_async_elem(dst + l * RS + q, rq + (l0 + l) * k + q);
      else
        dst[l * RS + q] = czero<V>();
    }
  };
  auto load_p = [&](int c, V (&pv)[RW][U]) {
    const int l0 = c * LC;
    if (l0 + LC <= m) {
#pragma unroll
      for (int t = 0; t < RW; ++t)
#pragma unroll
        for (int u = 0; u < U; ++u) pv[t][u] = __ldg(prow[t] + l0 + 32 * u);
    } else {
#pragma unroll
      for (int t = 0; t < RW; ++t)
#pragma unroll
        for (int u = 0; u < U; ++u) pv[t][u] = l0 + lane + 32 * u < m ? __ldg(prow[t] + l0 + 32 * u) : czero<V>();
    }
  };
  // Two real-scaled accumulators per output, sum Re(P) r and sum Im(P) r, combined as A + i B after the loop:
  // both updates are scalar x pair FMAs (FFMA2 with a broadcast operand), independent of each other. The
  // complex-FMA form needed an (Im P, Im P) register pair per product, which the compiler rebuilt with two
  // MOVs for every four FFMA2 (ncu: 21 % of the kernel's instructions), and chained its two FMAs.
  V accA[RW][KG], accB[RW][KG];
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q) accA[t][q] = accB[t][q] = czero<V>();
  // the row's chunks of P are loaded PF - 1 chunks ahead of the one being
  // multiplied (registers, rotated by unrolling)
  V pq[PF][RW][U];
#pragma unroll
  for (int f = 0; f < PF - 1; ++f)
    if (f < nch) load_p(f, pq[f]);
  pdl_wait();  // r and c_in come from the preceding step; P does not
  stage(0, rs[0]);
  tiled::cp_async_commit();
  for (int c0 = 0; c0 < nch; c0 += PF) {
#pragma unroll
    for (int f = 0; f < PF; ++f) {
      const int c = c0 + f;
      if (c < nch) {
        if (c + 1 < nch) stage(c + 1, rs[(c + 1) & 1]);
        if (c + PF - 1 < nch) load_p(c + PF - 1, pq[(f + PF - 1) % PF]);
        tiled::cp_async_commit();
        tiled::cp_async_wait<1>();
        __syncthreads();
        const V* b = rs[c & 1] + lane * RS;
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < KG; ++q) {
            const V rv = b[32 * u * RS + q];
#pragma unroll
            for (int t = 0; t < RW; ++t) {
              accA[t][q] = crfma(pq[f][t][u].x, rv, accA[t][q]);
              accB[t][q] = crfma(pq[f][t][u].y, rv, accB[t][q]);
            }
          }
        }
        __syncthreads();
      }
    }
  }
  tiled::cp_async_wait<0>();
  V acc[RW][KG];
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q) acc[t][q] = mk(accA[t][q].x - accB[t][q].y, accA[t][q].y + accB[t][q].x);
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[t][q].x += __shfl_xor_sync(0xffffffffu, acc[t][q].x, o);
        acc[t][q].y += __shfl_xor_sync(0xffffffffu, acc[t][q].y, o);
      }
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    if (!live[t]) continue;
#pragma unroll
    for (int q = 0; q < KG; ++q) {
      if (lane != q) continue;
      V v = acc[t][q];
      const int o = (i0 + w + NW * t) * k + q0 + q;
      if (c_in) {
        const V cv = c_in[o];
        v = mk(cv.x + sign * v.x, cv.y + sign * v.y);
      }
      out[o] = v;
    }
  }
}

// The plane step with all of r resident in shared memory (HZ_BT_RES): the
// row-owner kernel re-stages r chunk by chunk with two CTA barriers per
// chunk, and its warps spend most of their time between those barriers and
// the staging latency (ncu: issue 34 %, no dominant stall). Here a CTA of NW
// warps owns NW * RW rows, copies r once ([l][KG + 1] padded rows, conflict
// free for lane = l reads), and its warps then stream their rows of P with
// no barrier at all, the next chunk's loads always in flight. 16 warps x 2
// rows make 68 CTAs of 154 KB for a 2,145-node plane: one CTA per SM, the
// two chains of the two-sided sweep side by side on 136 SMs. Same per-lane
// and butterfly order as the row-owner kernel: bitwise the same results.
template <class T, int RW, int KG, int LC, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
bt_rows_res_kernel(int m, int k, const cplx_t<T>* __restrict__ P, int ld, const cplx_t<T>* __restrict__ r,
                   cplx_t<T>* out, const cplx_t<T>* c_in, T sign) {
  using V = cplx_t<T>;
  constexpr int U = LC / 32, RS = KG + 1;
  extern __shared__ __align__(16) unsigned char bt_smem[];
  V* rs = reinterpret_cast<V*>(bt_smem);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int i0 = int(blockIdx.x) * (NW * RW);
  const int q0 = blockIdx.y * KG;
  const int nch = (m + LC - 1) / LC;
  const V* prow[RW];
  bool live[RW];
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    const int row = i0 + w + NW * t;
    live[t] = row < m;
    prow[t] = P + int64_t(min(row, m - 1)) * ld + lane;
  }
  auto load_p = [&](int c, V (&pv)[RW][U]) {
    const int l0 = c * LC;
    if (l0 + LC <= m) {
#pragma unroll
      for (int t = 0; t < RW; ++t)
#pragma unroll
        for (int u = 0; u < U; ++u) pv[t][u] = __ldg(prow[t] + l0 + 32 * u);
    } else {
#pragma unroll
      for (int t = 0; t < RW; ++t)
#pragma unroll
        for (int u = 0; u < U; ++u) pv[t][u] = l0 + lane + 32 * u < m ? __ldg(prow[t] + l0 + 32 * u) : czero<V>();
    }
  };
  V pq[2][RW][U];
  load_p(0, pq[0]);  // P does not depend on the preceding step
  pdl_launch_dependents();
  pdl_wait();
  {  // r -> shared memory, rows past m zero
    const V* rq = r + q0;
    const int tot = nch * LC * KG;
    for (int e = tid; e < tot; e += 32 * NW) {
      const int l = e / KG, q = e % KG;
      if (l < m)
        cp_async_elem(rs + l * RS + q, rq + l * k + q);
      else
        rs[l * RS + q] = czero<V>();
    }
    tiled::cp_async_commit();
    tiled::cp_async_wait<0>();
  }
  __syncthreads();
  V accA[RW][KG], accB[RW][KG];
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q) accA[t][q] = accB[t][q] = czero<V>();
  for (int c0 = 0; c0 < nch; c0 += 2) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int c = c0 + f;
      if (c < nch) {
        if (c + 1 < nch) load_p(c + 1, pq[f ^ 1]);
        const V* b = rs + (c * LC + lane) * RS;
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < KG; ++q) {
            const V rv = b[32 * u * RS + q];
#pragma unroll
            for (int t = 0; t < RW; ++t) {
              accA[t][q] = crfma(pq[f][t][u].x, rv, accA[t][q]);
              accB[t][q] = crfma(pq[f][t][u].y, rv, accB[t][q]);
            }
          }
        }
      }
    }
  }
  V acc[RW][KG];
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q) acc[t][q] = mk(accA[t][q].x - accB[t][q].y, accA[t][q].y + accB[t][q].x);
#pragma unroll
  for (int t = 0; t < RW; ++t)
#pragma unroll
    for (int q = 0; q < KG; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[t][q].x += __shfl_xor_sync(0xffffffffu, acc[t][q].x, o);
        acc[t][q].y += __shfl_xor_sync(0xffffffffu, acc[t][q].y, o);
      }
#pragma unroll
  for (int t = 0; t < RW; ++t) {
    if (!live[t]) continue;
#pragma unroll
    for (int q = 0; q < KG; ++q) {
      if (lane != q) continue;
      V v = acc[t][q];
      const int o = (i0 + w + NW * t) * k + q0 + q;
      if (c_in) {
        const V cv = c_in[o];
        v = mk(cv.x + sign * v.x, cv.y + sign * v.y);
      }
      out[o] = v;
    }
  }
}

// HZ_BT_RES = "NW[:RW[:LC]]" (warps per CTA, rows per warp, columns per chunk) selects the resident-r kernel
// where r fits in shared memory; 0: off
template <class T>
bool bt_rows_res_go(int64_t m, int k, const cplx_t<T>* P, int64_t ld, const cplx_t<T>* r, cplx_t<T>* out,
                    const cplx_t<T>* c_in, T sign, cudaStream_t s) {
  using V = cplx_t<T>;
  int nw = sizeof(T) == 8 ? 8 : 16, rw = 2, lc = 128;  // c128: 8 warps (config 3, c128 W-cycle: 3.95 vs 4.06 ms with 16 x 1, 4.42 row-owner)
  const char* e = std::getenv("HZ_BT_RES");
  if (e) std::sscanf(e, "%d:%d:%d", &nw, &rw, &lc);
  if (nw <= 0 || k % 8 != 0) return false;
  const int64_t nch = (m + lc - 1) / lc;
  const size_t smem = size_t(nch) * lc * 9 * sizeof(V);
  if (smem > 200 * 1024) return false;
  auto launch = [&](auto kern, int nw_, int rw_) {
    allow_dyn_smem(reinterpret_cast<const void*>(kern), int(smem));
    const dim3 grid(unsigned((m + nw_ * rw_ - 1) / (nw_ * rw_)), unsigned(k / 8));
    launch_chain_smem(kern, grid, dim3(32 * nw_), smem, s, int(m), k, P, int(ld), r, out, c_in, sign);
  };
#define HZ_BT_RES_CASE(NW_, RW_, LC_)                          \
  if (nw == NW_ && rw == RW_ && lc == LC_) {                   \
    launch(bt_rows_res_kernel<T, RW_, 8, LC_, NW_>, NW_, RW_); \
    return true;                                               \
  }
  HZ_BT_RES_CASE(16, 2, 128)
  HZ_BT_RES_CASE(16, 1, 128)
  HZ_BT_RES_CASE(8, 2, 128)
  if constexpr (sizeof(T) == 4) {
    HZ_BT_RES_CASE(16, 2, 256)
    HZ_BT_RES_CASE(16, 1, 256)
    HZ_BT_RES_CASE(8, 2, 256)
    HZ_BT_RES_CASE(8, 4, 128)
    HZ_BT_RES_CASE(24, 1, 256)
    HZ_BT_RES_CASE(32, 1, 128)
  }
#undef HZ_BT_RES_CASE
  return false;
}

template <class T, int RW, int KG>
void bt_rows_go(int64_t m, int k, const cplx_t<T>* P, int64_t ld, const cplx_t<T>* r, cplx_t<T>* out,
                const cplx_t<T>* c_in, T sign, const cplx_t<T>* Pnext, cudaStream_t s) {
  constexpr int LC = sizeof(T) == 8 ? 128 : 256;  // r chunk: 32 KB of static shared memory, double-buffered
  // chunks of P in registers (PF - 1 in flight). One chunk ahead is the default: two or three ahead
  // (HZ_BT_PF=1) measured within noise on configs 3 and 4 in interleaved repetitions (8.90 vs 8.98 ms per
  // cycle on config 4, profiles/r02_bt_cycle_ab.txt) and its 165 registers keep the two chains of the
  // two-sided sweep from sharing the SMs
  static const int pf_env = [] {
    const char* e = std::getenv("HZ_BT_PF");
    return e ? std::atoi(e) : 0;
  }();
  const bool deep = pf_env == 1;
  // warps per CTA: 8; 4-warp CTAs (HZ_BT_NW=4: three per SM even with the deep prefetch, but each CTA stages
  // the whole chunk of r) measured equal or slower (8.98 vs 8.96, 1.92 vs 1.86 ms per cycle)
  static const int nw_env = [] {
    const char* e = std::getenv("HZ_BT_NW");
    return e ? std::atoi(e) : 0;
  }();
  const bool four = nw_env == 4;
  if (four) {
    const dim3 grid(unsigned((m + 4 * RW - 1) / (4 * RW)), unsigned(k / KG));
    if (deep)
      launch_chain(bt_rows_kernel<T, RW, KG, LC, (RW == 1 ? 4 : 3), 4>, grid, dim3(128), s, int(m), k, P, int(ld), r, out, c_in, sign, Pnext);
    else
      launch_chain(bt_rows_kernel<T, RW, KG, LC, 2, 4>, grid, dim3(128), s, int(m), k, P, int(ld), r, out, c_in, sign, Pnext);
    return;
  }
  const dim3 grid(unsigned((m + 8 * RW - 1) / (8 * RW)), unsigned(k / KG));
  if (deep)
    launch_chain(bt_rows_kernel<T, RW, KG, LC, (RW == 1 ? 4 : 3), 8>, grid, dim3(256), s, int(m), k, P, int(ld), r, out, c_in, sign, Pnext);
  else
    launch_chain(bt_rows_kernel<T, RW, KG, LC, 2, 8>, grid, dim3(256), s, int(m), k, P, int(ld), r, out, c_in, sign, Pnext);
}

template <class T>
void bt_rows(int64_t m, int k, const cplx_t<T>* P, int64_t ld, const cplx_t<T>* r, cplx_t<T>* out,
             const cplx_t<T>* c_in, T sign, const cplx_t<T>* Pnext, cudaStream_t s) {
  // two rows per warp above one CTA per SM (HZ_BT_RW=1 / 2 forces)
  static const int rw_env = [] {
    const char* e = std::getenv("HZ_BT_RW");
    return e ? std::atoi(e) : 0;
  }();
  const bool two = rw_env ? rw_env == 2 : m > int64_t(kNumSMs) * 8;
  if (bt_rows_res_go<T>(m, k, P, ld, r, out, c_in, sign, s)) return;
  auto go = [&](auto kg) {
    constexpr int KG = decltype(kg)::value;
    if (two)
      bt_rows_go<T, 2, KG>(m, k, P, ld, r, out, c_in, sign, Pnext, s);
    else
      bt_rows_go<T, 1, KG>(m, k, P, ld, r, out, c_in, sign, Pnext, s);
  };
  if (k % 8 == 0)
    go(std::integral_constant<int, 8>());
  else if (k % 4 == 0)
    go(std::integral_constant<int, 4>());
  else if (k % 2 == 0)
    go(std::integral_constant<int, 2>());
  else
    go(std::integral_constant<int, 1>());
}

// out = c_in + sign * P r for one plane block: row-major P and the row-owner
// kernel for small planes, P^T (stored transposed) and the split-K coarse
// GEMM above that size, where the GEMM's register tile is the better
// FP32-issue/HBM balance (profiles/r02_bt_rows_ab.txt)
template <class T>
void bt_step(int64_t m, int k, const cplx_t<T>* P, int64_t ld, const cplx_t<T>* r, cplx_t<T>* out,
             const cplx_t<T>* c_in, T sign, cplx_t<T>* part, const cplx_t<T>* Pnext, cudaStream_t s) {
  if (bt_rowmajor(m))
    bt_rows<T>(m, k, P, ld, r, out, c_in, sign, Pnext, s);
  else
    launch_coarse_gemm<T>(m, k, P, ld, r, out, c_in, sign, part, s);
}

}  // namespace

bool bt_rowmajor(int64_t m) {
  const char* e = std::getenv("HZ_BT_ROWS_MAX");
  return m <= (e ? int64_t(std::atoll(e)) : int64_t(2) * kNumSMs * 8);
}

// ---- sweep-axis permutation
// The factors hold 2 n_planes m^2 complex values with m the nodes per plane, so
// the solve streams N * m values: it pays to sweep along the LONGEST axis
// (planes of the two shortest). A 65 x 65 x 33 coarsest grid swept along y has
// planes of 65 x 33 = 2,145 nodes instead of 4,225: half the factor bytes
// per solve and a quarter of the Gauss-Jordan setup flops. The operator and
// the vectors are re-indexed onto the permuted grid (new axis a = old axis
// perm[a]); the solve itself is unchanged.
namespace {
struct Perm3 {
  int p[3];
  uint32_t n[3];  // old dims
};
__device__ __forceinline__ int64_t old_node(const Perm3& pm, const LevelGeom& gT, uint32_t nodeT) {
  uint32_t cT[3];
  gT.unpack(nodeT, cT[0], cT[1], cT[2]);
  uint32_t c[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < 3; ++a) c[pm.p[a]] = cT[a];
  return int64_t(c[0]) + int64_t(pm.n[0]) * (int64_t(c[1]) + int64_t(pm.n[1]) * c[2]);
}
__global__ void permute_coef_kernel(LevelGeom gT, Perm3 pm, const double2* __restrict__ coef,
                                    double2* __restrict__ coefT) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= int64_t(27) * gT.nodes) return;
  const int sT = int(e / gT.nodes);
  const uint32_t nodeT = uint32_t(e - int64_t(sT) * gT.nodes);
  const int dT[3] = {sT % 3 - 1, (sT / 3) % 3 - 1, sT / 9 - 1};
  int d[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < 3; ++a) d[pm.p[a]] = dT[a];
  coefT[e] = coef[int64_t(plane_s(d[0], d[1], d[2])) * gT.nodes + old_node(pm, gT, nodeT)];
}
// INV = false: dst[nodeT] = src[node]; true: dst[node] = src[nodeT] (k columns each)
template <class V, bool INV>
__global__ void permute_vec_kernel(LevelGeom gT, Perm3 pm, int k, const V* __restrict__ src, V* __restrict__ dst) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= int64_t(gT.nodes) * k) return;
  const uint32_t nodeT = uint32_t(e / k);
  const int q = int(e - int64_t(nodeT) * k);
  const int64_t o = old_node(pm, gT, nodeT) * k + q;
  if (INV)
    dst[o] = src[e];
  else
    dst[e] = src[o];
}
Perm3 make_perm(const LevelGeom& g, const int* perm) {
  Perm3 pm;
  for (int a = 0; a < 3; ++a) pm.p[a] = perm[a];
  pm.n[0] = g.n0;
  pm.n[1] = g.n1;
  pm.n[2] = g.n2;
  return pm;
}
}  // namespace

void bt_sweep_perm(const int64_t* dims, int* perm) {
  // sweep along the longest axis (ties: the slowest), the others in order
  int sweep = 2;
  for (int a = 1; a >= 0; --a)
    if (dims[a] > dims[sweep]) sweep = a;
  int q = 0;
  for (int a = 0; a < 3; ++a)
    if (a != sweep) perm[q++] = a;
  perm[2] = sweep;
  // planes the row-owner kernel already handles are not worth re-indexing (config 3: 33 x 33 planes, 594 vs
  // 637 us per solve); HZ_BT_PERMUTE=0 never re-indexes, =2 always does
  const char* e = std::getenv("HZ_BT_PERMUTE");
  const bool never = e && e[0] == '0', always = e && e[0] == '2';
  if (never || (!always && bt_rowmajor(dims[0] * dims[1]))) perm[0] = 0, perm[1] = 1, perm[2] = 2;
}

LevelGeom bt_permuted_geom(const LevelGeom& g, const int* perm) {
  const int64_t n[3] = {g.n0, g.n1, g.n2};
  return LevelGeom(n[perm[0]], n[perm[1]], n[perm[2]], int(g.k));
}

void bt_permute_coef(const LevelGeom& g, const int* perm, const double2* coef, double2* coefT, cudaStream_t s) {
  const LevelGeom gT = bt_permuted_geom(g, perm);
  permute_coef_kernel<<<grid_for(int64_t(27) * g.nodes, 256), 256, 0, s>>>(gT, make_perm(g, perm), coef, coefT);
  HZ_LAUNCH_CHECK();
}

template <class T>
void bt_permute_vec(const LevelGeom& g, const int* perm, int k, bool inverse, const cplx_t<T>* src, cplx_t<T>* dst,
                    cudaStream_t s) {
  using V = cplx_t<T>;
  const LevelGeom gT = bt_permuted_geom(g, perm);
  const int grid = grid_for(int64_t(g.nodes) * k, 256);
  if (inverse)
    permute_vec_kernel<V, true><<<grid, 256, 0, s>>>(gT, make_perm(g, perm), k, src, dst);
  else
    permute_vec_kernel<V, false><<<grid, 256, 0, s>>>(gT, make_perm(g, perm), k, src, dst);
  HZ_LAUNCH_CHECK();
}
template void bt_permute_vec<double>(const LevelGeom&, const int*, int, bool, const double2*, double2*, cudaStream_t);
template void bt_permute_vec<float>(const LevelGeom&, const int*, int, bool, const float2*, float2*, cudaStream_t);

// ---- twisted (two-sided) elimination
// The sweep is a chain of dependent plane steps, each too small to fill the
// GPU (latency bound), so the chain is cut in two: planes 0 .. mid-1 are
// eliminated top-down and planes np-1 .. mid+1 bottom-up, concurrently on two
// streams; the middle plane takes both Schur contributions, and the two back
// substitutions run outward concurrently again. Half the dependent steps,
// the same factor bytes. HZ_BT_TWISTED=0: mid = np-1, the one-sided sweep.
int bt_mid(int np) {
  const char* e = std::getenv("HZ_BT_TWISTED");
  if (e && e[0] == '0') return np - 1;
  return np / 2;
}

// ---- setup: E_j (every plane) and F_j (coupling factor towards the middle),
// f64, row stride inv_ld(m); row-major or transposed per bt_rowmajor(m)
void bt_factor(const LevelGeom& g, const double2* coef, double2* ET, double2* FT, cudaStream_t s) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int np = int(g.n2);
  const int mid = bt_mid(np);
  const int64_t ld = inv_ld(m);
  DevBuf<double2> S(size_t(m) * m), F1(size_t(m) * m), F2(size_t(m) * m), col(m), row(m);
  DevBuf<int> piv(m);
  const int gmm = grid_for(m * m, 256), gm = grid_for(m, 256);
  ProfScope prof("bt_factor", 0.0, s);
  auto store = [&](const double2* src, double2* dst) {
    if (bt_rowmajor(m))
      strided_copy_kernel<<<gmm, 256, 0, s>>>(m, src, dst, ld);
    else
      transpose_kernel<<<gmm, 256, 0, s>>>(m, src, dst, ld);
  };
  auto invert = [&](int j) {  // S <- S^{-1} (Gauss-Jordan, partial pivoting), stored as E_j
    for (int p = 0; p < m; ++p) {
      gj_pivot_kernel<<<1, 1024, 0, s>>>(m, S.get(), p, piv.get());
      gj_prepare_kernel<<<gm, 256, 0, s>>>(m, S.get(), p, piv.get(), col.get(), row.get());
      gj_scale_kernel<<<gm, 256, 0, s>>>(m, S.get(), p, piv.get(), col.get(), row.get());
      gj_eliminate_kernel<<<gmm, 256, 0, s>>>(m, S.get(), p, piv.get(), col.get(), row.get());
    }
    for (int p = int(m) - 1; p >= 0; --p) gj_unswap_kernel<<<gm, 256, 0, s>>>(m, S.get(), p, piv.get());
    std::vector<int> hpiv(m);
    HZ_CUDA(cudaMemcpyAsync(hpiv.data(), piv.get(), sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    HZ_CUDA(cudaStreamSynchronize(s));
    for (int64_t p = 0; p < m; ++p)
      if (hpiv[p] < 0) throw HzError(kFactorization, "block-tridiagonal coarse solve: singular plane block");
    store(S.get(), ET + int64_t(j) * m * ld);
  };
  // one chain: planes j0, j0+dir, ... up to (not including) mid
  auto chain = [&](int j0, int dir, double2* F) {
    for (int j = j0; j != mid; j += dir) {
      build_block_kernel<<<gmm, 256, 0, s>>>(g, coef, j, 0, S.get());
      if (j != j0) schur_kernel<<<gmm, 256, 0, s>>>(g, coef, j, dir, F, S.get());
      invert(j);
      mul_eu_kernel<<<gmm, 256, 0, s>>>(g, coef, j, dir, S.get(), F);
      store(F, FT + int64_t(j) * m * ld);
    }
  };
  chain(0, 1, F1.get());
  chain(np - 1, -1, F2.get());
  build_block_kernel<<<gmm, 256, 0, s>>>(g, coef, mid, 0, S.get());
  if (mid > 0) schur_kernel<<<gmm, 256, 0, s>>>(g, coef, mid, 1, F1.get(), S.get());
  if (mid < np - 1) schur_kernel<<<gmm, 256, 0, s>>>(g, coef, mid, -1, F2.get(), S.get());
  invert(mid);
  HZ_LAUNCH_CHECK();
  HZ_CUDA(cudaStreamSynchronize(s));
}

// ---- solve: x = A_c^{-1} b (k columns); scratch r (2 m k) and part (two
// split-K partial sets); aux = second stream + fork / join events
template <class T>
void bt_solve(const LevelGeom& g, const cplx_t<T>* coef, const cplx_t<T>* ET, const cplx_t<T>* FT, int k,
              const cplx_t<T>* b, cplx_t<T>* x, cplx_t<T>* r, cplx_t<T>* part, const BtAux& aux, cudaStream_t s) {
  using V = cplx_t<T>;
  const int64_t m = int64_t(g.n0) * g.n1;
  const int np = int(g.n2);
  const int mid = bt_mid(np);
  const int64_t ld = inv_ld(m);
  const int64_t pk = m * k;
  const int gk = grid_for(pk, 256);
  // (profiled by the caller, Hierarchy::coarse_solve: one scope around the direct chain or its graph)
  const bool two = mid < np - 1;  // a bottom-up chain exists
  // HZ_BT_L2PF (default 0): each row-owner plane step prefetches the chain's next factor block into L2.
  // Measured neutral on config 3 and 4 % slower on config 4 (profiles/r02_bt_pdl_ab.txt): the steps are not
  // bound by the latency of the factor loads
  const char* pfe = std::getenv("HZ_BT_L2PF");
  const int pf = pfe ? std::atoi(pfe) : 0;
  // 1: the chain's next block; 2: the step's own block (useful when the step is launched early, HZ_BT_PDL)
  auto nx = [&](const V* next, const V* self) -> const V* { return pf == 1 ? next : pf == 2 ? self : nullptr; };
  cudaStream_t s2 = two ? aux.s2 : s;
  V* r2 = r + pk;
  V* part2 = part + int64_t(std::max(coarse_split(m, k), 1)) * pk;
  auto fork = [&] {
    if (!two) return;
    HZ_CUDA(cudaEventRecord(aux.fork, s));
    HZ_CUDA(cudaStreamWaitEvent(s2, aux.fork, 0));
  };
  auto join = [&] {
    if (!two) return;
    HZ_CUDA(cudaEventRecord(aux.join, s2));
    HZ_CUDA(cudaStreamWaitEvent(s, aux.join, 0));
  };
  // forward elimination from both ends (x holds y)
  fork();
  for (int j = 0; j < mid; ++j) {
    const V* rhs = b + j * pk;
    if (j > 0) {
      launch_chain(couple_kernel<T>, dim3(gk), dim3(256), s, g, coef, j, 1, rhs, x + (j - 1) * pk, r, k);
      rhs = r;
    }
    // next on this chain: the next plane's E (the middle plane's after the last one)
    bt_step<T>(m, k, ET + int64_t(j) * m * ld, ld, rhs, x + j * pk, nullptr, T(1), part,
               nx(ET + int64_t(j + 1) * m * ld, ET + int64_t(j) * m * ld), s);
  }
  for (int j = np - 1; j > mid; --j) {
    const V* rhs = b + j * pk;
    if (j < np - 1) {
      launch_chain(couple_kernel<T>, dim3(gk), dim3(256), s2, g, coef, j, -1, rhs, x + (j + 1) * pk, r2, k);
      rhs = r2;
    }
    // next on this chain: E of plane j - 1, then the first block of its back substitution
    bt_step<T>(m, k, ET + int64_t(j) * m * ld, ld, rhs, x + j * pk, nullptr, T(1), part2,
               nx(j - 1 > mid ? ET + int64_t(j - 1) * m * ld : FT + int64_t(mid + 1) * m * ld,
                  ET + int64_t(j) * m * ld),
               s2);
  }
  join();
  {  // middle plane: both neighbours' contributions
    const V* rhs = b + mid * pk;
    if (mid > 0) {
      launch_chain(couple_kernel<T>, dim3(gk), dim3(256), s, g, coef, mid, 1, rhs, x + (mid - 1) * pk, r, k);
      rhs = r;
    }
    if (mid < np - 1) {
      launch_chain(couple_kernel<T>, dim3(gk), dim3(256), s, g, coef, mid, -1, rhs, x + (mid + 1) * pk, r, k);
      rhs = r;
    }
    bt_step<T>(m, k, ET + int64_t(mid) * m * ld, ld, rhs, x + mid * pk, nullptr, T(1), part,
               nx(mid > 0 ? FT + int64_t(mid - 1) * m * ld : nullptr, ET + int64_t(mid) * m * ld), s);
  }
  // back substitution outward: x_j = y_j - F_j x_{j +- 1}
  fork();
  for (int j = mid - 1; j >= 0; --j)
    bt_step<T>(m, k, FT + int64_t(j) * m * ld, ld, x + (j + 1) * pk, x + j * pk, x + j * pk, T(-1), part,
               nx(j > 0 ? FT + int64_t(j - 1) * m * ld : nullptr, FT + int64_t(j) * m * ld), s);
  for (int j = mid + 1; j < np; ++j)
    bt_step<T>(m, k, FT + int64_t(j) * m * ld, ld, x + (j - 1) * pk, x + j * pk, x + j * pk, T(-1), part2,
               nx(j + 1 < np ? FT + int64_t(j + 1) * m * ld : nullptr, FT + int64_t(j) * m * ld), s2);
  join();
  HZ_LAUNCH_CHECK();
}

namespace {
// B[i][q] = (i == c0 + q) for the chunk's k columns
__global__ void unit_columns_kernel(int64_t n, int k, int64_t c0, double2* __restrict__ B) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= n * k) return;
  const int64_t i = e / k;
  const int q = int(e - i * k);
  B[e] = make_double2(i == c0 + q ? 1.0 : 0.0, 0.0);
}
// ainvT[c0 + q][i] = X[i][q]  (row stride ld)
__global__ void chunk_transpose_kernel(int64_t n, int k, int64_t c0, const double2* __restrict__ X,
                                       double2* __restrict__ ainvT, int64_t ld) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= n * k) return;
  const int64_t i = e / k;
  const int q = int(e - i * k);
  if (c0 + q < n) ainvT[(c0 + q) * ld + i] = X[e];
}
}  // namespace

DevBuf<double2> bt_explicit_inverse(const LevelGeom& g, const double2* coef, const double2* ET, const double2* FT,
                                    cudaStream_t s) {
  const int64_t n = int64_t(g.nodes), m = int64_t(g.n0) * g.n1;
  constexpr int K = 64;
  DevBuf<double2> out(size_t(n) * inv_ld(n));
  DevBuf<double2> B(size_t(n) * K), X(size_t(n) * K), r(size_t(2) * m * K),
      part(size_t(2) * std::max(coarse_split(m, K), 1) * m * K);
  const LevelGeom gk(g.n0, g.n1, g.n2, K);
  BtAux aux;
  aux.ensure();
  for (int64_t c0 = 0; c0 < n; c0 += K) {
    unit_columns_kernel<<<grid_for(n * K, 256), 256, 0, s>>>(n, K, c0, B.get());
    bt_solve<double>(gk, coef, ET, FT, K, B.get(), X.get(), r.get(), part.get(), aux, s);
    chunk_transpose_kernel<<<grid_for(n * K, 256), 256, 0, s>>>(n, K, c0, X.get(), out.get(), inv_ld(n));
  }
  HZ_LAUNCH_CHECK();
  HZ_CUDA(cudaStreamSynchronize(s));
  return out;
}

template void bt_solve<double>(const LevelGeom&, const double2*, const double2*, const double2*, int,
                               const double2*, double2*, double2*, double2*, const BtAux&, cudaStream_t);
template void bt_solve<float>(const LevelGeom&, const float2*, const float2*, const float2*, int, const float2*,
                              float2*, float2*, float2*, const BtAux&, cudaStream_t);

void BtAux::ensure() {
  if (s2) return;
  HZ_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  HZ_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  HZ_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
}
BtAux::~BtAux() {
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
  if (s2) cudaStreamDestroy(s2);
}

}  // namespace hz
