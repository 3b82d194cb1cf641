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
// E_j and F_j are dense (stored transposed for the coarse GEMM kernel);
// L_j, U_j are read straight from the Galerkin stencil planes. Block LU
// without inter-plane pivoting on the shifted (complex, absorbing) operator;
// each S_j is inverted by Gauss-Jordan with partial pivoting. Agreement with
// the reference's banded LU is to cond(A_c) * eps (tested).
#include <cmath>
#include <vector>

#include "devbuf.hpp"
#include "kernels.hpp"
#include "profile.hpp"

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

// F[r][c] = sum_l E[r][l] U[l][c], U = plane j -> j+1 coupling (9 per column)
__global__ void mul_eu_kernel(LevelGeom g, const double2* __restrict__ coef, int j, const double2* __restrict__ E,
                              double2* __restrict__ F) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  const int ci = int(c % g.n0), cj = int(c / g.n0);
  double2 s = make_double2(0.0, 0.0);
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int li = ci - dx, lj = cj - dy;  // l + (dx, dy, +1) = c
      if (li < 0 || li >= int(g.n0) || lj < 0 || lj >= int(g.n1)) continue;
      const int64_t l = li + int64_t(g.n0) * lj;
      const double2 u = coef[int64_t(plane_s(dx, dy, 1)) * g.nodes + int64_t(j) * m + l];
      s = cfma(E[r * m + l], u, s);
    }
  F[e] = s;
}

// S[r][c] = D[r][c] - sum_l L[r][l] F[l][c], L = plane j+1 -> j coupling
__global__ void schur_kernel(LevelGeom g, const double2* __restrict__ coef, int j1, const double2* __restrict__ F,
                             double2* __restrict__ S) {
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
      const double2 a = coef[int64_t(plane_s(dx, dy, -1)) * g.nodes + int64_t(j1) * m + r];
      s = csub(s, cmul(a, F[l * m + c]));
    }
  S[e] = s;
}

// dst[c][r] = src[r][c] with row stride ld (transposed copy for the GEMM)
__global__ void transpose_kernel(int64_t m, const double2* __restrict__ src, double2* __restrict__ dst, int64_t ld) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * m) return;
  const int64_t r = e / m, c = e - r * m;
  dst[c * ld + r] = src[e];
}

// r = b_j - L_j y_{j-1} for one plane, all k columns
template <class T>
__global__ void couple_kernel(LevelGeom g, const cplx_t<T>* __restrict__ coef, int j, const cplx_t<T>* __restrict__ b,
                              const cplx_t<T>* __restrict__ yprev, cplx_t<T>* __restrict__ r, int k) {
  using V = cplx_t<T>;
  const int64_t m = int64_t(g.n0) * g.n1;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= m * k) return;
  const int64_t row = e / k;
  const int q = int(e - row * k);
  const int ri = int(row % g.n0), rj = int(row / g.n0);
  V s = b[e];
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int li = ri + dx, lj = rj + dy;
      if (li < 0 || li >= int(g.n0) || lj < 0 || lj >= int(g.n1)) continue;
      const int64_t l = li + int64_t(g.n0) * lj;
      const V a = coef[int64_t(plane_s(dx, dy, -1)) * g.nodes + int64_t(j) * m + row];
      s = csub(s, cmul(a, yprev[l * k + q]));
    }
  r[e] = s;
}

}  // namespace

// ---- setup: E_j^T and F_j^T (f64), row stride inv_ld(m)
void bt_factor(const LevelGeom& g, const double2* coef, double2* ET, double2* FT, cudaStream_t s) {
  const int64_t m = int64_t(g.n0) * g.n1;
  const int np = int(g.n2);
  const int64_t ld = inv_ld(m);
  DevBuf<double2> S(size_t(m) * m), F(size_t(m) * m), col(m), row(m);
  DevBuf<int> piv(m);
  const int gmm = grid_for(m * m, 256), gm = grid_for(m, 256);
  ProfScope prof("bt_factor", 0.0, s);
  build_block_kernel<<<gmm, 256, 0, s>>>(g, coef, 0, 0, S.get());
  for (int j = 0; j < np; ++j) {
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
    // S now holds E_j
    transpose_kernel<<<gmm, 256, 0, s>>>(m, S.get(), ET + int64_t(j) * m * ld, ld);
    if (j + 1 < np) {
      mul_eu_kernel<<<gmm, 256, 0, s>>>(g, coef, j, S.get(), F.get());
      transpose_kernel<<<gmm, 256, 0, s>>>(m, F.get(), FT + int64_t(j) * m * ld, ld);
      build_block_kernel<<<gmm, 256, 0, s>>>(g, coef, j + 1, 0, S.get());
      schur_kernel<<<gmm, 256, 0, s>>>(g, coef, j + 1, F.get(), S.get());
    }
  }
  HZ_LAUNCH_CHECK();
  HZ_CUDA(cudaStreamSynchronize(s));
}

// ---- solve: x = A_c^{-1} b (k columns), y/r scratch (n_c k and m k)
template <class T>
void bt_solve(const LevelGeom& g, const cplx_t<T>* coef, const cplx_t<T>* ET, const cplx_t<T>* FT, int k,
              const cplx_t<T>* b, cplx_t<T>* x, cplx_t<T>* r, cplx_t<T>* part, cudaStream_t s) {
  using V = cplx_t<T>;
  const int64_t m = int64_t(g.n0) * g.n1;
  const int np = int(g.n2);
  const int64_t ld = inv_ld(m);
  const int64_t pk = m * k;
  LevelGeom gk = g;
  ProfScope prof(sizeof(T) == 8 ? "coarse_bt_c128" : "coarse_bt_c64",
                 (2.0 * np - 1.0) * double(m) * m * sizeof(V), s, 8.0 * (2.0 * np - 1.0) * double(m) * m * k);
  // forward: x holds y
  launch_coarse_gemm<T>(m, k, ET, ld, b, x, nullptr, T(1), part, s);
  for (int j = 1; j < np; ++j) {
    couple_kernel<T><<<grid_for(pk, 256), 256, 0, s>>>(gk, coef, j, b + j * pk, x + (j - 1) * pk, r, k);
    launch_coarse_gemm<T>(m, k, ET + int64_t(j) * m * ld, ld, r, x + j * pk, nullptr, T(1), part, s);
  }
  // backward: x_j = y_j - F_j x_{j+1}
  for (int j = np - 2; j >= 0; --j)
    launch_coarse_gemm<T>(m, k, FT + int64_t(j) * m * ld, ld, x + (j + 1) * pk, x + j * pk, x + j * pk, T(-1),
                          part, s);
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
  DevBuf<double2> B(size_t(n) * K), X(size_t(n) * K), r(size_t(m) * K),
      part(size_t(std::max(coarse_split(m, K), 1)) * m * K);
  const LevelGeom gk(g.n0, g.n1, g.n2, K);
  for (int64_t c0 = 0; c0 < n; c0 += K) {
    unit_columns_kernel<<<grid_for(n * K, 256), 256, 0, s>>>(n, K, c0, B.get());
    bt_solve<double>(gk, coef, ET, FT, K, B.get(), X.get(), r.get(), part.get(), s);
    chunk_transpose_kernel<<<grid_for(n * K, 256), 256, 0, s>>>(n, K, c0, X.get(), out.get(), inv_ld(n));
  }
  HZ_LAUNCH_CHECK();
  HZ_CUDA(cudaStreamSynchronize(s));
  return out;
}

template void bt_solve<double>(const LevelGeom&, const double2*, const double2*, const double2*, int,
                               const double2*, double2*, double2*, double2*, cudaStream_t);
template void bt_solve<float>(const LevelGeom&, const float2*, const float2*, const float2*, int, const float2*,
                              float2*, float2*, float2*, cudaStream_t);

}  // namespace hz
