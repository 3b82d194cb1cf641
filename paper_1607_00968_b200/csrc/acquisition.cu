// The steps either side of the solve in FWI: receiver sampling
// P^T u / P d (SamplingOperator, inc/acquisition.hpp:30-62), the sensitivity
// right-hand side -w^2 (1 - i gamma/w) u v (src/helmholtz_solver.cpp:95-101)
// and the Compact16 wavefield quantisation (WavefieldBatch::append,
// src/helmholtz.cpp:137-151) -- all on blocks of k sources in the solver's
// node-major [node][k] layout, so they chain with the block solve without a
// host round trip.
//
// Bitwise parity: the reference evaluates these with std::complex<double>
// and no FMA contraction; the kernels use explicitly rounded operations in
// the same order (__dmul_rn / __dadd_rn cannot be contracted by nvcc).
#include <cuda_fp16.h>

#include "acquisition.hpp"
#include "profile.hpp"

namespace hz {

namespace {

constexpr int kBlk = 256;

__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {  // naive a*b, no contraction
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// D[r][c] = sum_q w_rq U[node_rq][c], q ascending from 0 (sample)
__global__ void __launch_bounds__(kBlk)
sample_kernel(int64_t nrec, int k, const int64_t* __restrict__ rp, const int64_t* __restrict__ nodes,
              const double* __restrict__ w, const double2* __restrict__ U, double2* __restrict__ D) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= nrec * k) return;
  const int64_t r = e / k, c = e - r * k;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t q = rp[r]; q < rp[r + 1]; ++q) {
    const double2 u = U[nodes[q] * k + c];
    const double wq = w[q];
    // (w + 0i) * u = (w u.re - 0 u.im, w u.im + 0 u.re)
    acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(wq, u.x), __dmul_rn(0.0, u.y)));
    acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(wq, u.y), __dmul_rn(0.0, u.x)));
  }
  D[e] = acc;
}

// U[node][c] = sum over receivers r touching node (r ascending) of
// w (conj?) D[r][c]: the reference's scatter loop (sample_adjoint) regrouped
// per node, in the order it visits each node. Untouched nodes are zeroed by
// the caller.
__global__ void __launch_bounds__(kBlk)
sample_adjoint_kernel(int64_t ntouch, int k, const int64_t* __restrict__ tnode, const int64_t* __restrict__ trp,
                      const int64_t* __restrict__ trec, const double* __restrict__ tw,
                      const double2* __restrict__ D, double2* __restrict__ U, int conj) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= ntouch * k) return;
  const int64_t t = e / k, c = e - t * k;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t q = trp[t]; q < trp[t + 1]; ++q) {
    double2 d = D[trec[q] * k + c];
    if (conj) d.y = -d.y;
    const double wq = tw[q];
    acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(wq, d.x), __dmul_rn(0.0, d.y)));
    acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(wq, d.y), __dmul_rn(0.0, d.x)));
  }
  U[tnode[t] * k + c] = acc;
}

// R[i][c] = ((-w2 * gf[i]) * U[i][c]) * v[i]   (fwi_sensitivity_rhs)
__global__ void __launch_bounds__(kBlk)
sens_rhs_kernel(int64_t n, int k, double w2, const double2* __restrict__ gf, const double2* __restrict__ U,
                const double* __restrict__ v, double2* __restrict__ R) {
  const int64_t e = int64_t(blockIdx.x) * kBlk + threadIdx.x;
  if (e >= n * k) return;
  const int64_t i = e / k;
  const double2 g = gf[i];
  const double2 a = make_double2(__dmul_rn(-w2, g.x), __dmul_rn(-w2, g.y));
  const double2 p = cmul_rn(a, U[e]);
  const double vi = v[i];
  R[e] = make_double2(__dmul_rn(p.x, vi), __dmul_rn(p.y, vi));
}

// per-slot column maxima of max(|re|, |im|) (max is order independent)
__global__ void __launch_bounds__(kBlk)
colmax_kernel(int64_t n, int k, const double2* __restrict__ X, double* __restrict__ part, int nslots) {
  extern __shared__ double red[];
  const int64_t rows_per = (n + nslots - 1) / nslots;
  const int64_t r0 = int64_t(blockIdx.x) * rows_per;
  const int64_t r1 = r0 + rows_per < n ? r0 + rows_per : n;
  // threads stride over (row, column) elements of the slot; column = e % k
  // stays fixed per thread when kBlk % k == 0 (k | 256 for k <= 256 powers
  // of two), otherwise a per-thread column table is used
  for (int c = threadIdx.x; c < k; c += kBlk) red[c] = 0.0;
  __syncthreads();
  const int64_t e0 = r0 * k, e1 = r1 * k;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kBlk) {
    const double2 x = X[e];
    const double m = fmax(fabs(x.x), fabs(x.y));
    const int c = int(e % k);
    // atomicMax on the bit pattern is exact for non-negative doubles
    atomicMax(reinterpret_cast<unsigned long long*>(&red[c]), __double_as_longlong(m));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kBlk) part[int64_t(blockIdx.x) * k + c] = red[c];
}

__global__ void colmax_reduce_kernel(int k, int nslots, const double* __restrict__ part, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  double m = 0.0;
  for (int s = 0; s < nslots; ++s) m = fmax(m, part[int64_t(s) * k + c]);
  out[c] = m;
}

// Q[c][i] = (half(float(re/scale_c)), half(float(im/scale_c))), source-major.
// A CTA transposes a 32-node x k tile through shared memory so both the
// node-major reads and the source-major writes are coalesced.
__global__ void __launch_bounds__(kBlk)
quantize_kernel(int64_t n, int k, const double2* __restrict__ X, const double* __restrict__ inv_scale,
                uint32_t* __restrict__ Q) {
  extern __shared__ uint32_t tile[];  // [k][33]
  const int64_t i0 = int64_t(blockIdx.x) * 32;
  const int rows = int(n - i0 < 32 ? n - i0 : 32);
  for (int e = threadIdx.x; e < rows * k; e += kBlk) {
    const int r = e / k, c = e - r * k;
    const double2 x = X[(i0 + r) * k + c];
    const double s = inv_scale[c];
    const __half hr = __float2half_rn(__double2float_rn(__dmul_rn(x.x, s)));
    const __half hi = __float2half_rn(__double2float_rn(__dmul_rn(x.y, s)));
    tile[c * 33 + r] = uint32_t(__half_as_ushort(hr)) | (uint32_t(__half_as_ushort(hi)) << 16);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * k; e += kBlk) {
    const int c = e / rows, r = e - c * rows;
    Q[int64_t(c) * n + i0 + r] = tile[c * 33 + r];
  }
}

}  // namespace

void launch_sample(const Sampling& s, int k, const double2* U, double2* D, cudaStream_t st) {
  if (s.nrec == 0) return;
  ProfScope prof("sample", double(s.nnz) * k * 16 + double(s.nrec) * k * 16, st);
  sample_kernel<<<grid_for(s.nrec * k, kBlk), kBlk, 0, st>>>(s.nrec, k, s.d_rp.get(), s.d_nodes.get(),
                                                             s.d_w.get(), U, D);
  HZ_LAUNCH_CHECK();
}

void launch_sample_adjoint(const Sampling& s, int k, const double2* D, double2* U, bool conj, cudaStream_t st) {
  HZ_CUDA(cudaMemsetAsync(U, 0, sizeof(double2) * size_t(s.n) * k, st));
  if (s.ntouch == 0) return;
  ProfScope prof("sample_adjoint", double(s.nnz) * k * 16 + double(s.ntouch) * k * 16, st);
  sample_adjoint_kernel<<<grid_for(s.ntouch * k, kBlk), kBlk, 0, st>>>(
      s.ntouch, k, s.d_tnode.get(), s.d_trp.get(), s.d_trec.get(), s.d_tw.get(), D, U, conj ? 1 : 0);
  HZ_LAUNCH_CHECK();
}

void launch_sens_rhs(int64_t n, int k, double w2, const double2* gf, const double2* U, const double* v, double2* R,
                     cudaStream_t st) {
  ProfScope prof("sensitivity_rhs", double(n) * (2.0 * k * 16 + 16 + 8), st);
  sens_rhs_kernel<<<grid_for(n * k, kBlk), kBlk, 0, st>>>(n, k, w2, gf, U, v, R);
  HZ_LAUNCH_CHECK();
}

void launch_colmax(int64_t n, int k, const double2* X, double* part, int nslots, double* out, cudaStream_t st) {
  ProfScope prof("colmax", double(n) * k * 16, st);
  colmax_kernel<<<nslots, kBlk, sizeof(double) * k, st>>>(n, k, X, part, nslots);
  HZ_LAUNCH_CHECK();
  colmax_reduce_kernel<<<grid_for(k, 64), 64, 0, st>>>(k, nslots, part, out);
  HZ_LAUNCH_CHECK();
}

void launch_quantize16(int64_t n, int k, const double2* X, const double* inv_scale, uint32_t* Q, cudaStream_t st) {
  ProfScope prof("quantize16", double(n) * k * (16 + 4), st);
  const size_t smem = sizeof(uint32_t) * size_t(k) * 33;
  allow_dyn_smem(reinterpret_cast<const void*>(quantize_kernel), int(smem));
  quantize_kernel<<<grid_for(n, 32), kBlk, smem, st>>>(n, k, X, inv_scale, Q);
  HZ_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- host side
// SamplingOperator ctor (src/acquisition.cpp:33-62) with the bounding-box
// check of RegularGrid::contains (src/grid.cpp:36-44).
Sampling::Sampling(int ndim, const int64_t* n3, const double* h3, const double* origin, int64_t nrec_,
                   const double* xyz, int device_)
    : device(device_), nrec(nrec_) {
  n = n3[0] * n3[1] * n3[2];
  if (nrec < 0) throw HzError(kValidation, "sampling: negative receiver count");
  rp.assign(1, 0);
  for (int64_t r = 0; r < nrec; ++r) {
    const double* x = xyz + 3 * r;
    for (int a = 0; a < ndim; ++a) {
      const double eps = 1e-9;
      const double lo = origin[a] - eps * h3[a];
      const double hi = origin[a] + (n3[a] - 1) * h3[a] + eps * h3[a];
      if (x[a] < lo || x[a] > hi)
        throw HzError(kValidation, "sampling: receiver " + std::to_string(r) + " outside grid");
    }
    int64_t base[3] = {0, 0, 0};
    double t[3] = {0, 0, 0};
    for (int a = 0; a < ndim; ++a) {
      double f = (x[a] - origin[a]) / h3[a];
      f = std::clamp(f, 0.0, double(n3[a] - 1));
      int64_t b = int64_t(std::floor(f));
      b = std::clamp<int64_t>(b, 0, n3[a] - 2);
      base[a] = b;
      t[a] = f - double(b);
    }
    const int corners = 1 << ndim;
    for (int c = 0; c < corners; ++c) {
      double wgt = 1.0;
      int64_t idx[3] = {base[0], base[1], base[2]};
      for (int a = 0; a < ndim; ++a) {
        const int bit = (c >> a) & 1;
        wgt *= bit ? t[a] : (1.0 - t[a]);
        idx[a] += bit;
      }
      if (wgt == 0.0) continue;
      nodes.push_back(idx[0] + n3[0] * (idx[1] + n3[1] * idx[2]));
      w.push_back(wgt);
    }
    rp.push_back(int64_t(nodes.size()));
  }
  nnz = int64_t(nodes.size());
  // node-major transpose, entries in the reference's visiting order (r, q)
  std::vector<std::pair<int64_t, int64_t>> ent;  // (node, entry)
  ent.reserve(nnz);
  for (int64_t e = 0; e < nnz; ++e) ent.push_back({nodes[e], e});
  std::stable_sort(ent.begin(), ent.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int64_t> rec_of(nnz);
  for (int64_t r = 0; r < nrec; ++r)
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) rec_of[e] = r;
  trp.assign(1, 0);
  for (size_t i = 0; i < ent.size(); ++i) {
    if (i == 0 || ent[i].first != ent[i - 1].first) {
      if (i > 0) trp.push_back(int64_t(i));
      tnode.push_back(ent[i].first);
    }
    trec.push_back(rec_of[ent[i].second]);
    tw.push_back(w[ent[i].second]);
  }
  if (!ent.empty()) trp.push_back(int64_t(ent.size()));
  ntouch = int64_t(tnode.size());
  DeviceGuard g(device);
  auto up64 = [](DevBuf<int64_t>& d, const std::vector<int64_t>& v) {
    d.alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) HZ_CUDA(cudaMemcpy(d.get(), v.data(), v.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  };
  auto upd = [](DevBuf<double>& d, const std::vector<double>& v) {
    d.alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) HZ_CUDA(cudaMemcpy(d.get(), v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
  };
  up64(d_rp, rp);
  up64(d_nodes, nodes);
  upd(d_w, w);
  up64(d_tnode, tnode);
  up64(d_trp, trp);
  up64(d_trec, trec);
  upd(d_tw, tw);
}

namespace {
constexpr int kMaxPointSources = 64;
struct PointSources {
  int64_t node[kMaxPointSources];
  double2 val[kMaxPointSources];
};
// one thread per source column (K15: k nonzeros per block)
__global__ void point_sources_kernel(int c, int ld, PointSources ps, double2* __restrict__ B) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < c) B[ps.node[j] * ld + j] = ps.val[j];
}
}  // namespace

void launch_point_sources(int k, const int64_t* nodes, const double2* vals, double2* B, cudaStream_t st) {
  for (int j0 = 0; j0 < k; j0 += kMaxPointSources) {
    // columns [j0, j0 + c) of the [n][k] block: view it as a block whose
    // column j0 is at B + j0 (same row stride k)
    const int c = std::min(kMaxPointSources, k - j0);
    PointSources ps;
    for (int j = 0; j < c; ++j) {
      ps.node[j] = nodes[j0 + j];
      ps.val[j] = vals[j0 + j];
    }
    ProfScope prof("point_sources", double(c) * 16, st);
    point_sources_kernel<<<1, kMaxPointSources, 0, st>>>(c, k, ps, B + j0);
    HZ_LAUNCH_CHECK();
  }
}

}  // namespace hz
