// Receiver sampling operator and FWI / wavefield-output kernels (acquisition.cu).
#pragma once

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "devbuf.hpp"

namespace hz {

// SamplingOperator (inc/acquisition.hpp:30-62): receiver r carries
// multilinear weights over the <= 2^ndim enclosing nodes. Stored twice on the
// device: receiver-major CSR for the gather P^T u, and its node-major
// transpose (entries in the reference's (r, q) visiting order) for the
// scatter P d, which therefore needs no atomics and sums in the reference
// order.
struct Sampling {
  Sampling(int ndim, const int64_t* n3, const double* h3, const double* origin, int64_t nrec, const double* xyz,
           int device);
  int device = 0;
  int64_t n = 0, nrec = 0, nnz = 0, ntouch = 0;
  std::vector<int64_t> rp, nodes, tnode, trp, trec;
  std::vector<double> w, tw;
  DevBuf<int64_t> d_rp, d_nodes, d_tnode, d_trp, d_trec;
  DevBuf<double> d_w, d_tw;
};

// D = P^T U  ([nrec][k] from [n][k])                      (sample)
void launch_sample(const Sampling& s, int k, const double2* U, double2* D, cudaStream_t st);
// U = P D or P conj(D)  ([n][k], fully written)           (sample_adjoint)
void launch_sample_adjoint(const Sampling& s, int k, const double2* D, double2* U, bool conj, cudaStream_t st);
// R = -w2 (1 - i gamma/w) U v                             (fwi_sensitivity_rhs)
void launch_sens_rhs(int64_t n, int k, double w2, const double2* gf, const double2* U, const double* v, double2* R,
                     cudaStream_t st);
// out[c] = max_i max(|re X[i][c]|, |im X[i][c]|)  (part: nslots * k scratch)
void launch_colmax(int64_t n, int k, const double2* X, double* part, int nslots, double* out, cudaStream_t st);
// Q[c][i] = packed (half re, half im) of X[i][c] * inv_scale[c]   (Compact16)
void launch_quantize16(int64_t n, int k, const double2* X, const double* inv_scale, uint32_t* Q, cudaStream_t st);

// B[node_j][j] = val_j for j < k (B already zeroed)      (point_source, batched)
void launch_point_sources(int k, const int64_t* nodes, const double2* vals, double2* B, cudaStream_t st);

}  // namespace hz
