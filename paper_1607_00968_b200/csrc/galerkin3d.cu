// Plane-streaming kernel of a 3D Galerkin level (27 coefficient planes), 8
// complex64 columns: apply / residual / damped Jacobi (Csr::mul_block in relax
// and cycle_rec, src/multigrid.cpp:119-136,173-175).
//
// Same scheme as stream3d.cu: 16 x 8 node tiles with all 8 columns, one
// persistent CTA per SM with an equal share of the (tile, plane) pairs, each
// plane of the tile staged by row-wise bulk copies into a 4-slot mbarrier
// ring, the issue duty rotated over the warps, z neighbours never in shared
// memory. The operator has 27 coefficients per node; a row's sum over the
// plane below, its own plane and the plane above is taken in three steps as
// those planes of the iterate pass through shared memory:
//     out(p) = sum_{s<9} c_s(p) u(p-1) + sum_{9<=s<18} c_s(p) u(p) + sum_{s>=18} c_s(p) u(p+1),
// in ascending s, i.e. in the order of the one-thread-per-element kernel
// (stencil.cu stencil_v4_kernel): bitwise equal. The coefficients therefore
// live in three per-node record arrays (s = 0..8 | 9..17 and D^-1 | 18..26,
// 80 bytes each, `LevelOp::cd`), so that the slot of iterate plane q carries
// exactly the records its three sums need -- hi(q-1), mid(q), lo(q+1) -- as
// contiguous, 16-byte aligned tile rows. Couplings that leave the grid are
// exact zeros in the records and the halo outside the grid is zero.
#include <cstdlib>
#include <map>
#include <mutex>

#include "kernels.hpp"
#include "profile.hpp"
#include "tma.cuh"

namespace hz {

namespace {

namespace g3 {

constexpr int TX = 16, TY = 8, PX = TX + 2, PY = TY + 2, CPT = 4;
constexpr int NTH = TX * TY * 2;  // 2 threads per node, 4 columns each
constexpr int NBX = 64;           // bytes per node of a complex64 8-column block
constexpr int RECB = 80;          // bytes per node of one record group
constexpr int kSlots = 4, kAhead = 2;
constexpr int U_OFF = 0;
constexpr int U_BYTES = PX * PY * NBX;                // 11,520
constexpr int REC_OFF = U_BYTES;                      // three groups of TX * TY records
constexpr int GRP_BYTES = TX * TY * RECB;             // 10,240
constexpr int B_OFF = REC_OFF + 3 * GRP_BYTES;
constexpr int B_BYTES = TX * TY * NBX;                // 8,192
constexpr int SLOT = B_OFF + B_BYTES;                 // 50,432
constexpr int kBarBytes = 128;
constexpr int SMEM = kBarBytes + kSlots * SLOT;

struct Args {
  LevelGeom g;
  const float2* x;
  const float2* b;
  float2* out;
  const float2* rec;  // [3][nodes][10]
  float wj;
  int tiles_x, tiles_y;
  const unsigned char* zeros;
};

__device__ __forceinline__ void lds4(const unsigned char* node, const int (&uo)[2], float2* v) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float4 a = *reinterpret_cast<const float4*>(node + uo[j]);
    v[2 * j] = make_float2(a.x, a.y);
    v[2 * j + 1] = make_float2(a.z, a.w);
  }
}

// MODE 0: out = A x; 1: out = b - A x; 2: out = x + wj D^-1 (b - A x)
template <int MODE>
__global__ void __launch_bounds__(NTH, 1) galerkin3d_kernel(const Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 8;
  unsigned char* slots = smem + kBarBytes;
  const LevelGeom& g = a.g;
  const int n0 = int(g.n0), n1 = int(g.n1), n2 = int(g.n2);
  const int tid = int(threadIdx.x), lane = tid & 31;
  if (tid == 0) {
    for (int q = 0; q < kSlots; ++q) {
      tma::mbar_init(&full[q], 1);
      tma::mbar_init(&empty[q], NTH / 32);
    }
    tma::fence_mbar_init();
  }
  __syncthreads();
  const int W = a.tiles_x * a.tiles_y * n2;
  const int w0 = int(int64_t(W) * blockIdx.x / gridDim.x), w1 = int(int64_t(W) * (blockIdx.x + 1) / gridDim.x);
  const int64_t grp = int64_t(g.nodes) * 10;  // float2 per record group

  // ---- producer cursor (tracked by every thread; the warps issue in turn)
  int pw = w0, ptile = 0, pz0 = 0, pz1 = 0, pp = 0, pi = 0;
  auto pseg = [&] {
    ptile = pw / n2;
    pz0 = pw - ptile * n2;
    pz1 = min(n2, pz0 + (w1 - pw));
    pp = max(pz0 - 1, 0);
  };
  if (pw < w1) pseg();
  auto issue = [&] {
    if (pw >= w1) return;
    if ((tid >> 5) == pi % (NTH / 32)) {
      const int ty = ptile / a.tiles_x;
      const int x0 = (ptile - ty * a.tiles_x) * TX, y0 = ty * TY;
      const int p = pp;
      const bool has_m = p >= pz0 && p < pz1;           // mid(p), b(p)
      const bool has_h = p - 1 >= pz0 && p - 1 < pz1;   // hi(p - 1)
      const bool has_l = p + 1 >= pz0 && p + 1 < pz1;   // lo(p + 1)
      const int slot = pi % kSlots;
      tma::mbar_wait(&empty[slot], ((pi / kSlots) & 1) ^ 1);
      unsigned char* sl = slots + slot * SLOT;
      const int xs = max(x0 - 1, 0), xe = min(x0 + TX, n0 - 1);
      const int cnt = xe - xs + 1, dcol = xs - (x0 - 1), rpad = PX - dcol - cnt;
      const int xin = min(x0 + TX, n0) - x0, rows_i = min(y0 + TY, n1) - y0;
      if (lane == 0) {
        const uint32_t ngrp = uint32_t(has_m) + uint32_t(has_h) + uint32_t(has_l);
        tma::mbar_arrive_expect_tx(&full[slot], uint32_t(U_BYTES) + uint32_t(rows_i * xin) *
                                                                       (ngrp * RECB + ((MODE != 0 && has_m) ? NBX : 0)));
      }
      __syncwarp();
      for (int c = lane; c < PY + 4 * TY; c += 32) {
        if (c < PY) {
          const int y = y0 - 1 + c;
          unsigned char* dst = sl + U_OFF + c * PX * NBX;
          if (y < 0 || y >= n1) {
            tma::bulk_g2s(dst, a.zeros, uint32_t(PX * NBX), &full[slot]);
            continue;
          }
          const unsigned char* src = reinterpret_cast<const unsigned char*>(a.x) + ((int64_t(p) * n1 + y) * n0 + xs) * NBX;
          if (dcol > 0) tma::bulk_g2s(dst, a.zeros, uint32_t(dcol * NBX), &full[slot]);
          tma::bulk_g2s(dst + dcol * NBX, src, uint32_t(cnt * NBX), &full[slot]);
          if (rpad > 0) tma::bulk_g2s(dst + (dcol + cnt) * NBX, a.zeros, uint32_t(rpad * NBX), &full[slot]);
        } else {
          const int q = (c - PY) / TY, by = (c - PY) % TY;  // q: 0 hi(p-1), 1 mid(p), 2 lo(p+1), 3 b(p)
          const int y = y0 + by;
          if (y >= n1) continue;
          if (q == 3) {
            if (MODE != 0 && has_m)
              tma::bulk_g2s(sl + B_OFF + by * TX * NBX,
                            reinterpret_cast<const unsigned char*>(a.b) + ((int64_t(p) * n1 + y) * n0 + x0) * NBX,
                            uint32_t(xin * NBX), &full[slot]);
            continue;
          }
          const bool has = q == 0 ? has_h : (q == 1 ? has_m : has_l);
          if (!has) continue;
          const int pz = p - 1 + q;        // the plane whose rows the records belong to
          const int group = 2 - q;         // hi = group 2, mid = 1, lo = 0
          const int64_t node = (int64_t(pz) * n1 + y) * n0 + x0;
          tma::bulk_g2s(sl + REC_OFF + q * GRP_BYTES + by * TX * RECB,
                        reinterpret_cast<const unsigned char*>(a.rec + group * grp) + node * RECB, uint32_t(xin * RECB),
                        &full[slot]);
        }
      }
    }
    ++pi;
    if (++pp > min(pz1, n2 - 1)) {
      pw += pz1 - pz0;
      if (pw < w1) pseg();
    }
  };
#pragma unroll 1
  for (int i = 0; i < kAhead; ++i) issue();

  // ---- consumer
  const int sub = tid & 1, nx = (tid >> 1) & (TX - 1), ny = tid >> 5;
  int uo[2];
  {
    const int swap = (nx >> 1) & 1;
    uo[0] = (2 * sub + swap) * 16;
    uo[1] = (2 * sub + 1 - swap) * 16;
  }
  const int cnode = (ny + 1) * PX + (nx + 1), inode = ny * TX + nx;
  const int64_t pstride = int64_t(n0) * n1;
  int zs = 0, ze = 0, ci = 0;
  bool active = false;
  float2* out0 = a.out;
  float2 accM[CPT], acc0[CPT];       // pending sums of out(p - 1), out(p)
  float2 xo[CPT], bo[CPT], wdo;      // own x, b and wj D^-1 of the pending plane p - 1
  float2 xc[CPT], bc[CPT], wdc;      // ... of plane p
#pragma unroll
  for (int q = 0; q < CPT; ++q) accM[q] = acc0[q] = xo[q] = bo[q] = xc[q] = bc[q] = czero<float2>();
  wdo = wdc = czero<float2>();

#pragma unroll 1
  for (int w = w0; w < w1; w += ze - zs) {
    const int tile = w / n2;
    const int ty = tile / a.tiles_x;
    const int gx = (tile - ty * a.tiles_x) * TX + nx, gy = ty * TY + ny;
    zs = w - tile * n2;
    ze = min(n2, zs + (w1 - w));
    active = gx < n0 && gy < n1;
    out0 = a.out + (int64_t(gy) * n0 + gx) * 8;
#pragma unroll 1
    for (int p = zs - 1; p <= ze; ++p) {
      const bool inside = p >= 0 && p < n2;
      const int slot = ci % kSlots;
      const unsigned char* sl = slots + slot * SLOT;
      const bool do_m = p >= zs && p < ze, do_h = p - 1 >= zs, do_l = p + 1 < ze;
      float2 accP[CPT];
#pragma unroll
      for (int q = 0; q < CPT; ++q) accP[q] = czero<float2>();
      if (inside) {
        issue();
        tma::mbar_wait(&full[slot], (ci / kSlots) & 1);
        if (active) {
          const unsigned char* un_p = sl + U_OFF + cnode * NBX;
          const float2* rh = reinterpret_cast<const float2*>(sl + REC_OFF) + inode * 10;
          const float2* rm = rh + GRP_BYTES / 8;
          const float2* rl = rm + GRP_BYTES / 8;
#pragma unroll
          for (int s9 = 0; s9 < 9; ++s9) {
            const int dy = s9 / 3 - 1, dx = s9 % 3 - 1;
            float2 u[CPT];
            lds4(un_p + (dy * PX + dx) * NBX, uo, u);
            if (s9 == 4) {
#pragma unroll
              for (int q = 0; q < CPT; ++q) xc[q] = u[q];
            }
            if (do_h) {
              const float2 c = rh[s9];
#pragma unroll
              for (int q = 0; q < CPT; ++q) accM[q] = cfma(c, u[q], accM[q]);
            }
            if (do_m) {
              const float2 c = rm[s9];
#pragma unroll
              for (int q = 0; q < CPT; ++q) acc0[q] = cfma(c, u[q], acc0[q]);
            }
            if (do_l) {
              const float2 c = rl[s9];
#pragma unroll
              for (int q = 0; q < CPT; ++q) accP[q] = cfma(c, u[q], accP[q]);
            }
          }
          if (do_m && MODE != 0) {
            lds4(sl + B_OFF + inode * NBX, uo, bc);
            const float2 d = rm[9];
            wdc = mk(a.wj * d.x, a.wj * d.y);
          }
        }
      }
      if (active && do_h) {  // plane p - 1 is complete
        float2 o[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q)
          o[q] = MODE == 0 ? accM[q] : (MODE == 1 ? csub(bo[q], accM[q]) : jacobi_upd(xo[q], wdo, bo[q], accM[q]));
        unsigned char* op_ = reinterpret_cast<unsigned char*>(out0 + int64_t(p - 1) * pstride * 8);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          *reinterpret_cast<float4*>(op_ + uo[j]) = make_float4(o[2 * j].x, o[2 * j].y, o[2 * j + 1].x, o[2 * j + 1].y);
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        accM[q] = acc0[q];
        acc0[q] = accP[q];
        xo[q] = xc[q];
        bo[q] = bc[q];
      }
      wdo = wdc;
      if (inside) {
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
        ++ci;
      }
    }
  }
}

// records [3][nodes][10] from the 27 coefficient planes and D^-1
__global__ void __launch_bounds__(256)
records_kernel(int64_t nodes, const float2* __restrict__ coef, const float2* __restrict__ inv_diag,
               float2* __restrict__ rec) {
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e >= nodes * 30) return;
  const int64_t gnode = e / 10;
  const int j = int(e - gnode * 10);
  const int group = int(gnode / nodes);
  const int64_t node = gnode - int64_t(group) * nodes;
  float2 v = make_float2(0.f, 0.f);
  if (j < 9)
    v = coef[int64_t(group * 9 + j) * nodes + node];
  else if (group == 1)
    v = inv_diag[node];
  rec[e] = v;
}

__device__ uint4 g_zeros[128];  // 2 KB >= one iterate row of the tile

const unsigned char* zeros_ptr() {
  static std::mutex mu;
  static std::map<int, const unsigned char*> ptr;
  int dev = 0;
  HZ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = ptr.find(dev);
  if (it != ptr.end()) return it->second;
  void* z = nullptr;
  HZ_CUDA(cudaGetSymbolAddress(&z, g_zeros));
  return ptr[dev] = static_cast<const unsigned char*>(z);
}

template <int MODE>
void go(const LevelOp<float>& op, float wj, const float2* x, const float2* b, float2* out, cudaStream_t s) {
  static_assert(PX * NBX <= int(sizeof(uint4)) * 128, "zero row");
  Args a;
  a.g = op.g;
  a.x = x;
  a.b = b;
  a.out = out;
  a.rec = op.cd;
  a.wj = wj;
  a.tiles_x = (int(op.g.n0) + TX - 1) / TX;
  a.tiles_y = (int(op.g.n1) + TY - 1) / TY;
  a.zeros = zeros_ptr();
  static const int forced = [] {
    const char* e = std::getenv("HZ_G3_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t W = int64_t(a.tiles_x) * a.tiles_y * op.g.n2;
  int ctas = int(std::min<int64_t>(kNumSMs, std::max<int64_t>(1, W / 8)));
  if (forced > 0) ctas = int(std::min<int64_t>(forced, W));
  auto kern = galerkin3d_kernel<MODE>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), SMEM);
  kern<<<ctas, NTH, SMEM, s>>>(a);
}

}  // namespace g3

}  // namespace

int64_t galerkin3d_min_nodes() {
  static const int64_t v = [] {
    const char* e = std::getenv("HZ_G3_MIN_NODES");
    // config 4's level 1 (129 x 129 x 65 = 1.08M nodes): sweep 235 -> 152 us; config 3's (65 x 65 x 33 = 139k
    // nodes, two groups in flight) 52.5 -> 46.6 us per sweep but 54.9 -> 50.3 RHS/s overall: one 202 KB CTA per
    // SM shuts the other group's kernels out, so small levels keep the element kernel
    return e ? int64_t(std::atoll(e)) : int64_t(500000);
  }();
  return v;
}

void launch_galerkin3d_records(int64_t nodes, const float2* coef, const float2* inv_diag, float2* rec,
                               cudaStream_t s) {
  g3::records_kernel<<<grid_for(nodes * 30, 256), 256, 0, s>>>(nodes, coef, inv_diag, rec);
  HZ_LAUNCH_CHECK();
}

bool launch_galerkin3d(const LevelOp<float>& op, int mode, float wj, const float2* x, const float2* b, float2* out,
                       cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("HZ_G3");
    return !(e && e[0] == '0');
  }();
  if (!on || op.kind != kStencil || op.ndim != 3 || op.g.k != 8 || !op.cd || op.g.z0 != 0 || op.g.z1 != op.g.n2 ||
      op.g.n2 < 2)
    return false;
  if (mode == 0)
    g3::go<0>(op, wj, x, b, out, s);
  else if (mode == 1)
    g3::go<1>(op, wj, x, b, out, s);
  else
    g3::go<2>(op, wj, x, b, out, s);
  HZ_LAUNCH_CHECK();
  return true;
}

}  // namespace hz
