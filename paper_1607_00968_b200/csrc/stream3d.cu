// Plane-streaming kernels of the 3D fine level for 8-column blocks.
//
// apply / residual / damped Jacobi of the 7-point (HelmholtzProblem::apply_block,
// src/helmholtz.cpp:71-100; relax, src/multigrid.cpp:119-136) and of the compact
// 27-point fine operator, over x[node][8]:
//
//  * A CTA owns an (x, y) tile of TX x TY nodes with all 8 columns and walks a
//    chunk of z planes. A producer warp streams each plane of the tile -- the
//    iterate with a one-node halo, the per-node 16-byte operator records with
//    the halo, b and D^-1 of the interior -- into a ring of shared-memory
//    slots with row-wise bulk copies (cp.async.bulk) that complete on the
//    slot's mbarrier; 16 consumer warps wait on it, compute, and hand the
//    slot back through a second mbarrier. There is no CTA-wide barrier in the
//    loop and no consumer thread ever waits on a global load.
//  * Every plane is read from L2/HBM once per tile (plus the halo ring), where
//    the one-thread-per-element kernels fetch each z / y neighbour plane again
//    through L2 (3-9 times the traffic into the SM for the 27-point operator).
//  * z neighbours never touch shared memory: a thread keeps its own node's
//    previous plane in registers and finishes the output of plane p - 1 when
//    plane p arrives.
//  * 7-point: the same per-column operations in the same order as the
//    element kernels (stencil.cu fine_v4_kernel), so the results are bitwise
//    equal. 27-point: the couplings lap[q] + mu[q] (M_i + M_j) / 2 are never
//    formed; with Qc(f) the sum of a field f over the in-plane neighbours of
//    class c (faces, corners) the row is
//        sum_j lap[q] u_j + (mu[q]/2) M_j u_j  +  M_i sum_j (mu[q]/2) u_j,
//    accumulated per plane as same-plane (A) and adjacent-plane (B) parts of
//    the two channels, out(p) = A1(p) + B1(p-1) + B1(p+1) + M_i (A2(p) +
//    B2(p-1) + B2(p+1)): 96 flops per column instead of 27 complex FMAs plus
//    the coupling arithmetic, and only the current plane in shared memory.
//  * Shared-memory reads are 16 bytes per thread; the two 16-byte units a
//    thread owns in a node are taken in opposite order by neighbouring nodes,
//    so the 8 threads of a quarter-warp always cover all 32 banks.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "profile.hpp"
#include "tma.cuh"

namespace hz {

namespace {

namespace s3 {

constexpr int kSlots = 4;
constexpr int kBarBytes = 128;

template <class T, class XV>
struct Tile;
template <>
struct Tile<float, float2> {
  static constexpr int TX = 32, TY = 8, CPT = 4;
};
template <>
struct Tile<double, double2> {
  static constexpr int TX = 16, TY = 8, CPT = 2;
};
template <>
struct Tile<double, float2> {  // complex128 operator on a complex64 block
  static constexpr int TX = 16, TY = 8, CPT = 2;
};

constexpr int pad128(int b) { return (b + 127) / 128 * 128; }

template <class T, class XV, int MODE>
struct Cfg {
  using V = cplx_t<T>;
  using TL = Tile<T, XV>;
  static constexpr int TX = TL::TX, TY = TL::TY, CPT = TL::CPT;
  static constexpr int PX = TX + 2, PY = TY + 2;
  static constexpr int NBX = 8 * int(sizeof(XV));  // bytes per node of x
  static constexpr int NBV = 8 * int(sizeof(V));   // bytes per node of b
  static constexpr int CPU = 16 / int(sizeof(XV));  // columns per 16-byte unit
  static constexpr int NU = CPT / CPU;              // units per thread
  static constexpr int TPN = 8 / CPT;               // threads per node
  static constexpr int NCONS = TX * TY * TPN;
  static constexpr int NTHREADS = NCONS + 32;
  static constexpr bool HAS_B = MODE != 0;
  static constexpr bool HAS_D = MODE == 2 && sizeof(T) == 8;
  static constexpr int U_OFF = 0;
  static constexpr int REC_OFF = pad128(PX * PY * NBX);
  static constexpr int B_OFF = REC_OFF + pad128(PX * PY * 16);
  static constexpr int D_OFF = B_OFF + (HAS_B ? pad128(TX * TY * NBV) : 0);
  static constexpr int SLOT = D_OFF + (HAS_D ? pad128(TX * TY * 16) : 0);
  static constexpr int SMEM = kBarBytes + kSlots * SLOT;
  static_assert(NU == 1 || NU == 2, "one or two 16-byte units per thread");
  static_assert(NCONS % 32 == 0 && PY + PY + TY + TY <= 64, "tile shape");
};

template <class T, class XV, class Out>
struct Args {
  LevelOp<T> op;
  const XV* x;
  const cplx_t<T>* b;
  Out* out;
  const void* rec;  // 16-byte per-node records: c64 (centre | M, D^-1); c128 centre | M
  T wj;
  int tiles_x, tiles_y, zlen;
};

// the CPT columns a thread owns of one node, read from a shared-memory tile
template <class V, class XV, int NU>
__device__ __forceinline__ void lds_cols(const unsigned char* node, const int (&uo)[2], V* v) {
  if constexpr (std::is_same<XV, float2>::value && std::is_same<V, float2>::value) {
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      const float4 a = *reinterpret_cast<const float4*>(node + uo[j]);
      v[2 * j] = make_float2(a.x, a.y);
      v[2 * j + 1] = make_float2(a.z, a.w);
    }
  } else if constexpr (std::is_same<XV, double2>::value) {
#pragma unroll
    for (int j = 0; j < NU; ++j) v[j] = *reinterpret_cast<const double2*>(node + uo[j]);
  } else {  // complex64 storage widened to complex128 (exact)
    const float4 a = *reinterpret_cast<const float4*>(node + uo[0]);
    v[0] = make_double2(double(a.x), double(a.y));
    v[1] = make_double2(double(a.z), double(a.w));
  }
}

// ... written to the node's record in global memory (Out may be wider than V)
template <class V, class XV, class Out, int NU>
__device__ __forceinline__ void stg_cols(Out* node, const int (&uo)[2], const V* v) {
  unsigned char* p = reinterpret_cast<unsigned char*>(node);
  if constexpr (std::is_same<Out, float2>::value) {
#pragma unroll
    for (int j = 0; j < NU; ++j)
      *reinterpret_cast<float4*>(p + uo[j]) = make_float4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
  } else if constexpr (std::is_same<XV, double2>::value) {
#pragma unroll
    for (int j = 0; j < NU; ++j) *reinterpret_cast<double2*>(p + uo[j]) = v[j];
  } else {  // 2 columns per 16-byte unit of x, 32 bytes of complex128 output
#pragma unroll
    for (int j = 0; j < NU; ++j) {
      *reinterpret_cast<double2*>(p + 2 * uo[j]) = make_double2(double(v[2 * j].x), double(v[2 * j].y));
      *reinterpret_cast<double2*>(p + 2 * uo[j] + 16) = make_double2(double(v[2 * j + 1].x), double(v[2 * j + 1].y));
    }
  }
}

template <class T>
__device__ __forceinline__ void rec_load(const unsigned char* p, cplx_t<T>& c, cplx_t<T>& d) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    c = make_float2(a.x, a.y);
    d = make_float2(a.z, a.w);
  } else {
    c = *reinterpret_cast<const double2*>(p);
    d = c;
  }
}
template <class T>
__device__ __forceinline__ cplx_t<T> rec_first(const unsigned char* p) {
  if constexpr (sizeof(T) == 4)
    return *reinterpret_cast<const float2*>(p);
  else
    return *reinterpret_cast<const double2*>(p);
}

// MODE 0: out = A x; 1: out = b - A x (Csr order); 2: out = x + wj D^-1 (b - A x);
// 3: out = b - A x with A x in apply_block order (kFine)
template <class T, class XV, class Out, int KIND, int MODE>
__global__ void __launch_bounds__((Cfg<T, XV, MODE>::NTHREADS), 1)
stream3d_kernel(const Args<T, XV, Out> a) {
  using C = Cfg<T, XV, MODE>;
  using V = cplx_t<T>;
  constexpr int CPT = C::CPT, NU = C::NU, TX = C::TX, TY = C::TY, PX = C::PX, PY = C::PY;
  constexpr bool CSR = MODE == 1 || MODE == 2;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kSlots;
  unsigned char* slots = smem + kBarBytes;

  const LevelGeom& g = a.op.g;
  const int n0 = int(g.n0), n1 = int(g.n1), n2 = int(g.n2);
  const int item = int(blockIdx.x);
  const int tx = item % a.tiles_x, tr = item / a.tiles_x;
  const int ty = tr % a.tiles_y, zc = tr / a.tiles_y;
  const int x0 = tx * TX, y0 = ty * TY;
  const int zs = zc * a.zlen, ze = min(zs + a.zlen, n2);
  const int tid = int(threadIdx.x);

  // out-of-grid halo positions stay zero for the whole kernel: the copies
  // below never write them
  for (int i = tid; i < kSlots * C::SLOT / 16; i += C::NTHREADS)
    reinterpret_cast<uint4*>(slots)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {
    for (int q = 0; q < kSlots; ++q) {
      tma::mbar_init(&full[q], 1);
      tma::mbar_init(&empty[q], C::NCONS / 32);
    }
    tma::fence_mbar_init();
  }
  tma::fence_proxy_async();
  __syncthreads();

  const int pfirst = max(zs - 1, 0), plast = min(ze, n2 - 1);  // planes streamed

  if (tid >= C::NCONS) {
    // ------------------------------------------------------------ producer
    const int lane = tid - C::NCONS;
    const int xs = max(x0 - 1, 0), xe = min(x0 + TX, n0 - 1);
    const int cnt = xe - xs + 1, dcol = xs - (x0 - 1);
    const int xin = min(x0 + TX, n0) - x0;
    const int rows_h = min(y0 + TY, n1 - 1) - max(y0 - 1, 0) + 1;
    const int rows_i = min(y0 + TY, n1) - y0;
    const uint32_t bytes_h = uint32_t(rows_h) * uint32_t(cnt) * uint32_t(C::NBX + 16);
    const uint32_t bytes_i = uint32_t(rows_i) * uint32_t(xin) * uint32_t((C::HAS_B ? C::NBV : 0) + (C::HAS_D ? 16 : 0));
    const unsigned char* xg = reinterpret_cast<const unsigned char*>(a.x);
    const unsigned char* rg = reinterpret_cast<const unsigned char*>(a.rec);
    const unsigned char* bg = reinterpret_cast<const unsigned char*>(a.b);
    const unsigned char* dg = reinterpret_cast<const unsigned char*>(a.op.inv_diag);
    int it = 0;
    for (int p = pfirst; p <= plast; ++p, ++it) {
      const int slot = it % kSlots;
      tma::mbar_wait(&empty[slot], ((it / kSlots) & 1) ^ 1);
      unsigned char* sl = slots + slot * C::SLOT;
      const bool outp = p >= zs && p < ze;
      if (lane == 0) tma::mbar_arrive_expect_tx(&full[slot], bytes_h + (outp ? bytes_i : 0u));
      __syncwarp();
      for (int c = lane; c < 2 * PY + 2 * TY; c += 32) {
        if (c < 2 * PY) {
          const int ry = c < PY ? c : c - PY;
          const int y = y0 - 1 + ry;
          if (y < 0 || y >= n1) continue;
          const int64_t node = (int64_t(p) * n1 + y) * n0 + xs;
          const int dn = ry * PX + dcol;
          if (c < PY)
            tma::bulk_g2s(sl + C::U_OFF + dn * C::NBX, xg + node * C::NBX, uint32_t(cnt) * C::NBX, &full[slot]);
          else
            tma::bulk_g2s(sl + C::REC_OFF + dn * 16, rg + node * 16, uint32_t(cnt) * 16, &full[slot]);
        } else {
          if (!outp) continue;
          const bool isb = c < 2 * PY + TY;
          const int by = isb ? c - 2 * PY : c - 2 * PY - TY;
          const int y = y0 + by;
          if (y >= n1) continue;
          const int64_t node = (int64_t(p) * n1 + y) * n0 + x0;
          if (isb) {
            if constexpr (C::HAS_B)
              tma::bulk_g2s(sl + C::B_OFF + by * TX * C::NBV, bg + node * C::NBV, uint32_t(xin) * C::NBV, &full[slot]);
          } else {
            if constexpr (C::HAS_D)
              tma::bulk_g2s(sl + C::D_OFF + by * TX * 16, dg + node * 16, uint32_t(xin) * 16, &full[slot]);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int lane = tid & 31;
  const int sub = tid % C::TPN, nx = (tid / C::TPN) % TX, ny = tid / (C::TPN * TX);
  const int gx = x0 + nx, gy = y0 + ny;
  const bool active = gx < n0 && gy < n1;
  int uo[2];
  if constexpr (NU == 2) {
    const int swap = (nx / (128 / C::NBX)) & 1;
    uo[0] = (2 * sub + swap) * 16;
    uo[1] = (2 * sub + 1 - swap) * 16;
  } else {
    uo[0] = sub * 16;
    uo[1] = 0;
  }
  const int cnode = (ny + 1) * PX + (nx + 1);
  const int inode = ny * TX + nx;
  const int64_t pstride = int64_t(n0) * n1;
  const int64_t node0 = int64_t(gy) * n0 + gx;
  const bool xm = gx > 0, xp = gx + 1 < n0, ym = gy > 0, yp = gy + 1 < n1;
  const T wx = a.op.w[0], wy = a.op.w[1], wz = a.op.w[2];

  V uprev[CPT], bh[CPT], wd = czero<V>();
#pragma unroll
  for (int q = 0; q < CPT; ++q) uprev[q] = bh[q] = czero<V>();

  auto finish = [&](int p, const V* ax) {  // output of plane p from A x
    V o[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      if (MODE == 0)
        o[q] = ax[q];
      else if (MODE == 1 || MODE == 3)
        o[q] = csub(bh[q], ax[q]);
      else if (KIND == kFine)
        o[q] = cadd(uprev[q], cmul(wd, csub(bh[q], ax[q])));
      else
        o[q] = jacobi_upd(uprev[q], wd, bh[q], ax[q]);
    }
    stg_cols<V, XV, Out, NU>(a.out + (int64_t(p) * pstride + node0) * 8, uo, o);
  };
  auto hold = [&](const unsigned char* sl, V dsm) {  // b and wj D^-1 of the plane being started
    if constexpr (C::HAS_B) lds_cols<V, V, NU>(sl + C::B_OFF + inode * C::NBV, uo, bh);
    if constexpr (MODE == 2) {
      V d = dsm;
      if constexpr (C::HAS_D) d = *reinterpret_cast<const V*>(sl + C::D_OFF + inode * 16);
      wd = mk(a.wj * d.x, a.wj * d.y);
    }
  };

  int it = 0;
  if constexpr (KIND == kFine) {
    V acc[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) acc[q] = czero<V>();
    for (int p = zs - 1; p <= ze; ++p) {
      const bool inside = p >= 0 && p < n2;
      const int slot = it % kSlots;
      const unsigned char* sl = slots + slot * C::SLOT;
      if (inside) tma::mbar_wait(&full[slot], (it / kSlots) & 1);
      if (active) {
        V un[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) un[q] = czero<V>();
        const unsigned char* un_p = sl + C::U_OFF + cnode * C::NBX;
        if (inside) lds_cols<V, XV, NU>(un_p, uo, un);
        if (p - 1 >= zs) {
          if (inside) {
#pragma unroll
            for (int q = 0; q < CPT; ++q) acc[q] = crfma(wz, un[q], acc[q]);
          }
          finish(p - 1, acc);
        }
        if (p >= zs && p < ze) {
          V uxm[CPT], uxp[CPT], uym[CPT], uyp[CPT], c, d;
          lds_cols<V, XV, NU>(un_p - C::NBX, uo, uxm);
          lds_cols<V, XV, NU>(un_p + C::NBX, uo, uxp);
          lds_cols<V, XV, NU>(un_p - PX * C::NBX, uo, uym);
          lds_cols<V, XV, NU>(un_p + PX * C::NBX, uo, uyp);
          rec_load<T>(sl + C::REC_OFF + cnode * 16, c, d);
          const bool zm = p > 0;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            V s;
            if (!CSR) {
              s = cmul(c, un[q]);
              if (xm) s = crfma(wx, uxm[q], s);
              if (xp) s = crfma(wx, uxp[q], s);
              if (ym) s = crfma(wy, uym[q], s);
              if (yp) s = crfma(wy, uyp[q], s);
              if (zm) s = crfma(wz, uprev[q], s);
            } else {
              s = czero<V>();
              if (zm) s = crfma(wz, uprev[q], s);
              if (ym) s = crfma(wy, uym[q], s);
              if (xm) s = crfma(wx, uxm[q], s);
              s = cfma(c, un[q], s);
              if (xp) s = crfma(wx, uxp[q], s);
              if (yp) s = crfma(wy, uyp[q], s);
            }
            acc[q] = s;
          }
          hold(sl, d);
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) uprev[q] = un[q];
      }
      if (inside) {
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
        ++it;
      }
    }
  } else {
    // compact 27-point operator: channel 1 = lap . u + (mu / 2) . (M u),
    // channel 2 = (mu / 2) . u (times the row's own M at the end)
    const T l0 = a.op.w27[0], l1 = a.op.w27[1], l2 = a.op.w27[2], l3 = a.op.w27[3];
    const T m0 = a.op.w27[4], h1 = T(0.5) * a.op.w27[5], h2 = T(0.5) * a.op.w27[6], h3 = T(0.5) * a.op.w27[7];
    V S1[CPT], S2[CPT], P1[CPT], P2[CPT], Mo = czero<V>();
#pragma unroll
    for (int q = 0; q < CPT; ++q) S1[q] = S2[q] = P1[q] = P2[q] = czero<V>();
    for (int p = zs - 1; p <= ze; ++p) {
      const bool inside = p >= 0 && p < n2;
      const int slot = it % kSlots;
      const unsigned char* sl = slots + slot * C::SLOT;
      if (inside) tma::mbar_wait(&full[slot], (it / kSlots) & 1);
      if (active) {
        V un[CPT], A1[CPT], A2[CPT], B1[CPT], B2[CPT], Mn = czero<V>(), dn = czero<V>();
#pragma unroll
        for (int q = 0; q < CPT; ++q) un[q] = A1[q] = A2[q] = B1[q] = B2[q] = czero<V>();
        if (inside) {
          const unsigned char* un_p = sl + C::U_OFF + cnode * C::NBX;
          const unsigned char* rc_p = sl + C::REC_OFF + cnode * 16;
          lds_cols<V, XV, NU>(un_p, uo, un);
          rec_load<T>(rc_p, Mn, dn);
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const V v0 = cmul(Mn, un[q]);
            A1[q] = crfma(m0, v0, cscale(l0, un[q]));
            B1[q] = crfma(h1, v0, cscale(l1, un[q]));
            B2[q] = cscale(h1, un[q]);
          }
          // in-plane faces, then corners: Q(u) and Q(M u) folded into the channels
#pragma unroll
          for (int cls = 1; cls <= 2; ++cls) {
            V qu[CPT], qv[CPT];
#pragma unroll
            for (int q = 0; q < CPT; ++q) qu[q] = qv[q] = czero<V>();
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
              const int dx = cls == 1 ? (nb == 0 ? -1 : nb == 1 ? 1 : 0) : (nb & 1 ? 1 : -1);
              const int dy = cls == 1 ? (nb == 2 ? -1 : nb == 3 ? 1 : 0) : (nb & 2 ? 1 : -1);
              V w[CPT];
              lds_cols<V, XV, NU>(un_p + (dy * PX + dx) * C::NBX, uo, w);
              const V Mj = rec_first<T>(rc_p + (dy * PX + dx) * 16);
#pragma unroll
              for (int q = 0; q < CPT; ++q) {
                qu[q] = cadd(qu[q], w[q]);
                qv[q] = cfma(Mj, w[q], qv[q]);
              }
            }
            const T la = cls == 1 ? l1 : l2, ha = cls == 1 ? h1 : h2;  // same plane
            const T lb = cls == 1 ? l2 : l3, hb = cls == 1 ? h2 : h3;  // adjacent planes
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              A1[q] = crfma(ha, qv[q], crfma(la, qu[q], A1[q]));
              A2[q] = crfma(ha, qu[q], A2[q]);
              B1[q] = crfma(hb, qv[q], crfma(lb, qu[q], B1[q]));
              B2[q] = crfma(hb, qu[q], B2[q]);
            }
          }
        }
        if (p - 1 >= zs) {
          V ax[CPT];
#pragma unroll
          for (int q = 0; q < CPT; ++q) ax[q] = cfma(Mo, cadd(S2[q], B2[q]), cadd(S1[q], B1[q]));
          finish(p - 1, ax);
        }
        if (p >= zs && p < ze) {
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            S1[q] = cadd(A1[q], P1[q]);
            S2[q] = cadd(A2[q], P2[q]);
          }
          Mo = Mn;
          hold(sl, dn);
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          P1[q] = B1[q];
          P2[q] = B2[q];
          uprev[q] = un[q];
        }
      }
      if (inside) {
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
        ++it;
      }
    }
  }
}

bool enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HZ_STREAM3D");
    return !(e && e[0] == '0');
  }();
  return on;
}

// planes per z chunk: whole waves of one CTA per SM, two halo planes per chunk
int choose_zlen(int tiles, int n2) {
  int best = n2;
  double best_cost = 1e300;
  for (int zc = 1; zc <= 32 && (zc == 1 || n2 / zc >= 4); ++zc) {
    const int zlen = (n2 + zc - 1) / zc;
    const int chunks = (n2 + zlen - 1) / zlen;
    const int waves = (tiles * chunks + kNumSMs - 1) / kNumSMs;
    const double cost = double(waves) * (zlen + 2 + 2);  // + ring fill
    if (cost < best_cost) {
      best_cost = cost;
      best = zlen;
    }
  }
  static const int forced = [] {
    const char* e = std::getenv("HZ_STREAM3D_ZLEN");
    return e ? std::atoi(e) : 0;
  }();
  return forced > 0 ? std::min(forced, n2) : best;
}

template <class T, class XV, class Out, int KIND, int MODE>
void go(const LevelOp<T>& op, const XV* x, const cplx_t<T>* b, Out* out, const void* rec, T wj, cudaStream_t s) {
  using C = Cfg<T, XV, MODE>;
  Args<T, XV, Out> a;
  a.op = op;
  a.x = x;
  a.b = b;
  a.out = out;
  a.rec = rec;
  a.wj = wj;
  a.tiles_x = (int(op.g.n0) + C::TX - 1) / C::TX;
  a.tiles_y = (int(op.g.n1) + C::TY - 1) / C::TY;
  a.zlen = choose_zlen(a.tiles_x * a.tiles_y, int(op.g.n2));
  const int chunks = (int(op.g.n2) + a.zlen - 1) / a.zlen;
  auto kern = stream3d_kernel<T, XV, Out, KIND, MODE>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), C::SMEM);
  kern<<<a.tiles_x * a.tiles_y * chunks, C::NTHREADS, C::SMEM, s>>>(a);
}

}  // namespace s3

template <class T>
const void* rec_of(const LevelOp<T>& op) {
  if constexpr (sizeof(T) == 4)
    return op.cd;
  else
    return op.center;
}

}  // namespace

template <class T>
bool stream3d_ok(const LevelOp<T>& op) {
  return s3::enabled() && op.ndim == 3 && op.g.k == 8 && (op.kind == kFine || op.kind == kFine27) &&
         op.g.z0 == 0 && op.g.z1 == op.g.n2 && op.g.n2 > 1 && rec_of(op) != nullptr;
}

template <class T, class Out>
bool launch_stream3d(const LevelOp<T>& op, int mode, T wj, const cplx_t<T>* x, const cplx_t<T>* b, Out* out,
                     cudaStream_t s) {
  using V = cplx_t<T>;
  if (!stream3d_ok(op)) return false;
  const void* rec = rec_of(op);
  if (mode == 2 && !op.inv_diag) return false;
  if constexpr (!std::is_same<Out, V>::value) {
    if (mode != 2) return false;
  }
  auto run = [&](auto kind) {
    constexpr int KIND = decltype(kind)::value;
    if (mode == 2) {
      s3::go<T, V, Out, KIND, 2>(op, x, b, out, rec, wj, s);
      return true;
    }
    if constexpr (std::is_same<Out, V>::value) {
      if (mode == 0) {
        s3::go<T, V, Out, KIND, 0>(op, x, b, out, rec, wj, s);
        return true;
      }
      if (mode == 1) {
        s3::go<T, V, Out, KIND, 1>(op, x, b, out, rec, wj, s);
        return true;
      }
      if constexpr (KIND == kFine) {
        if (mode == 3) {
          s3::go<T, V, Out, KIND, 3>(op, x, b, out, rec, wj, s);
          return true;
        }
      }
    }
    return false;
  };
  const bool ok = op.kind == kFine ? run(std::integral_constant<int, kFine>())
                                   : run(std::integral_constant<int, kFine27>());
  if (ok) HZ_LAUNCH_CHECK();
  return ok;
}

bool launch_stream3d_lo(const LevelOp<double>& op, const float2* x, double2* out, cudaStream_t s) {
  if (!stream3d_ok(op)) return false;
  if (op.kind == kFine)
    s3::go<double, float2, double2, kFine, 0>(op, x, nullptr, out, op.center, 0.0, s);
  else
    s3::go<double, float2, double2, kFine27, 0>(op, x, nullptr, out, op.center, 0.0, s);
  HZ_LAUNCH_CHECK();
  return true;
}

template bool stream3d_ok<float>(const LevelOp<float>&);
template bool stream3d_ok<double>(const LevelOp<double>&);
template bool launch_stream3d<float, float2>(const LevelOp<float>&, int, float, const float2*, const float2*, float2*,
                                             cudaStream_t);
template bool launch_stream3d<float, double2>(const LevelOp<float>&, int, float, const float2*, const float2*,
                                              double2*, cudaStream_t);
template bool launch_stream3d<double, double2>(const LevelOp<double>&, int, double, const double2*, const double2*,
                                               double2*, cudaStream_t);

}  // namespace hz
