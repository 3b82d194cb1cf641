// Plane-streaming kernels of the 3D fine level for 8-column blocks.
//
// apply / residual / damped Jacobi of the 7-point (HelmholtzProblem::apply_block,
// src/helmholtz.cpp:71-100; relax, src/multigrid.cpp:119-136) and of the compact
// 27-point fine operator, over x[node][8]:
//
//  * The grid is cut into (x, y) tiles of TX x TY nodes with all 8 columns;
//    one persistent CTA per SM takes an equal share of the (tile, plane)
//    pairs and walks it as runs of consecutive z planes of one tile. Each
//    plane of the tile is streamed -- the
//    iterate with a one-node halo, the per-node 16-byte operator records with
//    the halo, b and D^-1 of the interior -- into a ring of shared-memory
//    slots with row-wise bulk copies (cp.async.bulk, issued by the lanes of
//    warp 0 three planes ahead) that complete on the slot's mbarrier; the 16
//    warps wait on it, compute, and hand the slot back through a second
//    mbarrier. There is no CTA-wide barrier in the loop and no thread ever
//    waits on a global load.
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
#include <map>
#include <mutex>
#include <type_traits>

#include "kernels.hpp"
#include "profile.hpp"
#include "tma.cuh"

namespace hz {

namespace {

namespace s3 {

#ifndef HZ_S3_LATE
#define HZ_S3_LATE 1
#endif

constexpr int kSlots = 5;   // ring of plane slots
constexpr int kAhead = 3;   // planes in flight ahead of the one being computed
constexpr int kBarBytes = 256;  // mbarriers (128 B), then the 27-point weights

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
  static constexpr int NTHREADS = NCONS;
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
  int tiles_x, tiles_y;
  const unsigned char* zeros;  // >= one iterate row of the tile, all zero
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

// packed FP32 pairs (FFMA2 / FADD2 / FMUL2 on sm_100): one issue slot per
// complex value instead of two; per component the same IEEE operation as the
// scalar form, so results are bitwise those of crfma / cadd / cscale / cfma
__device__ __forceinline__ float2 p_rfma(float s, float2 b, float2 acc) { return __ffma2_rn(make_float2(s, s), b, acc); }
__device__ __forceinline__ double2 p_rfma(double s, double2 b, double2 acc) { return crfma(s, b, acc); }
__device__ __forceinline__ float2 p_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 p_add(double2 a, double2 b) { return cadd(a, b); }
__device__ __forceinline__ float2 p_scale(float s, float2 b) { return __fmul2_rn(make_float2(s, s), b); }
__device__ __forceinline__ double2 p_scale(double s, double2 b) { return cscale(s, b); }
// acc + a * b in cfma's operation order
__device__ __forceinline__ float2 p_cfma(float2 a, float2 b, float2 acc) {
  const float2 t = __ffma2_rn(make_float2(a.x, a.x), b, acc);
  return __ffma2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x), t);
}
__device__ __forceinline__ double2 p_cfma(double2 a, double2 b, double2 acc) { return cfma(a, b, acc); }

// Per-thread pipeline state carried from plane to plane (two copies used in
// alternation, so no register moves between planes)
template <class V, int CPT>
struct Carry {
  V u[CPT];    // the thread's own node of the last plane read
  V bh[CPT];   // b of the plane whose output is pending
  V wd;        // wj D^-1 of that plane
  V s1[CPT], s2[CPT];  // pending output: 7-point partial sum / 27-point same-plane + lower-plane parts
  V p1[CPT], p2[CPT];  // 27-point: the last plane's adjacent-plane parts
  V M;                 // 27-point: the pending row's own mass
};

// MODE 0: out = A x; 1: out = b - A x (Csr order); 2: out = x + wj D^-1 (b - A x);
// 3: out = b - A x with A x in apply_block order (kFine)
template <class T, class XV, class Out, int KIND, int MODE>
__global__ void __launch_bounds__((Cfg<T, XV, MODE>::NTHREADS), 1)
stream3d_kernel(const Args<T, XV, Out> a) {
  using C = Cfg<T, XV, MODE>;
  using V = cplx_t<T>;
  constexpr int CPT = C::CPT, NU = C::NU, TX = C::TX, TY = C::TY, PX = C::PX, PY = C::PY;
  constexpr bool CSR = MODE == 1 || MODE == 2;
  // 27-point Jacobi: the pending row's own x and D^-1 are read back from the
  // previous plane's slot when it is finished (held one step longer, one
  // plane less in flight) instead of being carried in registers
  constexpr bool LATE = KIND == kFine27 && MODE == 2 && HZ_S3_LATE;
  constexpr int AHEAD = LATE ? kAhead - 1 : kAhead;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kSlots;
  unsigned char* slots = smem + kBarBytes;

  const LevelGeom& g = a.op.g;
  const int n0 = int(g.n0), n1 = int(g.n1), n2 = int(g.n2);
  const int tid = int(threadIdx.x), lane = tid & 31;

  if (tid < 8) reinterpret_cast<T*>(smem + 128)[tid] = (tid < 5 ? T(1) : T(0.5)) * a.op.w27[tid];
  if (tid == 0) {
    for (int q = 0; q < kSlots; ++q) {
      tma::mbar_init(&full[q], 1);
      tma::mbar_init(&empty[q], C::NTHREADS / 32);
    }
    tma::fence_mbar_init();
  }
  __syncthreads();

  // This CTA's share of the (tile, plane) pairs, tiles in x-fastest order and
  // each tile's planes consecutive: an equal count per CTA whatever the
  // number of tiles, walked as segments (tile, [zs, ze)) of one tile each.
  const int W = a.tiles_x * a.tiles_y * n2;
  const int w0 = int(int64_t(W) * blockIdx.x / gridDim.x), w1 = int(int64_t(W) * (blockIdx.x + 1) / gridDim.x);

  // ---- producer role: the streamed planes of the segments in order (halo
  // plane below, the segment's planes, halo plane above; planes outside the
  // grid are skipped), the i-th into slot i % kSlots once every warp released
  // the slot's previous plane. The warps take the duty in turn (plane i is
  // issued by warp i mod 16, each lane a few rows), so no warp is slower than
  // the others on average and none is set aside. Every byte of a slot's
  // iterate / record tiles is rewritten per plane: parts of the tile outside
  // the grid are copied from a zero buffer. All threads track the cursor.
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
    if ((tid >> 5) == pi % (C::NTHREADS / 32)) {
      const int ty = ptile / a.tiles_x;
      const int x0 = (ptile - ty * a.tiles_x) * TX, y0 = ty * TY;
      const int p = pp;
      const bool outp = p >= pz0 && p < pz1;
      const int slot = pi % kSlots;
      tma::mbar_wait(&empty[slot], ((pi / kSlots) & 1) ^ 1);
      unsigned char* sl = slots + slot * C::SLOT;
      const int xs = max(x0 - 1, 0), xe = min(x0 + TX, n0 - 1);
      const int cnt = xe - xs + 1, dcol = xs - (x0 - 1), rpad = PX - dcol - cnt;
      const int xin = min(x0 + TX, n0) - x0;
      if (lane == 0) {
        const int rows_i = min(y0 + TY, n1) - y0;
        const uint32_t bytes_i =
            uint32_t(rows_i) * uint32_t(xin) * uint32_t((C::HAS_B ? C::NBV : 0) + (C::HAS_D ? 16 : 0));
        tma::mbar_arrive_expect_tx(&full[slot], uint32_t(PY * PX * (C::NBX + 16)) + (outp ? bytes_i : 0u));
      }
      __syncwarp();
      const unsigned char* zg = a.zeros;
      for (int c = lane; c < 2 * PY + 2 * TY; c += 32) {
        if (c < 2 * PY) {
          const bool isu = c < PY;
          const int ry = isu ? c : c - PY;
          const int y = y0 - 1 + ry;
          const int nb = isu ? C::NBX : 16;  // bytes per node
          unsigned char* dst = sl + (isu ? C::U_OFF : C::REC_OFF) + ry * PX * nb;
          if (y < 0 || y >= n1) {
            tma::bulk_g2s(dst, zg, uint32_t(PX * nb), &full[slot]);
            continue;
          }
          const unsigned char* src = reinterpret_cast<const unsigned char*>(isu ? static_cast<const void*>(a.x) : a.rec) +
                                     ((int64_t(p) * n1 + y) * n0 + xs) * nb;
          if (dcol > 0) tma::bulk_g2s(dst, zg, uint32_t(dcol * nb), &full[slot]);
          tma::bulk_g2s(dst + dcol * nb, src, uint32_t(cnt * nb), &full[slot]);
          if (rpad > 0) tma::bulk_g2s(dst + (dcol + cnt) * nb, zg, uint32_t(rpad * nb), &full[slot]);
        } else {
          if (!outp) continue;
          const bool isb = c < 2 * PY + TY;
          const int by = isb ? c - 2 * PY : c - 2 * PY - TY;
          const int y = y0 + by;
          if (y >= n1) continue;
          const int64_t node = (int64_t(p) * n1 + y) * n0 + x0;
          if (isb) {
            if constexpr (C::HAS_B)
              tma::bulk_g2s(sl + C::B_OFF + by * TX * C::NBV,
                            reinterpret_cast<const unsigned char*>(a.b) + node * C::NBV, uint32_t(xin) * C::NBV,
                            &full[slot]);
          } else {
            if constexpr (C::HAS_D)
              tma::bulk_g2s(sl + C::D_OFF + by * TX * 16,
                            reinterpret_cast<const unsigned char*>(a.op.inv_diag) + node * 16, uint32_t(xin) * 16,
                            &full[slot]);
          }
        }
      }
    }
    ++pi;
    if (++pp > min(pz1, n2 - 1)) {  // next segment
      pw += pz1 - pz0;
      if (pw < w1) pseg();
    }
  };
#pragma unroll 1
  for (int i = 0; i < AHEAD; ++i) issue();

  // ---- consumer role (every warp)
  const int sub = tid % C::TPN, nx = (tid / C::TPN) % TX, ny = tid / (C::TPN * TX);
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
  // of the segment being computed
  int zs = 0, ze = 0;
  bool active = false, xm = false, xp = false, ym = false, yp = false;
  Out* out0 = a.out;
  int ci = 0;  // planes consumed so far
  bool held = false;  // LATE: the last consumed plane's slot is still held
  const T wx = a.op.w[0], wy = a.op.w[1], wz = a.op.w[2];
  // the 27-point weights {lap0..3, mu0, mu1/2, mu2/2, mu3/2} are read from shared memory where they are used
  // (volatile: not hoisted back into eight live registers of a kernel that is short of them)
  const volatile T* wsm = reinterpret_cast<const volatile T*>(smem + 128);
  constexpr int kL0 = 0, kL1 = 1, kL2 = 2, kL3 = 3, kM0 = 4, kH1 = 5, kH2 = 6, kH3 = 7;

  using St = Carry<V, CPT>;
  auto finish = [&](int p, const St& in, const V* ax) {  // output of plane p from A x
    V o[CPT];
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      if (MODE == 0)
        o[q] = ax[q];
      else if (MODE == 1 || MODE == 3)
        o[q] = csub(in.bh[q], ax[q]);
      else if (KIND == kFine)
        o[q] = cadd(in.u[q], cmul(in.wd, csub(in.bh[q], ax[q])));
      else
        o[q] = jacobi_upd(in.u[q], in.wd, in.bh[q], ax[q]);
    }
    stg_cols<V, XV, Out, NU>(out0 + int64_t(p) * pstride * 8, uo, o);
  };
  // 27-point, MODE != 0: b is folded into the pending sum when the plane is
  // started (s1 carries A x - b), so it is not held until the plane finishes
  auto finish_nr = [&](int p, const St& in, const V* nr) {
    V o[CPT];
    if constexpr (MODE == 2 && !LATE) {
      const V nwd = mk(-in.wd.x, -in.wd.y);
#pragma unroll
      for (int q = 0; q < CPT; ++q) o[q] = p_cfma(nwd, nr[q], in.u[q]);
    } else if constexpr (MODE == 2) {
      const unsigned char* sl = slots + ((ci + kSlots - 1) % kSlots) * C::SLOT;  // plane p's slot
      V xo[CPT], Mx, d;
      lds_cols<V, XV, NU>(sl + C::U_OFF + cnode * C::NBX, uo, xo);
      rec_load<T>(sl + C::REC_OFF + cnode * 16, Mx, d);
      if constexpr (C::HAS_D) d = *reinterpret_cast<const V*>(sl + C::D_OFF + inode * 16);
      const V nwd = mk(-a.wj * d.x, -a.wj * d.y);
#pragma unroll
      for (int q = 0; q < CPT; ++q) o[q] = p_cfma(nwd, nr[q], xo[q]);
    } else {
#pragma unroll
      for (int q = 0; q < CPT; ++q) o[q] = mk(-nr[q].x, -nr[q].y);
    }
    stg_cols<V, XV, Out, NU>(out0 + int64_t(p) * pstride * 8, uo, o);
  };
  auto hold = [&](const unsigned char* sl, V dsm, St& out) {  // b and wj D^-1 of the plane being started
    if constexpr (C::HAS_B) lds_cols<V, V, NU>(sl + C::B_OFF + inode * C::NBV, uo, out.bh);
    if constexpr (MODE == 2) {
      V d = dsm;
      if constexpr (C::HAS_D) d = *reinterpret_cast<const V*>(sl + C::D_OFF + inode * 16);
      out.wd = mk(a.wj * d.x, a.wj * d.y);
    }
  };

  // one plane: finish the pending output of plane p - 1 with this plane's
  // contribution and start the output of plane p
  auto step = [&](int p, const St& in, St& out) {
    const bool inside = p >= 0 && p < n2;
    const int slot = ci % kSlots;
    const unsigned char* sl = slots + slot * C::SLOT;
    if (inside) {
      issue();
      tma::mbar_wait(&full[slot], (ci / kSlots) & 1);
    }
    if (active) {
      const unsigned char* un_p = sl + C::U_OFF + cnode * C::NBX;
      const unsigned char* rc_p = sl + C::REC_OFF + cnode * 16;
      if (inside) {
        lds_cols<V, XV, NU>(un_p, uo, out.u);
      } else {
#pragma unroll
        for (int q = 0; q < CPT; ++q) out.u[q] = czero<V>();
      }
      if constexpr (KIND == kFine) {
        if (p - 1 >= zs) {
          V ax[CPT];
#pragma unroll
          for (int q = 0; q < CPT; ++q) ax[q] = inside ? p_rfma(wz, out.u[q], in.s1[q]) : in.s1[q];
          finish(p - 1, in, ax);
        }
        if (p >= zs && p < ze) {
          V uxm[CPT], uxp[CPT], uym[CPT], uyp[CPT], c, d;
          lds_cols<V, XV, NU>(un_p - C::NBX, uo, uxm);
          lds_cols<V, XV, NU>(un_p + C::NBX, uo, uxp);
          lds_cols<V, XV, NU>(un_p - PX * C::NBX, uo, uym);
          lds_cols<V, XV, NU>(un_p + PX * C::NBX, uo, uyp);
          rec_load<T>(rc_p, c, d);
          const bool zm = p > 0;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            V s;
            if (!CSR) {
              s = cmul(c, out.u[q]);
              if (xm) s = p_rfma(wx, uxm[q], s);
              if (xp) s = p_rfma(wx, uxp[q], s);
              if (ym) s = p_rfma(wy, uym[q], s);
              if (yp) s = p_rfma(wy, uyp[q], s);
              if (zm) s = p_rfma(wz, in.u[q], s);
            } else {
              s = czero<V>();
              if (zm) s = p_rfma(wz, in.u[q], s);
              if (ym) s = p_rfma(wy, uym[q], s);
              if (xm) s = p_rfma(wx, uxm[q], s);
              s = p_cfma(c, out.u[q], s);
              if (xp) s = p_rfma(wx, uxp[q], s);
              if (yp) s = p_rfma(wy, uyp[q], s);
            }
            out.s1[q] = s;
          }
          hold(sl, d, out);
        }
      } else {
        // compact 27-point operator: channel 1 = lap . u + (mu / 2) . (M u),
        // channel 2 = (mu / 2) . u (times the row's own M at the end)
        V Mn = czero<V>(), dn = czero<V>();
        if (inside) {
          rec_load<T>(rc_p, Mn, dn);
          // the thread's own node: s = same-plane parts on top of the lower plane's, p = adjacent-plane parts
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const V v0 = cmul(Mn, out.u[q]);
            out.s1[q] = p_rfma(T(wsm[kM0]), v0, p_rfma(T(wsm[kL0]), out.u[q], in.p1[q]));
            out.s2[q] = in.p2[q];
            const T h1 = wsm[kH1];
            out.p1[q] = p_rfma(h1, v0, p_scale(T(wsm[kL1]), out.u[q]));
            out.p2[q] = p_scale(h1, out.u[q]);
          }
          // in-plane faces, then corners: Q(u) and Q(M u) folded into the channels
#pragma unroll
          for (int cls = 1; cls <= 2; ++cls) {
            V qu[CPT], qa[CPT], qb[CPT];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
              const int dx = cls == 1 ? (nb == 0 ? -1 : nb == 1 ? 1 : 0) : (nb & 1 ? 1 : -1);
              const int dy = cls == 1 ? (nb == 2 ? -1 : nb == 3 ? 1 : 0) : (nb & 2 ? 1 : -1);
              V w[CPT];
              lds_cols<V, XV, NU>(un_p + (dy * PX + dx) * C::NBX, uo, w);
              const V Mj = rec_first<T>(rc_p + (dy * PX + dx) * 16);
#pragma unroll
              for (int q = 0; q < CPT; ++q) {
                // M_j w accumulated as Re(M_j) w and Im(M_j) w (combined below)
                if (nb == 0) {
                  qu[q] = w[q];
                  qa[q] = p_scale(Mj.x, w[q]);
                  qb[q] = p_scale(Mj.y, w[q]);
                } else {
                  qu[q] = p_add(qu[q], w[q]);
                  qa[q] = p_rfma(Mj.x, w[q], qa[q]);
                  qb[q] = p_rfma(Mj.y, w[q], qb[q]);
                }
              }
            }
            const T la = wsm[cls == 1 ? kL1 : kL2], ha = wsm[cls == 1 ? kH1 : kH2];  // same plane
            const T lb = wsm[cls == 1 ? kL2 : kL3], hb = wsm[cls == 1 ? kH2 : kH3];  // adjacent planes
#pragma unroll
            for (int q = 0; q < CPT; ++q) {
              const V qv = mk(qa[q].x - qb[q].y, qa[q].y + qb[q].x);
              out.s1[q] = p_rfma(ha, qv, p_rfma(la, qu[q], out.s1[q]));
              out.s2[q] = p_rfma(ha, qu[q], out.s2[q]);
              out.p1[q] = p_rfma(hb, qv, p_rfma(lb, qu[q], out.p1[q]));
              out.p2[q] = p_rfma(hb, qu[q], out.p2[q]);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < CPT; ++q) out.p1[q] = out.p2[q] = out.s1[q] = out.s2[q] = czero<V>();
        }
        if (p - 1 >= zs) {
          V ax[CPT];
#pragma unroll
          for (int q = 0; q < CPT; ++q)
            ax[q] = p_cfma(in.M, p_add(in.s2[q], out.p2[q]), p_add(in.s1[q], out.p1[q]));
          if constexpr (MODE == 0)
            finish(p - 1, in, ax);
          else
            finish_nr(p - 1, in, ax);
        }
        if (p >= zs && p < ze) {
          out.M = Mn;
          if constexpr (C::HAS_B) {
            V bv[CPT];
            lds_cols<V, V, NU>(sl + C::B_OFF + inode * C::NBV, uo, bv);
#pragma unroll
            for (int q = 0; q < CPT; ++q) out.s1[q] = csub(out.s1[q], bv[q]);
          }
          if constexpr (MODE == 2 && !LATE) {
            V d = dn;
            if constexpr (C::HAS_D) d = *reinterpret_cast<const V*>(sl + C::D_OFF + inode * 16);
            out.wd = mk(a.wj * d.x, a.wj * d.y);
          }
        }
      }
    }
    if (inside) {
      __syncwarp();
      if constexpr (LATE) {
        if (lane == 0 && held) tma::mbar_arrive(&empty[(ci + kSlots - 1) % kSlots]);
        held = true;
      } else {
        if (lane == 0) tma::mbar_arrive(&empty[slot]);
      }
      ++ci;
    }
  };

  St A, B;
#pragma unroll
  for (int q = 0; q < CPT; ++q) A.u[q] = A.bh[q] = A.s1[q] = A.s2[q] = A.p1[q] = A.p2[q] = czero<V>();
  A.wd = A.M = czero<V>();
  B = A;
#pragma unroll 1
  for (int w = w0; w < w1; w += ze - zs) {
    const int tile = w / n2;
    const int ty = tile / a.tiles_x;
    const int gx = (tile - ty * a.tiles_x) * TX + nx, gy = ty * TY + ny;
    zs = w - tile * n2;
    ze = min(n2, zs + (w1 - w));
    active = gx < n0 && gy < n1;
    xm = gx > 0, xp = gx + 1 < n0, ym = gy > 0, yp = gy + 1 < n1;
    out0 = a.out + (int64_t(gy) * n0 + gx) * 8;
    // whatever the carry holds from the previous segment only reaches outputs that are never written
#pragma unroll 1
    for (int p = zs - 1; p <= ze; p += 2) {
      step(p, A, B);
      if (p + 1 <= ze) step(p + 1, B, A);
    }
    if constexpr (LATE) {
      __syncwarp();
      if (lane == 0 && held) tma::mbar_arrive(&empty[(ci + kSlots - 1) % kSlots]);
      held = false;
    }
  }
}

// HZ_STREAM3D: 0 = off; 1 (default) = the 27-point operator; 2 = the 7-point
// operator too. The 7-point element kernels (stencil.cu) already run at 0.7 of
// HBM and measure equal or faster (config 4: sweep 377 vs 394 us, residual 363
// vs 397, apply 421 vs 490), so the streaming form stays opt-in there.
int level() {
  static const int v = [] {
    const char* e = std::getenv("HZ_STREAM3D");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

__device__ uint4 g_zeros[320];  // 5 KB >= (TX + 2) nodes of an iterate row

// the current device's zero buffer (looked up once per device)
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

template <class T, class XV, class Out, int KIND, int MODE>
void go(const LevelOp<T>& op, const XV* x, const cplx_t<T>* b, Out* out, const void* rec, T wj, cudaStream_t s) {
  using C = Cfg<T, XV, MODE>;
  static_assert(C::PX * C::NBX <= int(sizeof(uint4)) * 320, "zero row");
  Args<T, XV, Out> a;
  a.op = op;
  a.x = x;
  a.b = b;
  a.out = out;
  a.rec = rec;
  a.wj = wj;
  a.tiles_x = (int(op.g.n0) + C::TX - 1) / C::TX;
  a.tiles_y = (int(op.g.n1) + C::TY - 1) / C::TY;
  a.zeros = zeros_ptr();
  // one persistent CTA per SM, each with an equal share of the (tile, plane)
  // pairs; small grids: at least 8 planes per CTA (HZ_STREAM3D_CTAS forces)
  static const int forced = [] {
    const char* e = std::getenv("HZ_STREAM3D_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t W = int64_t(a.tiles_x) * a.tiles_y * op.g.n2;
  int ctas = int(std::min<int64_t>(kNumSMs, std::max<int64_t>(1, W / 8)));
  if (forced > 0) ctas = int(std::min<int64_t>(forced, W));
  auto kern = stream3d_kernel<T, XV, Out, KIND, MODE>;
  allow_dyn_smem(reinterpret_cast<const void*>(kern), C::SMEM);
  kern<<<ctas, C::NTHREADS, C::SMEM, s>>>(a);
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
  return ((op.kind == kFine27 && s3::level() >= 1) || (op.kind == kFine && s3::level() >= 2)) && op.ndim == 3 &&
         op.g.k == 8 &&
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
