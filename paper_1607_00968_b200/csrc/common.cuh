// Shared device/host helpers for the B200 multi-RHS Helmholtz solver.
//
// Complex values are stored as interleaved (re, im) pairs -- double2 for
// complex128, float2 for complex64 -- which is bit-compatible with the
// reference's std::complex<double> (inc/block.hpp:13-27) and lets every load
// be one 128-bit (c128) or 64-bit (c64) transaction.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <stdexcept>
#include <string>

namespace hz {

// ---------------------------------------------------------------- errors
// Status codes of the C ABI; the exception classes carry them
// through the host driver to hz_* entry points.
enum Status : int {
  kOk = 0,
  kValidation = 1,
  kConvergence = 2,
  kBreakdown = 3,
  kFactorization = 4,
  kState = 5,
  kIo = 6,
  kCuda = 7,
  kNccl = 8,
};

struct HzError : std::runtime_error {
  int code;
  HzError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw HzError(kCuda, std::string("CUDA error in ") + what + " (" + file + ":" +
                             std::to_string(line) + "): " + cudaGetErrorString(e));
}
// process-wide count of this library's kernel launches (bench.py reports it)
void count_launch();
void add_launches(int64_t n);
void set_capturing(bool on);  // this thread is capturing a CUDA graph
bool is_capturing();
#define HZ_CUDA(x) ::hz::cuda_check((x), #x, __FILE__, __LINE__)
#define HZ_LAUNCH_CHECK()                                                              \
  do {                                                                                 \
    ::hz::count_launch();                                                              \
    ::hz::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);         \
  } while (0)

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
// current device. Monotonic and serialised: concurrent solves (RHS groups,
// frequencies) launching the same kernel with different sizes never lower
// the limit under one another's launch; per device, so slab parts on other
// GPUs get it too.
inline void allow_dyn_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[{kern, dev}];
  if (cur >= bytes) return;
  HZ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cur = bytes;
}

// ---------------------------------------------------------------- complex
template <class T> struct CT;
template <> struct CT<double> { using type = double2; };
template <> struct CT<float> { using type = float2; };
template <class T> using cplx_t = typename CT<T>::type;

template <class V> struct RealOf;
template <> struct RealOf<double2> { using type = double; };
template <> struct RealOf<float2> { using type = float; };

__host__ __device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
__host__ __device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
template <class V> __host__ __device__ __forceinline__ V czero() {
  V z;
  z.x = 0;
  z.y = 0;
  return z;
}

template <class V> __host__ __device__ __forceinline__ V cadd(V a, V b) {
  V r;
  r.x = a.x + b.x;
  r.y = a.y + b.y;
  return r;
}
template <class V> __host__ __device__ __forceinline__ V csub(V a, V b) {
  V r;
  r.x = a.x - b.x;
  r.y = a.y - b.y;
  return r;
}
// a * b
template <class V> __host__ __device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
// conj(a) * b
template <class V> __host__ __device__ __forceinline__ V cmulc(V a, V b) {
  V r;
  r.x = a.x * b.x + a.y * b.y;
  r.y = a.x * b.y - a.y * b.x;
  return r;
}
// acc + a * b
template <class V> __host__ __device__ __forceinline__ V cfma(V a, V b, V acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a) * b
template <class V> __host__ __device__ __forceinline__ V cfmac(V a, V b, V acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc + s * b (s real)
template <class V, class T> __host__ __device__ __forceinline__ V crfma(T s, V b, V acc) {
  acc.x = fma(s, b.x, acc.x);
  acc.y = fma(s, b.y, acc.y);
  return acc;
}
template <class V, class T> __host__ __device__ __forceinline__ V cscale(T s, V b) {
  V r;
  r.x = s * b.x;
  r.y = s * b.y;
  return r;
}
// complex64 on the device: packed FP32 pairs (FFMA2 / FADD2 / FMUL2 on sm_100),
// one issue slot per complex value instead of two. Per component these are the
// IEEE operations of the generic forms above in the same order, so the bits
// are the same. HZ_NO_PACKED_F32 (compile time) keeps the scalar forms.
#if defined(__CUDA_ARCH__) && !defined(HZ_NO_PACKED_F32)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 crfma(float s, float2 b, float2 acc) {
  return __ffma2_rn(make_float2(s, s), b, acc);
}
__device__ __forceinline__ float2 cscale(float s, float2 b) { return __fmul2_rn(make_float2(s, s), b); }
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  const float2 t = __ffma2_rn(make_float2(a.x, a.x), b, acc);
  return __ffma2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x), t);
}
#endif

template <class V> __host__ __device__ __forceinline__ typename RealOf<V>::type cabs2(V a) {
  return a.x * a.x + a.y * a.y;
}

// damped-Jacobi update x + d (b - a) with every operation rounded as written
// (no FMA contraction): the Galerkin-level kernels (plain, 4-column,
// bulk-copy) then produce the same bits whatever nvcc would fuse in each
__device__ __forceinline__ float2 jacobi_upd(float2 x, float2 d, float2 b, float2 a) {
  const float sx = __fsub_rn(b.x, a.x), sy = __fsub_rn(b.y, a.y);
  const float mx = __fsub_rn(__fmul_rn(d.x, sx), __fmul_rn(d.y, sy));
  const float my = __fadd_rn(__fmul_rn(d.x, sy), __fmul_rn(d.y, sx));
  return make_float2(__fadd_rn(x.x, mx), __fadd_rn(x.y, my));
}
__device__ __forceinline__ double2 jacobi_upd(double2 x, double2 d, double2 b, double2 a) {
  const double sx = __dsub_rn(b.x, a.x), sy = __dsub_rn(b.y, a.y);
  const double mx = __dsub_rn(__dmul_rn(d.x, sx), __dmul_rn(d.y, sy));
  const double my = __dadd_rn(__dmul_rn(d.x, sy), __dmul_rn(d.y, sx));
  return make_double2(__dadd_rn(x.x, mx), __dadd_rn(x.y, my));
}

template <class Dst, class Src> __host__ __device__ __forceinline__ Dst ccast(Src s) {
  Dst d;
  d.x = static_cast<decltype(d.x)>(s.x);
  d.y = static_cast<decltype(d.y)>(s.y);
  return d;
}

// ---------------------------------------------------------------- indexing
// Division by a runtime constant via multiply-high (Granlund-Montgomery),
// for 32-bit unsigned operands: node index -> (i, j, k) without IDIV.
struct FastDiv {
  uint32_t d = 1, mul = 0, shr = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d == 1) {
      mul = 0;
      shr = 0;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    shr = l - 1;
    mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
#ifdef __CUDA_ARCH__
    uint32_t t = __umulhi(n, mul);
#else
    uint32_t t = static_cast<uint32_t>((static_cast<uint64_t>(n) * mul) >> 32);
#endif
    return (t + ((n - t) >> 1)) >> shr;
  }
  __host__ __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// Structured grid of one multigrid level: node counts per axis (axis 0
// fastest, inc/grid.hpp:23-40) plus the RHS block width k.
struct LevelGeom {
  uint32_t n0 = 1, n1 = 1, n2 = 1;
  uint32_t nodes = 1;
  uint32_t k = 1;
  // planes [z0, z1) of the slow axis (axis 2, or axis 1 of a 2D grid) this
  // launch computes: a slab of the grid; neighbours outside it are still
  // read, through the global layout
  uint32_t z0 = 0, z1 = 1;
  FastDiv div_k, div_n0, div_n1;
  LevelGeom() = default;
  LevelGeom(int64_t a, int64_t b, int64_t c, int kk)
      : n0(uint32_t(a)), n1(uint32_t(b)), n2(uint32_t(c)), nodes(uint32_t(a * b * c)), k(uint32_t(kk)),
        z1(uint32_t(c > 1 ? c : b)), div_k(uint32_t(kk)), div_n0(uint32_t(a)), div_n1(uint32_t(b)) {}
  LevelGeom slab(int64_t za, int64_t zb) const {
    LevelGeom g = *this;
    g.z0 = uint32_t(za);
    g.z1 = uint32_t(zb);
    return g;
  }
  __host__ __device__ __forceinline__ uint32_t plane_elems() const { return (n2 > 1 ? n0 * n1 : n0) * k; }
  __host__ __device__ __forceinline__ uint32_t e_begin() const { return z0 * plane_elems(); }
  __host__ __device__ __forceinline__ uint32_t e_end() const { return z1 * plane_elems(); }
  int64_t owned_elems() const { return int64_t(z1 - z0) * plane_elems(); }
  int64_t owned_nodes() const { return int64_t(z1 - z0) * (n2 > 1 ? n0 * n1 : n0); }
  __host__ __device__ __forceinline__ void unpack(uint32_t node, uint32_t& i, uint32_t& j,
                                                  uint32_t& kz) const {
    uint32_t r;
    div_n0.divmod(node, r, i);
    div_n1.divmod(r, kz, j);
  }
};

constexpr int kNumSMs = 148;

inline int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace hz
