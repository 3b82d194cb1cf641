// Slab decomposition: plane cuts per level, inter-part stream ordering and
// slab-spanning (multi-GPU) vector storage. See slabs.hpp.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <string>

#include <atomic>
#include <cstdlib>

#include "slabs.hpp"

namespace hz {

namespace {

struct Vmm {
  PFN_cuMemGetAllocationGranularity gran = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemSetAccess access = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemRelease release = nullptr;
  PFN_cuMemAddressFree free = nullptr;
};

template <class F>
void load(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  HZ_CUDA(cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q));
  if (!p || q != cudaDriverEntryPointSuccess)
    throw HzError(kCuda, std::string("driver entry point unavailable: ") + name);
  fn = reinterpret_cast<F>(p);
}

const Vmm& vmm() {
  static const Vmm v = [] {
    Vmm t;
    load("cuMemGetAllocationGranularity", t.gran);
    load("cuMemCreate", t.create);
    load("cuMemAddressReserve", t.reserve);
    load("cuMemMap", t.map);
    load("cuMemSetAccess", t.access);
    load("cuMemUnmap", t.unmap);
    load("cuMemRelease", t.release);
    load("cuMemAddressFree", t.free);
    return t;
  }();
  return v;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw HzError(kCuda, std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}

}  // namespace

Slabs::Slabs(const std::vector<int>& devices, const std::vector<std::array<int64_t, 3>>& level_dims, int ndim,
             cudaStream_t root_stream) {
  const int P = int(devices.size());
  if (P < 1) throw HzError(kValidation, "slabs: need at least one part");
  if (level_dims.empty()) throw HzError(kValidation, "slabs: empty hierarchy");
  slow_ = ndim == 3 ? 2 : 1;
  const int L = int(level_dims.size());
  const int64_t n0 = level_dims[0][slow_];
  if (n0 < 2 * P) throw HzError(kValidation, "slabs: fewer than 2 planes per part on the fine grid");
  // level-0 cuts on multiples of 2^(L-1) planes, so every level's cut is the
  // exact image of the fine one (cut_l = cut_0 >> l)
  const int64_t unit = int64_t(1) << (L - 1);
  const int64_t m = std::max<int64_t>((n0 - 1) / unit, 1);
  std::vector<int64_t> c0(P + 1);
  for (int p = 0; p < P; ++p) c0[p] = unit * ((int64_t(p) * m + P / 2) / P);
  c0[P] = n0;
  cut_.assign(L, std::vector<int64_t>(P + 1));
  plane_.resize(L);
  agg_ = L - 1;
  for (int l = 0; l < L; ++l) {
    const int64_t nl = level_dims[l][slow_];
    plane_[l] = slow_ == 2 ? level_dims[l][0] * level_dims[l][1] : level_dims[l][0];
    for (int p = 0; p < P; ++p) cut_[l][p] = std::min<int64_t>(c0[p] >> l, nl);
    cut_[l][P] = nl;
    bool thin = false;
    for (int p = 0; p < P; ++p) thin = thin || cut_[l][p + 1] - cut_[l][p] < 2;
    if (l == 0 && thin) throw HzError(kValidation, "slabs: a part owns fewer than 2 fine planes");
    if (thin && l < agg_) agg_ = l;
  }
  if (L == 1) agg_ = 0;
  part_.resize(P);
  for (int p = 0; p < P; ++p) {
    part_[p].device = devices[p];
    if (devices[p] != devices[0]) multi_device_ = true;
  }
  for (int p = 0; p < P; ++p) {
    DeviceGuard g(devices[p]);
    if (p == 0) {
      part_[p].stream = root_stream;
    } else {
      HZ_CUDA(cudaStreamCreateWithFlags(&part_[p].stream, cudaStreamNonBlocking));
      part_[p].own_stream = true;
    }
    HZ_CUDA(cudaEventCreateWithFlags(&part_[p].ev, cudaEventDisableTiming));
  }
  if (multi_device_) {
    // peer access for the small k x k operands kept on part 0 and for the
    // neighbour planes of the spanning vectors
    for (int a : devices)
      for (int b : devices) {
        if (a == b) continue;
        int can = 0;
        HZ_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
        if (!can) throw HzError(kCuda, "slabs: GPUs " + std::to_string(a) + " and " + std::to_string(b) +
                                           " have no peer access");
        DeviceGuard g(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
          cudaGetLastError();
        else
          HZ_CUDA(e);
      }
  }
}

Slabs::~Slabs() {
  for (auto& p : part_) {
    DeviceGuard g(p.device);
    if (p.ev) cudaEventDestroy(p.ev);
    if (p.own_stream && p.stream) cudaStreamDestroy(p.stream);
  }
}

void Slabs::record(int p) const {
  DeviceGuard g(part_[p].device);
  HZ_CUDA(cudaEventRecord(part_[p].ev, part_[p].stream));
}

void Slabs::neighbours() const {
  const int P = parts();
  if (P == 1) return;
  for (int p = 0; p < P; ++p) record(p);
  for (int p = 0; p < P; ++p) {
    DeviceGuard g(part_[p].device);
    if (p > 0) HZ_CUDA(cudaStreamWaitEvent(part_[p].stream, part_[p - 1].ev, 0));
    if (p + 1 < P) HZ_CUDA(cudaStreamWaitEvent(part_[p].stream, part_[p + 1].ev, 0));
  }
}

void Slabs::join() const {
  const int P = parts();
  if (P == 1) return;
  for (int p = 1; p < P; ++p) record(p);
  DeviceGuard g(part_[0].device);
  for (int p = 1; p < P; ++p) HZ_CUDA(cudaStreamWaitEvent(part_[0].stream, part_[p].ev, 0));
}

void Slabs::fork() const {
  const int P = parts();
  if (P == 1) return;
  record(0);
  for (int p = 1; p < P; ++p) {
    DeviceGuard g(part_[p].device);
    HZ_CUDA(cudaStreamWaitEvent(part_[p].stream, part_[0].ev, 0));
  }
}

// HZ_SLAB_VMM=1 builds the spanning vectors from one cuMemCreate chunk per
// part mapped into one reservation even when all parts share one GPU, so the
// multi-GPU allocation path (chunk cuts at the page granularity, mapping,
// access rights) runs and is tested on a single device.
static bool force_vmm() {
  static const bool on = [] {
    const char* e = std::getenv("HZ_SLAB_VMM");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool Slabs::spanning_vmm() const { return multi_device_ || force_vmm(); }

static std::atomic<int64_t> g_vmm_chunks{0};
int64_t vmm_chunks_created() { return g_vmm_chunks.load(); }

std::shared_ptr<void> Slabs::alloc(int l, size_t row_bytes) const {
  const size_t bytes = size_t(rows(l)) * row_bytes;
  if (!spanning_vmm()) {
    const int dev = part_[0].device;
    DeviceGuard g(dev);
    void* p = nullptr;
    HZ_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 1)));
    return std::shared_ptr<void>(p, [dev](void* q) {
      DeviceGuard g2(dev);
      cudaFree(q);
    });
  }
  const Vmm& v = vmm();
  const int P = parts();
  size_t gran = 0;
  for (int p = 0; p < P; ++p) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = part_[p].device;
    size_t g = 0;
    cu_check(v.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    gran = std::max(gran, g);
  }
  const size_t total = (std::max<size_t>(bytes, 1) + gran - 1) / gran * gran;
  // chunk boundaries: each part's first byte rounded to the page granularity
  std::vector<size_t> b(P + 1);
  b[0] = 0;
  b[P] = total;
  for (int p = 1; p < P; ++p) {
    const size_t at = size_t(row0(l, p)) * row_bytes;
    b[p] = std::min(total, std::max(b[p - 1], (at + gran / 2) / gran * gran));
  }
  struct Span {
    CUdeviceptr va = 0;
    size_t total = 0;
    std::vector<std::pair<CUdeviceptr, size_t>> maps;
    std::vector<CUmemGenericAllocationHandle> handles;
  };
  auto* sp = new Span;
  sp->total = total;
  auto cleanup = [](Span* s) {
    const Vmm& vv = vmm();
    for (auto& m : s->maps) vv.unmap(m.first, m.second);
    for (auto h : s->handles) vv.release(h);
    if (s->va) vv.free(s->va, s->total);
    delete s;
  };
  try {
    cu_check(v.reserve(&sp->va, total, gran, 0, 0), "cuMemAddressReserve");
    for (int p = 0; p < P; ++p) {
      const size_t sz = b[p + 1] - b[p];
      if (sz == 0) continue;
      CUmemAllocationProp prop{};
      prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      prop.location.id = part_[p].device;
      CUmemGenericAllocationHandle h{};
      cu_check(v.create(&h, sz, &prop, 0), "cuMemCreate");
      g_vmm_chunks.fetch_add(1);
      sp->handles.push_back(h);
      cu_check(v.map(sp->va + b[p], sz, 0, h, 0), "cuMemMap");
      sp->maps.push_back({sp->va + b[p], sz});
    }
    std::vector<CUmemAccessDesc> acc;
    std::vector<int> seen;
    for (int p = 0; p < P; ++p) {
      if (std::find(seen.begin(), seen.end(), part_[p].device) != seen.end()) continue;
      seen.push_back(part_[p].device);
      CUmemAccessDesc d{};
      d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      d.location.id = part_[p].device;
      d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      acc.push_back(d);
    }
    cu_check(v.access(sp->va, total, acc.data(), acc.size()), "cuMemSetAccess");
  } catch (...) {
    cleanup(sp);
    throw;
  }
  void* ptr = reinterpret_cast<void*>(sp->va);
  return std::shared_ptr<void>(ptr, [sp, cleanup](void*) { cleanup(sp); });
}

}  // namespace hz
