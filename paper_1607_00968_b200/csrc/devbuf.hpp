// Owning device allocation (RAII). All hot-path storage of the solver lives in
// these: problem coefficients, the multigrid hierarchy, Krylov bases.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <utility>

#include "common.cuh"

namespace hz {

template <class E>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), owner_(std::move(o.owner_)) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      owner_ = std::move(o.owner_);
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    HZ_CUDA(cudaMalloc(&p_, count * sizeof(E)));
    n_ = count;
  }
  // grow-only (keeps the allocation when large enough)
  void ensure(size_t count) {
    if (count > n_) alloc(count);
  }
  // take an allocation owned elsewhere (e.g. a slab-spanning mapping)
  void adopt(std::shared_ptr<void> owner, size_t count) {
    release();
    p_ = static_cast<E*>(owner.get());
    n_ = count;
    owner_ = std::move(owner);
  }
  void release() {
    if (owner_)
      owner_.reset();
    else if (p_)
      cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void zero(cudaStream_t s) {
    if (n_) HZ_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(E), s));
  }
  void upload(const void* host, size_t count, cudaStream_t s) {
    HZ_CUDA(cudaMemcpyAsync(p_, host, count * sizeof(E), cudaMemcpyHostToDevice, s));
  }
  void download(void* host, size_t count, cudaStream_t s) const {
    HZ_CUDA(cudaMemcpyAsync(host, p_, count * sizeof(E), cudaMemcpyDeviceToHost, s));
  }
  E* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(E); }

 private:
  E* p_ = nullptr;
  size_t n_ = 0;
  std::shared_ptr<void> owner_;
};

// Pinned host staging for the small k x k / k-vector results the host driver
// reads back every Krylov iteration (async D2H without a pageable bounce).
template <class E>
class PinnedBuf {
 public:
  PinnedBuf() = default;
  ~PinnedBuf() {
    if (p_) cudaFreeHost(p_);
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  void ensure(size_t count) {
    if (count <= n_) return;
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    HZ_CUDA(cudaMallocHost(&p_, count * sizeof(E)));
    n_ = count;
  }
  E* get() const { return p_; }
  E& operator[](size_t i) { return p_[i]; }
  const E& operator[](size_t i) const { return p_[i]; }
  size_t size() const { return n_; }

 private:
  E* p_ = nullptr;
  size_t n_ = 0;
};

// Make `device` current for the lifetime of the guard.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    HZ_CUDA(cudaGetDevice(&prev));
    if (prev != dev) HZ_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace hz
