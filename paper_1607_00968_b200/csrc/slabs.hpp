// Slab decomposition of the slow grid axis over several "parts" -- one per
// GPU, or several on one GPU.
//
// B200 design: vectors keep the global node-major [node][k] layout in ONE
// virtual address range whose pages for part p's planes are physically on
// part p's GPU (CUDA virtual memory management), mapped read/write for every
// participating GPU. A stencil / restriction / prolongation kernel of part p
// computes only its own planes, and reads the one neighbour plane it needs
// across a slab face straight out of the peer GPU's HBM over NVLink/NVSwitch:
// the per-level halo exchange is fused into the kernels themselves, with no
// staging copy and no separate exchange launch. Streams of neighbouring parts
// are ordered by events (one exchange step per stencil); the
// k x k Gram/norm partials of the Krylov method are summed on part 0 in a
// fixed slot order, so the reduction is deterministic for any part count.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "devbuf.hpp"

namespace hz {

struct SlabPart {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev = nullptr;
  bool own_stream = false;
};

class Slabs {
 public:
  // devices[p] = GPU of part p; root_stream becomes part 0's stream.
  // level_dims: the hierarchy's per-level grids (slow axis = axis 2, or
  // axis 1 for 2D grids).
  Slabs(const std::vector<int>& devices, const std::vector<std::array<int64_t, 3>>& level_dims, int ndim,
        cudaStream_t root_stream);
  ~Slabs();
  Slabs(const Slabs&) = delete;
  Slabs& operator=(const Slabs&) = delete;

  int parts() const { return int(part_.size()); }
  const SlabPart& part(int p) const { return part_[p]; }
  cudaStream_t root() const { return part_[0].stream; }
  bool multi_device() const { return multi_device_; }
  // spanning vectors built from per-part VMM chunks (multi-GPU, or forced by HZ_SLAB_VMM=1)
  bool spanning_vmm() const;
  int levels() const { return int(cut_.size()); }
  int slow_axis() const { return slow_; }
  // first level handled by part 0 alone (coarse agglomeration): the first
  // level on which some part would own fewer than 2 planes
  int agg_level() const { return agg_; }
  // planes [z0, z1) of part p on level l (slow axis)
  int64_t z0(int l, int p) const { return cut_[l][p]; }
  int64_t z1(int l, int p) const { return cut_[l][p + 1]; }
  // rows (nodes) of part p on level l
  int64_t row0(int l, int p) const { return cut_[l][p] * plane_[l]; }
  int64_t row1(int l, int p) const { return cut_[l][p + 1] * plane_[l]; }
  int64_t rows(int l) const { return cut_[l].back() * plane_[l]; }

  // ---- stream ordering between parts
  // every part waits for the work already enqueued by its slab neighbours
  void neighbours() const;
  // part 0 waits for every part
  void join() const;
  // every part waits for part 0
  void fork() const;

  // ---- storage: a level-l block vector of `row_bytes` per node whose pages
  // follow the slabs (single cudaMalloc when every part is on one GPU)
  std::shared_ptr<void> alloc(int l, size_t row_bytes) const;

  template <class F>
  void each(int l, F&& f) const {
    for (int p = 0; p < parts(); ++p) {
      DeviceGuard g(part_[p].device);
      f(p, row0(l, p), row1(l, p) - row0(l, p), part_[p].stream);
    }
  }

 private:
  void record(int p) const;
  std::vector<SlabPart> part_;
  std::vector<std::vector<int64_t>> cut_;  // [level][parts + 1]
  std::vector<int64_t> plane_;             // nodes per slow-axis plane, per level
  int slow_ = 2;
  int agg_ = 0;
  bool multi_device_ = false;
};

// Spanning allocation helper for DevBuf (see Slabs::alloc).
template <class E>
void alloc_span(DevBuf<E>& b, const Slabs& sl, int l, int k) {
  b.release();  // free first: these blocks are large and HBM may be nearly full
  b.adopt(sl.alloc(l, sizeof(E) * size_t(k)), size_t(sl.rows(l)) * k);
}

// cuMemCreate chunks made for spanning vectors so far (diagnostic)
int64_t vmm_chunks_created();

}  // namespace hz
