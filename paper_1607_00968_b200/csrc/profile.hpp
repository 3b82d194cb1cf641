// Optional per-kernel CUDA-event profiling of the library's own launches.
// When enabled (hz_profile_begin), every launch wrapper brackets its kernel
// with events on the stream it launches on and records the kernel's
// ALGORITHMIC bytes (the SURVEY §8d formulas), so bench.py can report
// achieved GB/s per kernel class against the HBM roofline.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace hz {

bool profiling_enabled();
bool is_capturing();  // common.cuh: this thread is capturing a CUDA graph (no event records then)
void profile_record(const char* name, double bytes, double flops, cudaEvent_t a, cudaEvent_t b,
                    cudaStream_t s = nullptr);
cudaEvent_t profile_event();
// interned "<base>_L<level>" (stable pointer for the profile records)
const char* profile_name_level(const char* base, int level);

class ProfScope {
 public:
  ProfScope(const char* name, double bytes, cudaStream_t s, double flops = 0.0)
      : name_(name), bytes_(bytes), flops_(flops), s_(s) {
    if (profiling_enabled() && !is_capturing()) {
      a_ = profile_event();
      b_ = profile_event();
      cudaEventRecord(a_, s_);
    }
  }
  ~ProfScope() {
    if (a_) {
      cudaEventRecord(b_, s_);
      profile_record(name_, bytes_, flops_, a_, b_, s_);
    }
  }

 private:
  const char* name_;
  double bytes_, flops_;
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

}  // namespace hz
