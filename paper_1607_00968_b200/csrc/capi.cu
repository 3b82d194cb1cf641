// extern "C" boundary (include/hz_b200.h). Maps the reference's exception
// classes to status codes and owns the device-side state behind the opaque
// hz_problem / hz_solver handles.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <exception>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hz_b200.h"
#include "acquisition.hpp"
#include "solver.hpp"

#include <map>
#include <mutex>
#include <sstream>

#include "profile.hpp"

namespace hz {

static std::atomic<int64_t> g_launches{0};
// kernels enqueued while this thread captures a CUDA graph run only when the
// graph is launched: counted then (add_launches), not at capture
thread_local bool g_capturing = false;
void count_launch() {
  if (!g_capturing) g_launches.fetch_add(1, std::memory_order_relaxed);
}
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_capturing(bool on) { g_capturing = on; }
bool is_capturing() { return g_capturing; }

// ---- per-kernel event profiler (profile.hpp)
namespace {
struct ProfRec {
  const char* name;
  double bytes, flops;
  cudaEvent_t a, b;
  cudaStream_t s;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
// events are created up front (hz_profile_begin) and handed out by an atomic
// index, so concurrent solves do not serialise on the profiler
constexpr size_t kProfPool = size_t(1) << 17;
std::vector<cudaEvent_t> g_prof_pool;
std::atomic<size_t> g_prof_next{0};
std::vector<cudaEvent_t> g_prof_extra;
std::vector<ProfRec> g_prof_recs;
}  // namespace

bool profiling_enabled() { return g_prof_on; }

cudaEvent_t profile_event() {
  const size_t i = g_prof_next.fetch_add(1);
  if (i < g_prof_pool.size()) return g_prof_pool[i];  // never resized while profiling
  // pool exhausted: fresh events kept apart (destroyed at the next begin)
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t e;
  HZ_CUDA(cudaEventCreate(&e));
  g_prof_extra.push_back(e);
  return e;
}

const char* profile_name_level(const char* base, int level) {
  if (!g_prof_on) return base;
  static std::mutex mu;
  static std::map<std::string, std::unique_ptr<std::string>> names;
  std::string key = std::string(base) + "_L" + std::to_string(level);
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = names[key];
  if (!slot) slot = std::make_unique<std::string>(key);
  return slot->c_str();
}

void profile_record(const char* name, double bytes, double flops, cudaEvent_t a, cudaEvent_t b,
                    cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.push_back({name, bytes, flops, a, b, s});
}

}  // namespace hz

using namespace hz;

struct hz_problem {
  std::shared_ptr<Problem> p;
};

struct hz_sampling {
  std::unique_ptr<Sampling> s;
};

// One RHS group of a blocked solve (hz_options.rhs_block): its own stream,
// hierarchy views (shared operators, private cycle workspace), Krylov
// workspace and column-gathered [n][kg] blocks.
struct RhsGroup {
  cudaStream_t stream = nullptr;
  std::unique_ptr<Hierarchy<double>> h64;
  std::unique_ptr<Hierarchy<float>> h32;
  std::unique_ptr<Fgmres<double>> fgm;
  std::unique_ptr<Bicgstab> bicg;
  DevBuf<double2> B, X;
  ~RhsGroup() {
    fgm.reset();
    bicg.reset();
    h32.reset();
    h64.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};

struct hz_solver {
  std::shared_ptr<Problem> prob;
  hz_options opts{};
  CycleSpec spec;
  bool bicgstab = true;
  bool dense = false;
  cudaStream_t stream = nullptr;
  std::unique_ptr<Hierarchy<double>> h64;
  std::unique_ptr<Hierarchy<float>> h32;
  std::unique_ptr<Fgmres<double>> fgm;
  std::unique_ptr<Bicgstab> bicg;
  DevBuf<double2> dB, dX;
  std::vector<std::unique_ptr<RhsGroup>> groups;  // blocked solves (rhs_block > 0)
  // DenseLuSmall: explicit inverse of the unshifted operator
  DevBuf<double2> dense_ainvT;
  // slab decomposition (slabs.hpp): per-GPU copies of the fine centre and of
  // the cycle's hierarchy for parts not on the problem's GPU
  std::unique_ptr<Slabs> slabs;
  std::map<int, std::unique_ptr<Hierarchy<double>>> rep64;
  std::map<int, std::unique_ptr<Hierarchy<float>>> rep32;
  std::map<int, DevBuf<double2>> center_rep;
  // FWI / wavefield-output scratch (grow-only)
  DevBuf<double2> fU, fR, fX, fD;
  DevBuf<double> fv, fpart, fmax;
  DevBuf<uint32_t> fQ;
  int span_k = 0;  // k the spanning dB/dX are laid out for
  const double2* center_on(int device) const {
    if (device == prob->device) return prob->d_center.get();
    return center_rep.at(device).get();
  }
  // (re)lay out the solver-owned level-0 blocks for k columns
  void ensure_blocks(int k) {
    const size_t e = size_t(prob->num_nodes()) * k;
    if (!slabs) {
      dB.ensure(e);
      dX.ensure(e);
      return;
    }
    if (span_k == k) return;
    alloc_span(dB, *slabs, 0, k);
    alloc_span(dX, *slabs, 0, k);
    span_k = k;
  }
  ~hz_solver() {
    groups.clear();  // views of h64 / h32
    fgm.reset();
    h32.reset();
    h64.reset();
    rep32.clear();
    rep64.clear();
    slabs.reset();
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const HzError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return kCuda;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kState;
  }
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw HzError(kCuda, "no CUDA device visible (this library has no CPU fallback)");
}

void check_block(const Problem& p, int64_t n, int k) {
  if (n != p.num_nodes()) throw HzError(kValidation, "helmholtz: block size does not match grid");
  if (k < 1) throw HzError(kValidation, "helmholtz: block needs at least one column");
  if (n * int64_t(k) >= (int64_t(1) << 32))
    throw HzError(kValidation, "helmholtz: n*k too large for one device block");
}

void require_converged(const Report& r, const char* what) {
  for (char c : r.converged)
    if (!c) throw HzError(kConvergence, what);
}

// The solver runs on its own non-blocking stream. Device entry points order
// it after the caller's work on `stream` (nullptr: the legacy default
// stream, which the plain *_device entry points assume), so a block the
// caller wrote asynchronously is complete before the solve reads it.
void order_after_caller(hz_solver* s, void* stream) {
  cudaEvent_t ev = nullptr;
  HZ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  const cudaError_t e1 = cudaEventRecord(ev, stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy);
  const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(s->stream, ev, 0) : e1;
  cudaEventDestroy(ev);
  HZ_CUDA(e2);
}

void fill_report(const Report& r, int k, hz_report* out) {
  if (!out) return;
  out->cycles = r.cycles;
  out->qr_factorizations = r.qr_factorizations;
  out->block_gram_products = r.block_gram_products;
  out->wall_s = r.wall_s;
  out->history_len = int(r.history.size());
  for (int j = 0; j < k; ++j) {
    if (out->col_cycles) out->col_cycles[j] = r.col_cycles[j];
    if (out->rel_residual) out->rel_residual[j] = r.rel_residual[j];
    if (out->converged) out->converged[j] = r.converged[j];
  }
  if (out->history)
    for (int i = 0; i < std::min<int>(out->history_cap, int(r.history.size())); ++i)
      out->history[i] = r.history[i];
}

// Slab mode (hz_solver_set_slabs): the fine operator and the casts run per
// part on the part's planes / rows; the cycle is the hierarchy's slab cycle.
DevOp<double> make_slab_op(hz_solver* s, int k) {
  DevOp<double> op;
  Problem* P = s->prob.get();
  const Slabs* sl = s->slabs.get();
  op.n = P->num_nodes();
  op.apply = [s, P, sl](const double2* in, double2* out, int kk, cudaStream_t) {
    sl->neighbours();
    sl->each(0, [&](int p, int64_t, int64_t, cudaStream_t st) {
      LevelOp<double> o = P->fine_op(kk);
      o.center = s->center_on(sl->part(p).device);
      o.g = o.g.slab(sl->z0(0, p), sl->z1(0, p));
      launch_apply<double>(o, in, out, st);
    });
  };
  op.resid = [s, P, sl](const double2* x, const double2* b, double2* r, int kk, cudaStream_t) {
    sl->neighbours();
    sl->each(0, [&](int p, int64_t, int64_t, cudaStream_t st) {
      LevelOp<double> o = P->fine_op(kk);
      o.center = s->center_on(sl->part(p).device);
      o.g = o.g.slab(sl->z0(0, p), sl->z1(0, p));
      launch_apply_residual<double>(o, x, b, r, st);
    });
  };
  if (s->opts.precond_precision == HZ_C64) {
    op.prec = [s](const double2* in, double2* out, int kk, cudaStream_t st) {
      s->h32->cycle_cast(s->spec, kk, in, out, st);
    };
  } else {
    op.prec = [s](const double2* in, double2* out, int kk, cudaStream_t st) {
      s->h64->cycle(s->spec, kk, in, out, true, st);
    };
  }
  return op;
}

// the unpreconditioned fine operator + the cycle of hierarchy h64 / h32
DevOp<double> make_op_with(hz_solver* s, Hierarchy<double>* h64, Hierarchy<float>* h32) {
  DevOp<double> op;
  Problem* P = s->prob.get();
  op.n = P->num_nodes();
  op.apply = [P](const double2* in, double2* out, int kk, cudaStream_t st) {
    launch_apply<double>(P->fine_op(kk), in, out, st);
  };
  op.resid = [P](const double2* x, const double2* b, double2* r, int kk, cudaStream_t st) {
    launch_apply_residual<double>(P->fine_op(kk), x, b, r, st);
  };
  const CycleSpec* spec = &s->spec;
  if (s->opts.precond_precision == HZ_C64) {
    op.prec = [spec, h32](const double2* in, double2* out, int kk, cudaStream_t st) {
      h32->cycle_cast_graph(*spec, kk, in, out, st);
    };
    {  // complex64 Z blocks: the fine apply widens them on load
      if (P->stencil != 7) op.lo_ok = [P](int kk) { return stream3d_ok(P->fine_op(kk)); };
      op.prec_lo = [spec, h32](const double2* in, float2* out, int kk, cudaStream_t st) {
        h32->cycle_cast_graph(*spec, kk, in, out, st);
      };
      op.apply_lo = [P](const float2* in, double2* out, int kk, cudaStream_t st) {
        launch_apply_lo(P->fine_op(kk), in, out, st);
      };
      if (P->stencil == 7)
        op.apply_lo_gram = [P](const float2* Z, double2* W, const BlockTab<double>& X, int nb, double2* part,
                               int max_slots, cudaStream_t st) {
          return launch_gram8_apply(P->fine_op(8), nb, X, Z, W, part, max_slots, st);
        };
    }
  }
  else
    op.prec = [spec, h64](const double2* in, double2* out, int kk, cudaStream_t st) {
      h64->cycle(*spec, kk, in, out, true, st);
    };
  return op;
}

DevOp<double> make_op(hz_solver* s, int k) {
  if (s->slabs) return make_slab_op(s, k);
  return make_op_with(s, s->h64.get(), s->h32.get());
}

// host <-> solver block copies, one per part (each part's rows live on its GPU)
void upload_rows(hz_solver* s, int k, const double* host, double2* dev) {
  const auto* h = reinterpret_cast<const double2*>(host);
  if (!s->slabs) {
    HZ_CUDA(cudaMemcpyAsync(dev, h, size_t(s->prob->num_nodes()) * k * sizeof(double2), cudaMemcpyHostToDevice,
                            s->stream));
    return;
  }
  s->slabs->each(0, [&](int, int64_t r0, int64_t nr, cudaStream_t st) {
    HZ_CUDA(cudaMemcpyAsync(dev + r0 * k, h + r0 * k, size_t(nr) * k * sizeof(double2), cudaMemcpyHostToDevice, st));
  });
}
void download_rows(hz_solver* s, int k, const double2* dev, double* host) {
  auto* h = reinterpret_cast<double2*>(host);
  if (!s->slabs) {
    HZ_CUDA(cudaMemcpyAsync(h, dev, size_t(s->prob->num_nodes()) * k * sizeof(double2), cudaMemcpyDeviceToHost,
                            s->stream));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    return;
  }
  s->slabs->each(0, [&](int, int64_t r0, int64_t nr, cudaStream_t st) {
    HZ_CUDA(cudaMemcpyAsync(h + r0 * k, dev + r0 * k, size_t(nr) * k * sizeof(double2), cudaMemcpyDeviceToHost, st));
  });
  s->slabs->join();
  HZ_CUDA(cudaStreamSynchronize(s->stream));
}

Report run_grouped(hz_solver* s, int k, const double2* B, double2* X);

Report run_solve(hz_solver* s, int k, const double2* B, double2* X) {
  Report rep;
  if (!s->dense && s->opts.rhs_block > 0 && k > s->opts.rhs_block) return run_grouped(s, k, B, X);
  if (s->dense) {
    // DenseLuSmall (src/helmholtz_solver.cpp:38-59): direct solve, then the
    // reported residuals
    const int64_t n = s->prob->num_nodes();
    DevBuf<double2> part(size_t(std::max(coarse_split(n, k), 1)) * n * k);
    launch_coarse_solve<double>(n, k, s->dense_ainvT.get(), B, X, part.get(), s->stream);
    BlockAlgebra<double> alg;
    alg.ensure(n, k, 1);
    DevBuf<double2> R(size_t(n) * k);
    launch_apply<double>(s->prob->fine_op(k), X, R.get(), s->stream);
    launch_axpby<double>(n * k, mk(-1.0, 0.0), R.get(), mk(1.0, 0.0), B, s->stream);
    std::vector<double> rn, bn;
    alg.col_norms(R.get(), rn, s->stream);
    alg.col_norms(B, bn, s->stream);
    rep.col_cycles.assign(k, 0);
    for (int j = 0; j < k; ++j) {
      const double b = bn[j] > 0 ? bn[j] : 1.0;
      rep.rel_residual.push_back(rn[j] / b);
      rep.converged.push_back(1);
    }
    return rep;
  }
  DevOp<double> op = make_op(s, k);
  if (s->bicgstab) {
    if (!s->bicg) s->bicg = std::make_unique<Bicgstab>();
    return s->bicg->solve(op, k, B, X, s->opts.tol, s->opts.max_cycles, s->stream);
  }
  if (!s->fgm) s->fgm = std::make_unique<Fgmres<double>>();
  return s->fgm->solve(op, k, B, X, s->opts.fgmres_restart, s->opts.tol, s->opts.max_cycles,
                       s->stream);
}

// Blocked solve (hz_options.rhs_block = b): the k columns of B are solved as
// ceil(k/b) independent block Krylov solves of <= b contiguous columns --
// each exactly the reference's block_fgmres / block_bicgstab on its columns
// (src/krylov.cpp:60-280), i.e. solve_block called per column group. The
// groups run concurrently (one host thread + stream each, hierarchy views
// sharing the operators). B and X are level-0 device blocks [n][k], ready on
// s->stream; X is complete when this returns.
Report run_grouped(hz_solver* s, int k, const double2* B, double2* X) {
  if (s->slabs) throw HzError(kValidation, "rhs_block: blocked solves are not supported in slab mode");
  const int kb = s->opts.rhs_block;
  const int G = (k + kb - 1) / kb;
  const int64_t n = s->prob->num_nodes();
  while (int(s->groups.size()) < G) {
    auto g = std::make_unique<RhsGroup>();
    HZ_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->h64 = s->h64->share();
    if (s->h32) g->h32 = s->h32->share();
    s->groups.push_back(std::move(g));
  }
  cudaEvent_t ready = nullptr;
  HZ_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  std::shared_ptr<void> ev_guard(ready, [](void* e) { cudaEventDestroy(static_cast<cudaEvent_t>(e)); });
  HZ_CUDA(cudaEventRecord(ready, s->stream));
  std::vector<Report> reps(static_cast<size_t>(G));
  std::vector<std::exception_ptr> errs(static_cast<size_t>(G));
  auto one = [&](int i) {
    try {
      DeviceGuard dg(s->prob->device);
      RhsGroup& g = *s->groups[i];
      const int c0 = i * kb, kg = std::min(kb, k - c0);
      const size_t pitch = size_t(k) * sizeof(double2), gp = size_t(kg) * sizeof(double2);
      g.B.ensure(size_t(n) * kg);
      g.X.ensure(size_t(n) * kg);
      HZ_CUDA(cudaStreamWaitEvent(g.stream, ready, 0));
      HZ_CUDA(cudaMemcpy2DAsync(g.B.get(), gp, B + c0, pitch, gp, size_t(n), cudaMemcpyDeviceToDevice, g.stream));
      DevOp<double> op = make_op_with(s, g.h64.get(), g.h32.get());
      if (s->bicgstab) {
        if (!g.bicg) g.bicg = std::make_unique<Bicgstab>();
        reps[i] = g.bicg->solve(op, kg, g.B.get(), g.X.get(), s->opts.tol, s->opts.max_cycles, g.stream);
      } else {
        if (!g.fgm) g.fgm = std::make_unique<Fgmres<double>>();
        reps[i] = g.fgm->solve(op, kg, g.B.get(), g.X.get(), s->opts.fgmres_restart, s->opts.tol,
                               s->opts.max_cycles, g.stream);
      }
      HZ_CUDA(cudaMemcpy2DAsync(X + c0, pitch, g.X.get(), gp, gp, size_t(n), cudaMemcpyDeviceToDevice, g.stream));
      HZ_CUDA(cudaStreamSynchronize(g.stream));
    } catch (...) {
      errs[i] = std::current_exception();
    }
  };
  if (G == 1) {
    one(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(size_t(G));
    for (int i = 0; i < G; ++i) th.emplace_back(one, i);
    for (auto& t : th) t.join();
  }
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  // merged report: columns in order; cycles / wall = slowest group; the
  // history is the worst column estimate over the groups per cycle
  Report rep;
  size_t hl = 0;
  for (const Report& r : reps) {
    rep.cycles = std::max(rep.cycles, r.cycles);
    rep.wall_s = std::max(rep.wall_s, r.wall_s);
    rep.qr_factorizations += r.qr_factorizations;
    rep.block_gram_products += r.block_gram_products;
    rep.col_cycles.insert(rep.col_cycles.end(), r.col_cycles.begin(), r.col_cycles.end());
    rep.rel_residual.insert(rep.rel_residual.end(), r.rel_residual.begin(), r.rel_residual.end());
    rep.converged.insert(rep.converged.end(), r.converged.begin(), r.converged.end());
    hl = std::max(hl, r.history.size());
  }
  rep.history.assign(hl, 0.0);
  for (const Report& r : reps)
    for (size_t t = 0; t < hl && !r.history.empty(); ++t)
      rep.history[t] = std::max(rep.history[t], r.history[std::min(t, r.history.size() - 1)]);
  return rep;
}

}  // namespace

extern "C" {

int hz_abi_version(void) { return HZ_ABI_VERSION; }
const char* hz_last_error_message(void) { return g_err.c_str(); }
int hz_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
int64_t hz_kernel_launch_count(void) { return g_launches.load(); }

int hz_measure_fp64_peak(double* tflops) {
  return guarded([&] {
    if (!tflops) throw HzError(kValidation, "hz_measure_fp64_peak: null output");
    *tflops = measure_dmma_tflops();
  });
}

int hz_profile_begin(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    HZ_CUDA(cudaDeviceSynchronize());
    g_prof_recs.clear();
    g_prof_recs.reserve(kProfPool / 2);
    for (cudaEvent_t e : g_prof_extra) cudaEventDestroy(e);
    g_prof_extra.clear();
    while (g_prof_pool.size() < kProfPool) {
      cudaEvent_t e;
      HZ_CUDA(cudaEventCreate(&e));
      g_prof_pool.push_back(e);
    }
    g_prof_next = 0;
    g_prof_on = true;
  });
}

int hz_profile_end(void) {
  return guarded([&] { g_prof_on = false; });
}

// Per-launch timeline of the profiled region: JSON list of
// [name, stream, start_ms, dur_ms, bytes] with start relative to the first
// recorded launch (events on different streams of one device compare).
int64_t hz_profile_trace(char* buf, int64_t cap) {
  std::string js;
  const int st = guarded([&] {
    HZ_CUDA(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::map<cudaStream_t, int> sid;
    std::ostringstream os;
    os.precision(9);
    os << "[";
    for (size_t i = 0; i < g_prof_recs.size(); ++i) {
      const auto& r = g_prof_recs[i];
      float t0 = 0, d = 0;
      HZ_CUDA(cudaEventElapsedTime(&t0, g_prof_recs[0].a, r.a));
      HZ_CUDA(cudaEventElapsedTime(&d, r.a, r.b));
      const int id = sid.emplace(r.s, int(sid.size())).first->second;
      os << (i ? "," : "") << "[\"" << r.name << "\"," << id << "," << t0 << "," << d << "," << r.bytes << "]";
    }
    os << "]";
    js = os.str();
  });
  if (st != kOk) return -1;
  const int64_t need = int64_t(js.size()) + 1;
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, int64_t(js.size()));
    std::memcpy(buf, js.data(), size_t(n));
    buf[n] = 0;
  }
  return need;
}

int64_t hz_profile_report(char* buf, int64_t cap) {
  std::string js;
  const int st = guarded([&] {
    HZ_CUDA(cudaDeviceSynchronize());
    struct Agg {
      int64_t count = 0;
      double ms = 0, bytes = 0, flops = 0;
    };
    std::map<std::string, Agg> agg;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (const auto& r : g_prof_recs) {
      float ms = 0;
      HZ_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      Agg& a = agg[r.name];
      a.count += 1;
      a.ms += ms;
      a.bytes += r.bytes;
      a.flops += r.flops;
    }
    std::ostringstream os;
    os.precision(17);
    os << "{";
    bool first = true;
    for (const auto& kv : agg) {
      if (!first) os << ",";
      first = false;
      os << "\"" << kv.first << "\":{\"count\":" << kv.second.count << ",\"ms\":" << kv.second.ms
         << ",\"bytes\":" << kv.second.bytes << ",\"flops\":" << kv.second.flops << "}";
    }
    os << "}";
    js = os.str();
  });
  if (st != kOk) return -1;
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(size_t(cap) - 1, js.size());
    std::memcpy(buf, js.data(), n);
    buf[n] = 0;
  }
  return int64_t(js.size()) + 1;
}

void hz_options_default(hz_options* o) {
  if (!o) return;
  o->method = HZ_METHOD_MG_BICGSTAB;
  o->tol = 1e-6;
  o->max_cycles = 200;
  o->nlevels = 3;
  o->shift_factor = 0.2;
  o->cycle_kind = HZ_CYCLE_W;
  o->pre = 2;
  o->post = 2;
  o->jacobi_weight = 0.8;
  o->k_inner = 2;
  o->fgmres_restart = 5;
  o->dense_threshold = 3000;
  o->precond_precision = HZ_C128;
  o->rhs_block = 0;
}

int hz_problem_create(int ndim, const int64_t n[3], const double h[3], const double* m,
                      double omega, double gamma_base, const double* ramp, int allow_coarse_ppw,
                      int device, hz_problem** out) {
  return hz_problem_create_ex(ndim, n, h, m, omega, gamma_base, ramp, allow_coarse_ppw, device, 7, out);
}

int hz_problem_create_ex(int ndim, const int64_t n[3], const double h[3], const double* m, double omega,
                         double gamma_base, const double* ramp, int allow_coarse_ppw, int device, int stencil,
                         hz_problem** out) {
  return guarded([&] {
    if (!out || !n || !h) throw HzError(kValidation, "hz_problem_create: null argument");
    require_device();
    DeviceGuard dg(device);
    auto* hp = new hz_problem;
    try {
      hp->p = std::make_shared<Problem>(ndim, n, h, m, omega, gamma_base, ramp, allow_coarse_ppw != 0,
                                        device, stencil);
    } catch (...) {
      delete hp;
      throw;
    }
    *out = hp;
  });
}

int hz_problem_destroy(hz_problem* p) {
  return guarded([&] {
    if (p) {
      DeviceGuard dg(p->p->device);
      delete p;
    }
  });
}

int hz_problem_ppw(const hz_problem* p, double* ppw) {
  return guarded([&] {
    if (!p || !ppw) throw HzError(kValidation, "null argument");
    *ppw = p->p->points_per_wavelength();
  });
}

int64_t hz_problem_num_nodes(const hz_problem* p) { return p ? p->p->num_nodes() : 0; }

int hz_apply_block_device(hz_problem* p, int64_t n, int k, const void* u, void* out, void* stream) {
  return guarded([&] {
    if (!p) throw HzError(kValidation, "null problem");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    launch_apply<double>(p->p->fine_op(k), static_cast<const double2*>(u), static_cast<double2*>(out),
                         static_cast<cudaStream_t>(stream));
  });
}

int hz_apply_block(hz_problem* p, int64_t n, int k, const double* u, double* out) {
  return guarded([&] {
    if (!p || !u || !out) throw HzError(kValidation, "null argument");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    const size_t e = size_t(n) * k;
    DevBuf<double2> du(e), dv(e);
    HZ_CUDA(cudaMemcpy(du.get(), u, e * sizeof(double2), cudaMemcpyHostToDevice));
    launch_apply<double>(p->p->fine_op(k), du.get(), dv.get(), nullptr);
    HZ_CUDA(cudaMemcpy(out, dv.get(), e * sizeof(double2), cudaMemcpyDeviceToHost));
  });
}

int hz_solver_create(hz_problem* p, const hz_options* opts, hz_solver** out) {
  return guarded([&] {
    if (!p || !out) throw HzError(kValidation, "hz_solver_create: null argument");
    DeviceGuard dg(p->p->device);
    auto s = std::make_unique<hz_solver>();
    s->prob = p->p;
    if (opts)
      s->opts = *opts;
    else
      hz_options_default(&s->opts);
    const hz_options& o = s->opts;
    if (o.precond_precision != HZ_C128 && o.precond_precision != HZ_C64)
      throw HzError(kValidation, "precond_precision must be HZ_C128 or HZ_C64");
    if (o.rhs_block < 0) throw HzError(kValidation, "rhs_block must be >= 0");
    HZ_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->spec.pre = o.pre;
    s->spec.post = o.post;
    s->spec.jacobi_weight = o.jacobi_weight;
    s->spec.k_inner = o.k_inner;
    if (o.pre < 0 || o.post < 0) throw HzError(kValidation, "relaxation counts must be >= 0");
    switch (o.method) {  // src/helmholtz_solver.cpp:19-29
      case HZ_METHOD_MG_BICGSTAB:
        s->spec.kind = CycleKind::W;
        s->bicgstab = true;
        break;
      case HZ_METHOD_MG_FGMRES_W:
        s->spec.kind = CycleKind::W;
        s->bicgstab = false;
        break;
      case HZ_METHOD_MG_FGMRES_K:
        s->spec.kind = CycleKind::K;
        s->bicgstab = false;
        break;
      case HZ_METHOD_MG_FGMRES:
        s->spec.kind = static_cast<CycleKind>(o.cycle_kind);
        s->bicgstab = false;
        break;
      case HZ_METHOD_MG_BICGSTAB_CYCLE:
        s->spec.kind = static_cast<CycleKind>(o.cycle_kind);
        s->bicgstab = true;
        break;
      case HZ_METHOD_DENSE_LU_SMALL:
        s->dense = true;
        break;
      default:
        throw HzError(kValidation, "unknown method");
    }
    if (o.cycle_kind < 0 || o.cycle_kind > 2) throw HzError(kValidation, "unknown cycle kind");
    const Problem& P = *s->prob;
    if (s->dense) {
      if (P.stencil == 27) throw HzError(kValidation, "dense_lu_small: 7-point operator only");
      const int64_t n = P.num_nodes();
      if (n > o.dense_threshold)
        throw HzError(kValidation, "dense_lu_small: grid has " + std::to_string(n) +
                                       " nodes, above the threshold " + std::to_string(o.dense_threshold));
      s->dense_ainvT = dense_inverse(P, s->stream);
      *out = s.release();
      return;
    }
    s->h64 = Hierarchy<double>::build(P, o.nlevels, o.shift_factor, s->stream);
    if (o.precond_precision == HZ_C64) s->h32 = Hierarchy<float>::rounded(*s->h64, s->stream);
    *out = s.release();
  });
}

int hz_solver_set_slabs(hz_solver* s, int nparts, const int* devices) {
  return guarded([&] {
    if (!s) throw HzError(kValidation, "null solver");
    if (s->prob->stencil == 27 && (nparts > 1 || devices))
      throw HzError(kValidation, "slabs: the 7-point fine operator only");
    DeviceGuard dg(s->prob->device);
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    auto detach = [&] {
      if (s->h64) s->h64->attach_slabs(nullptr, {});
      if (s->h32) s->h32->attach_slabs(nullptr, {});
      if (s->fgm) s->fgm->set_slabs(nullptr);
      s->dB.release();
      s->dX.release();
      s->span_k = 0;
      s->slabs.reset();
      s->rep32.clear();
      s->rep64.clear();
      s->center_rep.clear();
    };
    if (nparts <= 1 && !devices) {
      detach();
      return;
    }
    if (nparts < 1) throw HzError(kValidation, "slabs: nparts must be >= 1");
    if (s->dense || s->bicgstab)
      throw HzError(kValidation, "slab decomposition supports the block FGMRES methods");
    if (s->spec.kind == CycleKind::K) throw HzError(kValidation, "slab decomposition supports V and W cycles");
    std::vector<int> devs(nparts, s->prob->device);
    if (devices) devs.assign(devices, devices + nparts);
    if (devs[0] != s->prob->device) throw HzError(kValidation, "slabs: part 0 must be on the problem's GPU");
    int ndev = 0;
    HZ_CUDA(cudaGetDeviceCount(&ndev));
    for (int d : devs)
      if (d < 0 || d >= ndev) throw HzError(kValidation, "slabs: device index out of range");
    detach();
    std::vector<std::array<int64_t, 3>> dims;
    for (int l = 0; l < s->h64->num_levels(); ++l) dims.push_back(s->h64->level(l).dims);
    s->slabs = std::make_unique<Slabs>(devs, dims, s->prob->ndim, s->stream);
    const bool c64 = s->opts.precond_precision == HZ_C64;
    std::vector<const Hierarchy<double>*> r64;
    std::vector<const Hierarchy<float>*> r32;
    const size_t nn = size_t(s->prob->num_nodes());
    for (int d : devs) {
      if (d != s->prob->device && !s->center_rep.count(d)) {
        DeviceGuard g(d);
        DevBuf<double2>& c = s->center_rep[d];
        c.alloc(nn);
        HZ_CUDA(cudaMemcpyPeer(c.get(), d, s->prob->d_center.get(), s->prob->device, nn * sizeof(double2)));
        if (c64)
          s->rep32[d] = s->h32->replica(d, nullptr);
        else
          s->rep64[d] = s->h64->replica(d, nullptr);
      }
      r64.push_back(d == s->prob->device || c64 ? nullptr : s->rep64[d].get());
      r32.push_back(d == s->prob->device || !c64 ? nullptr : s->rep32[d].get());
    }
    if (c64)
      s->h32->attach_slabs(s->slabs.get(), r32);
    else
      s->h64->attach_slabs(s->slabs.get(), r64);
    if (!s->fgm) s->fgm = std::make_unique<Fgmres<double>>();
    s->fgm->set_slabs(s->slabs.get());
  });
}

int hz_solver_slab_info(const hz_solver* s, int* nparts, int* agg_level, int64_t* planes, int cap) {
  return guarded([&] {
    if (!s || !nparts) throw HzError(kValidation, "null argument");
    if (!s->slabs) {
      *nparts = 1;
      if (agg_level) *agg_level = 0;
      return;
    }
    const Slabs& sl = *s->slabs;
    *nparts = sl.parts();
    if (agg_level) *agg_level = sl.agg_level();
    // planes[l * (P + 1) + p] = first plane of part p on level l
    if (planes)
      for (int l = 0; l < sl.levels(); ++l)
        for (int p = 0; p <= sl.parts(); ++p) {
          const int i = l * (sl.parts() + 1) + p;
          if (i < cap) planes[i] = p < sl.parts() ? sl.z0(l, p) : sl.z1(l, sl.parts() - 1);
        }
  });
}

int hz_solver_destroy(hz_solver* s) {
  return guarded([&] {
    if (s) {
      DeviceGuard dg(s->prob->device);
      delete s;
    }
  });
}

int hz_solver_set_tolerance(hz_solver* s, double tol) {
  return guarded([&] {
    if (!s) throw HzError(kValidation, "null solver");
    s->opts.tol = tol;
  });
}

int hz_solve_block_device_stream(hz_solver* s, int64_t n, int k, const void* B, void* X, hz_report* rep,
                                 void* stream) {
  return guarded([&] {
    if (!s || !B || !X) throw HzError(kValidation, "null argument");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    order_after_caller(s, stream);
    Report r = run_solve(s, k, static_cast<const double2*>(B), static_cast<double2*>(X));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
  });
}

int hz_solve_block_device(hz_solver* s, int64_t n, int k, const void* B, void* X, hz_report* rep) {
  return guarded([&] {
    if (!s || !B || !X) throw HzError(kValidation, "null argument");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    order_after_caller(s, nullptr);
    Report r = run_solve(s, k, static_cast<const double2*>(B), static_cast<double2*>(X));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
  });
}

int hz_solve_block(hz_solver* s, int64_t n, int k, const double* B, double* X, hz_report* rep) {
  return guarded([&] {
    if (!s || !B || !X) throw HzError(kValidation, "null argument");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    s->ensure_blocks(k);
    upload_rows(s, k, B, s->dB.get());
    Report r = run_solve(s, k, s->dB.get(), s->dX.get());
    download_rows(s, k, s->dX.get(), X);
    fill_report(r, k, rep);
  });
}

}  // extern "C"

namespace {
std::string thread_error() { return g_err; }
void set_thread_error(const std::string& m) { g_err = m; }
// one host thread per solve: every solve keeps its own host control flow
// (syncs included) while the kernels of all of them share the GPU
template <class F>
int run_concurrent(int count, hz_solver* const* solvers, F&& one) {
  if (count < 0) {
    set_thread_error("multi solve: negative count");
    return kValidation;
  }
  if (count > 0 && !solvers) {
    set_thread_error("null argument");
    return kValidation;
  }
  for (int i = 0; i < count; ++i) {
    if (!solvers[i]) {
      set_thread_error("multi solve: null solver");
      return kValidation;
    }
    for (int j = 0; j < i; ++j)
      if (solvers[j] == solvers[i]) {
        set_thread_error("multi solve: solvers must be distinct (each owns its stream and workspace)");
        return kValidation;
      }
  }
  std::vector<int> st(size_t(count), kOk);
  std::vector<std::string> errs(static_cast<size_t>(count));
  std::vector<std::thread> th;
  th.reserve(size_t(count));
  for (int i = 0; i < count; ++i)
    th.emplace_back([&st, &errs, &one, i] {
      st[i] = one(i);
      if (st[i] != kOk) errs[i] = thread_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < count; ++i)
    if (st[i] != kOk) {
      set_thread_error("multi solve " + std::to_string(i) + ": " + errs[i]);
      return st[i];
    }
  return kOk;
}
}  // namespace

extern "C" {

int hz_solve_blocks_multi(int count, hz_solver* const* solvers, const int64_t* n, const int* k,
                          const double* const* B, double* const* X, hz_report* reps) {
  if (count > 0 && (!n || !k || !B || !X)) {
    g_err = "null argument";
    return kValidation;
  }
  return run_concurrent(count, solvers, [&](int i) {
    return hz_solve_block(solvers[i], n[i], k[i], B[i], X[i], reps ? &reps[i] : nullptr);
  });
}

int hz_solve_blocks_multi_device(int count, hz_solver* const* solvers, const int64_t* n, const int* k,
                                 const void* const* B, void* const* X, hz_report* reps) {
  if (count > 0 && (!n || !k || !B || !X)) {
    g_err = "null argument";
    return kValidation;
  }
  return run_concurrent(count, solvers, [&](int i) {
    return hz_solve_block_device(solvers[i], n[i], k[i], B[i], X[i], reps ? &reps[i] : nullptr);
  });
}

// Block algebra of the Arnoldi step on caller device blocks (current
// device, synchronous), for kernel-level parity with the reference.
int hz_block_gram_device(int64_t n, int k, int nb, const void* const* X, const void* Y, double* G) {
  return guarded([&] {
    if (!X || !Y || !G) throw HzError(kValidation, "null argument");
    if (n < 1 || nb < 1 || nb > kMaxBlocks) throw HzError(kValidation, "block gram: bad n / nb");
    BlockAlgebra<double> alg;
    alg.ensure(n, k, nb);
    BlockTab<double> tab{};
    for (int i = 0; i < nb; ++i) tab.p[i] = static_cast<const double2*>(X[i]);
    DevBuf<double2> out(size_t(nb) * k * k);
    alg.gram(tab, nb, static_cast<const double2*>(Y), out.get(), nullptr);
    HZ_CUDA(cudaMemcpy(G, out.get(), out.bytes(), cudaMemcpyDeviceToHost));
  });
}

int hz_block_add_scaled_device(int64_t n, int k, int nb, const void* const* X, const double* C, void* Y) {
  return guarded([&] {
    if (!X || !C || !Y) throw HzError(kValidation, "null argument");
    if (n < 1 || nb < 1 || nb > kMaxBlocks) throw HzError(kValidation, "block update: bad n / nb");
    if (k < 1 || k > 64) throw HzError(kValidation, "block width must be in [1, 64]");
    BlockTab<double> tab{};
    for (int i = 0; i < nb; ++i) tab.p[i] = static_cast<const double2*>(X[i]);
    DevBuf<double2> c(size_t(nb) * k * k);
    HZ_CUDA(cudaMemcpy(c.get(), C, c.bytes(), cudaMemcpyHostToDevice));
    auto* y = static_cast<double2*>(Y);
    launch_multi_update<double>(n, k, nb, tab, c.get(), y, y, 1.0, nullptr);
    HZ_CUDA(cudaDeviceSynchronize());
  });
}

// solve_helmholtz (src/helmholtz_solver.cpp:81-93): the convergence check runs
// on the internal Report, so it holds whether or not the caller passes a
// report (or its converged buffer).
int hz_solve_helmholtz(hz_solver* s, int64_t n, int k, const double* B, double* X, hz_report* rep) {
  return guarded([&] {
    if (!s || !B || !X) throw HzError(kValidation, "null argument");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    s->ensure_blocks(k);
    upload_rows(s, k, B, s->dB.get());
    Report r = run_solve(s, k, s->dB.get(), s->dX.get());
    download_rows(s, k, s->dX.get(), X);
    fill_report(r, k, rep);
    require_converged(r, "helmholtz solve: tolerance not met within cycle cap");
  });
}

int hz_cycle_device_stream(hz_solver* s, int64_t n, int k, const void* b, void* x, void* stream) {
  return guarded([&] {
    if (!s || !b || !x) throw HzError(kValidation, "null argument");
    if (s->dense) throw HzError(kState, "dense solver has no multigrid cycle");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    order_after_caller(s, stream);
    DevOp<double> op = make_op(s, k);
    op.prec(static_cast<const double2*>(b), static_cast<double2*>(x), k, s->stream);
    if (s->slabs) s->slabs->join();
    HZ_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int hz_cycle_device(hz_solver* s, int64_t n, int k, const void* b, void* x) {
  return guarded([&] {
    if (!s || !b || !x) throw HzError(kValidation, "null argument");
    if (s->dense) throw HzError(kState, "dense solver has no multigrid cycle");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    order_after_caller(s, nullptr);
    DevOp<double> op = make_op(s, k);
    op.prec(static_cast<const double2*>(b), static_cast<double2*>(x), k, s->stream);
    if (s->slabs) s->slabs->join();
    HZ_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int hz_cycle(hz_solver* s, int64_t n, int k, const double* b, double* x) {
  return guarded([&] {
    if (!s || !b || !x) throw HzError(kValidation, "null argument");
    if (s->dense) throw HzError(kState, "dense solver has no multigrid cycle");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    s->ensure_blocks(k);
    upload_rows(s, k, b, s->dB.get());
    DevOp<double> op = make_op(s, k);
    op.prec(s->dB.get(), s->dX.get(), k, s->stream);
    download_rows(s, k, s->dX.get(), x);
  });
}

int hz_coarse_solve(hz_solver* s, int64_t nc, int k, const double* b, double* x) {
  return guarded([&] {
    if (!s || !b || !x) throw HzError(kValidation, "null argument");
    if (!s->h64) throw HzError(kState, "no hierarchy");
    if (nc != s->h64->coarse_n()) throw HzError(kValidation, "coarse size mismatch");
    DeviceGuard dg(s->prob->device);
    const size_t e = size_t(nc) * k;
    DevBuf<double2> db(e), dx(e);
    HZ_CUDA(cudaMemcpyAsync(db.get(), b, e * sizeof(double2), cudaMemcpyHostToDevice, s->stream));
    s->h64->coarse_solve(k, db.get(), dx.get(), s->stream);
    HZ_CUDA(cudaMemcpyAsync(x, dx.get(), e * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int hz_hierarchy_num_levels(const hz_solver* s, int* nlevels) {
  return guarded([&] {
    if (!s || !nlevels) throw HzError(kValidation, "null argument");
    *nlevels = s->h64 ? s->h64->num_levels() : 0;
  });
}

int hz_hierarchy_level_dims(const hz_solver* s, int level, int64_t dims[3]) {
  return guarded([&] {
    if (!s || !dims || !s->h64) throw HzError(kValidation, "null argument");
    if (level < 0 || level >= s->h64->num_levels()) throw HzError(kValidation, "level out of range");
    for (int a = 0; a < 3; ++a) dims[a] = s->h64->level(level).dims[a];
  });
}

int hz_hierarchy_level_coefficients(const hz_solver* s, int level, double* out, int64_t count) {
  return guarded([&] {
    if (!s || !out || !s->h64) throw HzError(kValidation, "null argument");
    if (level < 0 || level >= s->h64->num_levels()) throw HzError(kValidation, "level out of range");
    DeviceGuard dg(s->prob->device);
    std::vector<cplx> c;
    s->h64->download_level(level, c);
    if (count != int64_t(c.size())) throw HzError(kValidation, "coefficient count mismatch");
    std::memcpy(out, c.data(), c.size() * sizeof(cplx));
  });
}

int hz_sensitivity_accumulate_device(hz_problem* p, int64_t n, int k, const void* U, const void* L,
                                     double* g, int accumulate, void* stream) {
  return guarded([&] {
    if (!p || !U || !L || !g) throw HzError(kValidation, "null argument");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    launch_sensitivity(n, k, p->p->omega * p->p->omega, p->p->d_gf.get(),
                       static_cast<const double2*>(U), static_cast<const double2*>(L), g, accumulate,
                       static_cast<cudaStream_t>(stream));
  });
}

int hz_sensitivity_accumulate(hz_problem* p, int64_t n, int k, const double* U, const double* L,
                              double* g, int accumulate) {
  return guarded([&] {
    if (!p || !U || !L || !g) throw HzError(kValidation, "null argument");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    const size_t e = size_t(n) * k;
    DevBuf<double2> du(e), dl(e);
    DevBuf<double> dg_(n);
    HZ_CUDA(cudaMemcpy(du.get(), U, e * sizeof(double2), cudaMemcpyHostToDevice));
    HZ_CUDA(cudaMemcpy(dl.get(), L, e * sizeof(double2), cudaMemcpyHostToDevice));
    if (accumulate) HZ_CUDA(cudaMemcpy(dg_.get(), g, n * sizeof(double), cudaMemcpyHostToDevice));
    launch_sensitivity(n, k, p->p->omega * p->p->omega, p->p->d_gf.get(), du.get(), dl.get(),
                       dg_.get(), accumulate, nullptr);
    HZ_CUDA(cudaMemcpy(g, dg_.get(), n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

// ---------------------------------------------------------------- FWI path
int hz_sampling_create(const hz_problem* p, const double origin[3], int64_t nrec, const double* xyz,
                       hz_sampling** out) {
  return guarded([&] {
    if (!p || !out || (nrec > 0 && !xyz)) throw HzError(kValidation, "hz_sampling_create: null argument");
    const Problem& P = *p->p;
    const double zero[3] = {0, 0, 0};
    auto* hs = new hz_sampling;
    try {
      hs->s = std::make_unique<Sampling>(P.ndim, P.n.data(), P.h.data(), origin ? origin : zero, nrec, xyz,
                                         P.device);
    } catch (...) {
      delete hs;
      throw;
    }
    *out = hs;
  });
}

int hz_sampling_destroy(hz_sampling* s) {
  return guarded([&] {
    if (s) {
      DeviceGuard dg(s->s->device);
      delete s;
    }
  });
}

int64_t hz_sampling_num_receivers(const hz_sampling* s) { return s ? s->s->nrec : 0; }

int hz_sampling_receiver(const hz_sampling* s, int64_t r, int64_t nodes[8], double weights[8], int* count) {
  return guarded([&] {
    if (!s || !nodes || !weights || !count) throw HzError(kValidation, "null argument");
    const Sampling& S = *s->s;
    if (r < 0 || r >= S.nrec) throw HzError(kValidation, "receiver index out of range");
    *count = int(S.rp[r + 1] - S.rp[r]);
    for (int q = 0; q < *count; ++q) {
      nodes[q] = S.nodes[S.rp[r] + q];
      weights[q] = S.w[S.rp[r] + q];
    }
  });
}

int hz_sample_device(hz_sampling* s, int k, const void* U, void* D, void* stream) {
  return guarded([&] {
    if (!s || !U || (!D && s->s->nrec)) throw HzError(kValidation, "null argument");
    if (k < 1) throw HzError(kValidation, "sample: k must be >= 1");
    DeviceGuard dg(s->s->device);
    launch_sample(*s->s, k, static_cast<const double2*>(U), static_cast<double2*>(D),
                  static_cast<cudaStream_t>(stream));
  });
}

int hz_sample_adjoint_device(hz_sampling* s, int k, const void* D, void* U, int conj, void* stream) {
  return guarded([&] {
    if (!s || !U || (!D && s->s->nrec)) throw HzError(kValidation, "null argument");
    if (k < 1) throw HzError(kValidation, "sample_adjoint: k must be >= 1");
    DeviceGuard dg(s->s->device);
    launch_sample_adjoint(*s->s, k, static_cast<const double2*>(D), static_cast<double2*>(U), conj != 0,
                          static_cast<cudaStream_t>(stream));
  });
}

int hz_sample(hz_sampling* s, int k, const double* U, double* D) {
  return guarded([&] {
    if (!s || !U || (!D && s->s->nrec)) throw HzError(kValidation, "null argument");
    if (k < 1) throw HzError(kValidation, "sample: k must be >= 1");
    const Sampling& S = *s->s;
    DeviceGuard dg(S.device);
    DevBuf<double2> du(size_t(S.n) * k), dd(std::max<size_t>(size_t(S.nrec) * k, 1));
    HZ_CUDA(cudaMemcpy(du.get(), U, du.bytes(), cudaMemcpyHostToDevice));
    launch_sample(S, k, du.get(), dd.get(), nullptr);
    if (S.nrec) HZ_CUDA(cudaMemcpy(D, dd.get(), sizeof(double2) * S.nrec * k, cudaMemcpyDeviceToHost));
  });
}

int hz_sample_adjoint(hz_sampling* s, int k, const double* D, double* U, int conj) {
  return guarded([&] {
    if (!s || !U || (!D && s->s->nrec)) throw HzError(kValidation, "null argument");
    if (k < 1) throw HzError(kValidation, "sample_adjoint: k must be >= 1");
    const Sampling& S = *s->s;
    DeviceGuard dg(S.device);
    DevBuf<double2> du(size_t(S.n) * k), dd(std::max<size_t>(size_t(S.nrec) * k, 1));
    if (S.nrec) HZ_CUDA(cudaMemcpy(dd.get(), D, sizeof(double2) * S.nrec * k, cudaMemcpyHostToDevice));
    launch_sample_adjoint(S, k, dd.get(), du.get(), conj != 0, nullptr);
    HZ_CUDA(cudaMemcpy(U, du.get(), du.bytes(), cudaMemcpyDeviceToHost));
  });
}

int hz_fwi_sensitivity_rhs_device(hz_problem* p, int64_t n, int k, const void* U, const void* v, void* R,
                                  void* stream) {
  return guarded([&] {
    if (!p || !U || !v || !R) throw HzError(kValidation, "null argument");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    launch_sens_rhs(n, k, p->p->omega * p->p->omega, p->p->d_gf.get(), static_cast<const double2*>(U),
                    static_cast<const double*>(v), static_cast<double2*>(R), static_cast<cudaStream_t>(stream));
  });
}

namespace {
// fwi_jacobian_vec (src/helmholtz_solver.cpp:113-125) for k stored fields at
// once: D = P^T A^{-1} (-w^2 gf U v), one block solve
void jacobian_vec(hz_solver* s, hz_sampling* smp, int k, const double2* U, const double* v, double2* D,
                  Report& rep) {
  const Problem& P = *s->prob;
  const int64_t n = P.num_nodes();
  s->fR.ensure(size_t(n) * k);
  s->fX.ensure(size_t(n) * k);
  launch_sens_rhs(n, k, P.omega * P.omega, P.d_gf.get(), U, v, s->fR.get(), s->stream);
  rep = run_solve(s, k, s->fR.get(), s->fX.get());
  launch_sample(*smp->s, k, s->fX.get(), D, s->stream);
}
// fwi_jacobian_transpose_vec (src/helmholtz_solver.cpp:127-139) for k
// sources: g (+)= sum_s Re(-w^2 gf u_s lambda_s), lambda = A^{-1} P conj(w_s)
void jacobian_transpose_vec(hz_solver* s, hz_sampling* smp, int k, const double2* U, const double2* W, double* g,
                            int accumulate, Report& rep) {
  const Problem& P = *s->prob;
  const int64_t n = P.num_nodes();
  s->fR.ensure(size_t(n) * k);
  s->fX.ensure(size_t(n) * k);
  launch_sample_adjoint(*smp->s, k, W, s->fR.get(), true, s->stream);
  rep = run_solve(s, k, s->fR.get(), s->fX.get());
  launch_sensitivity(n, k, P.omega * P.omega, P.d_gf.get(), U, s->fX.get(), g, accumulate, s->stream);
}
void check_fwi(hz_solver* s, hz_sampling* smp, int64_t n, int k) {
  if (!s || !smp) throw HzError(kValidation, "null argument");
  if (s->slabs) throw HzError(kState, "FWI block functions run on a single-domain solver");
  check_block(*s->prob, n, k);
  if (smp->s->n != n) throw HzError(kValidation, "sampling operator does not match the grid");
  if (smp->s->device != s->prob->device) throw HzError(kValidation, "sampling operator on another GPU");
}
}  // namespace

int hz_fwi_jacobian_vec_device(hz_solver* s, hz_sampling* smp, int64_t n, int k, const void* U, const void* v,
                               void* D, hz_report* rep) {
  return guarded([&] {
    check_fwi(s, smp, n, k);
    if (!U || !v || (!D && smp->s->nrec)) throw HzError(kValidation, "null argument");
    DeviceGuard dg(s->prob->device);
    Report r;
    jacobian_vec(s, smp, k, static_cast<const double2*>(U), static_cast<const double*>(v),
                 static_cast<double2*>(D), r);
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
    require_converged(r, "fwi_jacobian_vec: sensitivity solve did not converge");
  });
}

int hz_fwi_jacobian_vec(hz_solver* s, hz_sampling* smp, int64_t n, int k, const double* U, const double* v,
                        double* D, hz_report* rep) {
  return guarded([&] {
    check_fwi(s, smp, n, k);
    if (!U || !v || (!D && smp->s->nrec)) throw HzError(kValidation, "null argument");
    DeviceGuard dg(s->prob->device);
    const int64_t nr = smp->s->nrec;
    s->fU.ensure(size_t(n) * k);
    s->fv.ensure(size_t(n));
    s->fD.ensure(std::max<size_t>(size_t(nr) * k, 1));
    HZ_CUDA(cudaMemcpyAsync(s->fU.get(), U, sizeof(double2) * n * k, cudaMemcpyHostToDevice, s->stream));
    HZ_CUDA(cudaMemcpyAsync(s->fv.get(), v, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    Report r;
    jacobian_vec(s, smp, k, s->fU.get(), s->fv.get(), s->fD.get(), r);
    if (nr) HZ_CUDA(cudaMemcpyAsync(D, s->fD.get(), sizeof(double2) * nr * k, cudaMemcpyDeviceToHost, s->stream));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
    require_converged(r, "fwi_jacobian_vec: sensitivity solve did not converge");
  });
}

int hz_fwi_jacobian_transpose_vec_device(hz_solver* s, hz_sampling* smp, int64_t n, int k, const void* U,
                                         const void* W, double* g, int accumulate, hz_report* rep) {
  return guarded([&] {
    check_fwi(s, smp, n, k);
    if (!U || !g || (!W && smp->s->nrec)) throw HzError(kValidation, "null argument");
    DeviceGuard dg(s->prob->device);
    Report r;
    jacobian_transpose_vec(s, smp, k, static_cast<const double2*>(U), static_cast<const double2*>(W), g,
                           accumulate, r);
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
    require_converged(r, "fwi_jacobian_transpose_vec: adjoint solve did not converge");
  });
}

int hz_fwi_jacobian_transpose_vec(hz_solver* s, hz_sampling* smp, int64_t n, int k, const double* U,
                                  const double* W, double* g, int accumulate, hz_report* rep) {
  return guarded([&] {
    check_fwi(s, smp, n, k);
    if (!U || !g || (!W && smp->s->nrec)) throw HzError(kValidation, "null argument");
    DeviceGuard dg(s->prob->device);
    const int64_t nr = smp->s->nrec;
    s->fU.ensure(size_t(n) * k);
    s->fD.ensure(std::max<size_t>(size_t(nr) * k, 1));
    s->fv.ensure(size_t(n));
    HZ_CUDA(cudaMemcpyAsync(s->fU.get(), U, sizeof(double2) * n * k, cudaMemcpyHostToDevice, s->stream));
    if (nr) HZ_CUDA(cudaMemcpyAsync(s->fD.get(), W, sizeof(double2) * nr * k, cudaMemcpyHostToDevice, s->stream));
    if (accumulate) HZ_CUDA(cudaMemcpyAsync(s->fv.get(), g, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    Report r;
    jacobian_transpose_vec(s, smp, k, s->fU.get(), s->fD.get(), s->fv.get(), accumulate, r);
    HZ_CUDA(cudaMemcpyAsync(g, s->fv.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
    HZ_CUDA(cudaStreamSynchronize(s->stream));
    fill_report(r, k, rep);
    require_converged(r, "fwi_jacobian_transpose_vec: adjoint solve did not converge");
  });
}

// ---------------------------------------------------------------- Compact16
namespace {
// WavefieldBatch::append Compact16 (src/helmholtz.cpp:143-151) for k
// columns: scale_c = 2^ceil(log2(peak_c)) (1 when the column is zero)
void compact16(int64_t n, int k, const double2* X, uint32_t* Q, double* scales, DevBuf<double>& part,
               DevBuf<double>& mx, cudaStream_t st) {
  const int nslots = int(std::min<int64_t>(4 * kNumSMs, std::max<int64_t>(1, n / 1024)));
  part.ensure(size_t(nslots) * k);
  mx.ensure(2 * size_t(k));
  launch_colmax(n, k, X, part.get(), nslots, mx.get(), st);
  std::vector<double> peak(k), inv(k);
  HZ_CUDA(cudaMemcpyAsync(peak.data(), mx.get(), sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  HZ_CUDA(cudaStreamSynchronize(st));
  for (int c = 0; c < k; ++c) {
    scales[c] = peak[c] > 0.0 ? std::exp2(std::ceil(std::log2(peak[c]))) : 1.0;
    inv[c] = 1.0 / scales[c];  // exact: scales are powers of two
  }
  HZ_CUDA(cudaMemcpyAsync(mx.get() + k, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
  launch_quantize16(n, k, X, mx.get() + k, Q, st);
  HZ_CUDA(cudaStreamSynchronize(st));  // inv lives on this stack frame
}
}  // namespace

int hz_compact16_device(int64_t n, int k, const void* X, void* Q, double* scales, void* stream) {
  return guarded([&] {
    if (!X || !Q || !scales) throw HzError(kValidation, "null argument");
    if (n < 1 || k < 1) throw HzError(kValidation, "compact16: empty block");
    DevBuf<double> part, mx;
    compact16(n, k, static_cast<const double2*>(X), static_cast<uint32_t*>(Q), scales, part, mx,
              static_cast<cudaStream_t>(stream));
  });
}

int hz_compact16(int64_t n, int k, const double* X, uint16_t* Q, double* scales) {
  return guarded([&] {
    if (!X || !Q || !scales) throw HzError(kValidation, "null argument");
    if (n < 1 || k < 1) throw HzError(kValidation, "compact16: empty block");
    require_device();
    DevBuf<double2> dx(size_t(n) * k);
    DevBuf<uint32_t> dq(size_t(n) * k);
    DevBuf<double> part, mx;
    HZ_CUDA(cudaMemcpy(dx.get(), X, dx.bytes(), cudaMemcpyHostToDevice));
    compact16(n, k, dx.get(), dq.get(), scales, part, mx, nullptr);
    HZ_CUDA(cudaMemcpy(Q, dq.get(), dq.bytes(), cudaMemcpyDeviceToHost));
  });
}

int hz_solve_helmholtz_compact16(hz_solver* s, int64_t n, int k, const double* B, uint16_t* Q, double* scales,
                                 hz_report* rep) {
  return guarded([&] {
    if (!s || !B || !Q || !scales) throw HzError(kValidation, "null argument");
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    s->ensure_blocks(k);
    upload_rows(s, k, B, s->dB.get());
    Report r = run_solve(s, k, s->dB.get(), s->dX.get());
    if (s->slabs) s->slabs->join();
    fill_report(r, k, rep);
    require_converged(r, "helmholtz solve: tolerance not met within cycle cap");
    s->fQ.ensure(size_t(n) * k);
    compact16(n, k, s->dX.get(), s->fQ.get(), scales, s->fpart, s->fmax, s->stream);
    HZ_CUDA(cudaMemcpy(Q, s->fQ.get(), sizeof(uint32_t) * n * k, cudaMemcpyDeviceToHost));
  });
}


// ---------------------------------------------------------------- drop-in surface
// (include/hz_b200.hpp's seistomo-compatible classes; reference file:line
// next to each)

int hz_problem_mass(const hz_problem* p, double* out) {
  return guarded([&] {
    if (!p || !out) throw HzError(kValidation, "null argument");
    std::memcpy(out, p->p->mass.data(), p->p->mass.size() * sizeof(cplx));
  });
}

int hz_problem_gamma_factor(const hz_problem* p, double* out) {
  return guarded([&] {
    if (!p || !out) throw HzError(kValidation, "null argument");
    std::memcpy(out, p->p->gamma_factor.data(), p->p->gamma_factor.size() * sizeof(cplx));
  });
}

}  // extern "C"

namespace {
// RegularGrid::contains / nearest_node (src/grid.cpp:34-55) on the problem's
// grid placed at `origin`
bool grid_contains(const Problem& P, const double* origin, const double* x) {
  const double eps = 1e-9;
  for (int a = 0; a < P.ndim; ++a) {
    const double lo = origin[a] - eps * P.h[a];
    const double hi = origin[a] + double(P.n[a] - 1) * P.h[a] + eps * P.h[a];
    if (x[a] < lo || x[a] > hi) return false;
  }
  return true;
}
int64_t grid_nearest(const Problem& P, const double* origin, const double* x) {
  int64_t c[3] = {0, 0, 0};
  for (int a = 0; a < P.ndim; ++a) {
    const double f = (x[a] - origin[a]) / P.h[a];
    int64_t i = static_cast<int64_t>(std::floor(f + 0.5));
    if (static_cast<double>(i) - f == 0.5) --i;  // exact tie: toward the lower index
    c[a] = std::clamp<int64_t>(i, 0, P.n[a] - 1);
  }
  return c[0] + P.n[0] * (c[1] + P.n[1] * c[2]);
}
// HelmholtzProblem::point_source (src/helmholtz.cpp:124-132): node + amplitude / prod(h)
std::pair<int64_t, cplx> point_source_entry(const Problem& P, const double* origin, const double* x, cplx amp) {
  if (!grid_contains(P, origin, x)) throw HzError(kValidation, "point_source: position outside grid");
  double cell = 1.0;
  for (int a = 0; a < P.ndim; ++a) cell *= P.h[a];
  return {grid_nearest(P, origin, x), amp / cell};
}
const double kZeroOrigin[3] = {0.0, 0.0, 0.0};
}  // namespace

extern "C" {

int hz_problem_nearest_node(const hz_problem* p, const double origin[3], const double x[3], int64_t* node) {
  return guarded([&] {
    if (!p || !x || !node) throw HzError(kValidation, "null argument");
    *node = grid_nearest(*p->p, origin ? origin : kZeroOrigin, x);
  });
}

int hz_problem_point_source(const hz_problem* p, const double origin[3], const double x[3], double amp_re,
                            double amp_im, double* q) {
  return guarded([&] {
    if (!p || !x || !q) throw HzError(kValidation, "null argument");
    const auto e = point_source_entry(*p->p, origin ? origin : kZeroOrigin, x, cplx(amp_re, amp_im));
    std::memset(q, 0, size_t(p->p->num_nodes()) * sizeof(cplx));
    reinterpret_cast<cplx*>(q)[e.first] = e.second;
  });
}

int hz_point_sources_device(hz_problem* p, const double origin[3], int k, const double* xyz, const double* amp,
                            void* B, void* stream) {
  return guarded([&] {
    if (!p || !xyz || !B) throw HzError(kValidation, "null argument");
    check_block(*p->p, p->p->num_nodes(), k);
    std::vector<int64_t> nodes(k);
    std::vector<double2> vals(k);
    for (int j = 0; j < k; ++j) {
      const cplx a = amp ? cplx(amp[2 * j], amp[2 * j + 1]) : cplx(1.0, 0.0);
      const auto e = point_source_entry(*p->p, origin ? origin : kZeroOrigin, xyz + 3 * j, a);
      nodes[j] = e.first;
      vals[j] = make_double2(e.second.real(), e.second.imag());
    }
    DeviceGuard dg(p->p->device);
    auto st = static_cast<cudaStream_t>(stream);
    HZ_CUDA(cudaMemsetAsync(B, 0, size_t(p->p->num_nodes()) * k * sizeof(double2), st));
    launch_point_sources(k, nodes.data(), vals.data(), static_cast<double2*>(B), st);
  });
}

// HelmholtzProblem::to_csr (src/helmholtz.cpp:102-122): rows in node order,
// columns ascending (CsrBuilder), nnz = 5/7 per interior row
int hz_problem_to_csr(const hz_problem* p, double shift, int64_t* rp, int32_t* ci, double* v, int64_t cap,
                      int64_t* nnz) {
  return guarded([&] {
    if (!p || !nnz) throw HzError(kValidation, "null argument");
    const Problem& P = *p->p;
    if (P.stencil == 27) {
      // the compact operator's planes, shifted on the device, in ascending column order
      const int64_t nn = P.num_nodes();
      int64_t cnt27 = 0;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int64_t c = 1;
            const int d[3] = {dx, dy, dz};
            for (int a = 0; a < 3; ++a) c *= P.n[a] - (d[a] != 0 ? 1 : 0);
            cnt27 += c;
          }
      *nnz = cnt27;
      if (!rp || !ci || !v) return;
      if (cap < cnt27) throw HzError(kValidation, "to_csr: output capacity below nnz");
      DeviceGuard dg(P.device);
      DevBuf<double2> planes(size_t(27) * nn);
      P.build_coef27(shift, planes.get(), nullptr);
      std::vector<cplx> hp(size_t(27) * nn);
      HZ_CUDA(cudaMemcpy(hp.data(), planes.get(), planes.bytes(), cudaMemcpyDeviceToHost));
      auto* vv = reinterpret_cast<cplx*>(v);
      int64_t e = 0;
      rp[0] = 0;
      const int64_t n0 = P.n[0], n1 = P.n[1], n2 = P.n[2];
      for (int64_t kz = 0; kz < n2; ++kz)
        for (int64_t j = 0; j < n1; ++j)
          for (int64_t i = 0; i < n0; ++i) {
            const int64_t idx = i + n0 * (j + n1 * kz);
            for (int dz = -1; dz <= 1; ++dz)
              for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                  const int64_t ii = i + dx, jj = j + dy, kk = kz + dz;
                  if (ii < 0 || ii >= n0 || jj < 0 || jj >= n1 || kk < 0 || kk >= n2) continue;
                  ci[e] = int32_t(ii + n0 * (jj + n1 * kk));
                  vv[e] = hp[size_t((dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)) * nn + idx];
                  ++e;
                }
            rp[idx + 1] = e;
          }
      return;
    }
    const int64_t n0 = P.n[0], n1 = P.n[1], n2 = P.n[2], s1 = n0, s2 = n0 * n1;
    int64_t cnt = 0;
    for (int a = 0; a < 3; ++a) cnt += P.n[a] > 1 ? 2 * (P.n[a] - 1) * (P.num_nodes() / P.n[a]) : 0;
    cnt += P.num_nodes();
    *nnz = cnt;
    if (!rp || !ci || !v) return;  // size query
    if (cap < cnt) throw HzError(kValidation, "to_csr: output capacity below nnz");
    if (P.num_nodes() > int64_t(INT32_MAX)) throw HzError(kValidation, "to_csr: int32 column indices overflow");
    const auto c = P.shifted_center(shift);
    auto* vv = reinterpret_cast<cplx*>(v);
    int64_t e = 0;
    rp[0] = 0;
    for (int64_t kz = 0; kz < n2; ++kz)
      for (int64_t j = 0; j < n1; ++j)
        for (int64_t i = 0; i < n0; ++i) {
          const int64_t idx = i + n0 * (j + n1 * kz);
          auto put = [&](int64_t col, cplx val) {
            ci[e] = int32_t(col);
            vv[e] = val;
            ++e;
          };
          if (kz > 0) put(idx - s2, P.inv_h2[2]);
          if (j > 0) put(idx - s1, P.inv_h2[1]);
          if (i > 0) put(idx - 1, P.inv_h2[0]);
          put(idx, c[idx]);
          if (i + 1 < n0) put(idx + 1, P.inv_h2[0]);
          if (j + 1 < n1) put(idx + s1, P.inv_h2[1]);
          if (kz + 1 < n2) put(idx + s2, P.inv_h2[2]);
          rp[idx + 1] = e;
        }
  });
}

int hz_fwi_sensitivity_rhs(hz_problem* p, int64_t n, int k, const double* U, const double* v, double* R) {
  return guarded([&] {
    if (!p || !U || !v || !R) throw HzError(kValidation, "null argument");
    check_block(*p->p, n, k);
    DeviceGuard dg(p->p->device);
    DevBuf<double2> dU(size_t(n) * k), dR(size_t(n) * k);
    DevBuf<double> dv{size_t(n)};
    HZ_CUDA(cudaMemcpy(dU.get(), U, dU.bytes(), cudaMemcpyHostToDevice));
    HZ_CUDA(cudaMemcpy(dv.get(), v, dv.bytes(), cudaMemcpyHostToDevice));
    launch_sens_rhs(n, k, p->p->omega * p->p->omega, p->p->d_gf.get(), dU.get(), dv.get(), dR.get(), nullptr);
    HZ_CUDA(cudaMemcpy(R, dR.get(), dR.bytes(), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

namespace {
CycleSpec spec_from(const hz_cycle_spec* c) {
  if (!c) throw HzError(kValidation, "null cycle spec");
  if (c->kind < 0 || c->kind > 2) throw HzError(kValidation, "cycle: unknown kind");
  if (c->pre < 0 || c->post < 0 || c->k_inner < 1) throw HzError(kValidation, "cycle: bad sweep counts");
  CycleSpec sp;
  sp.kind = static_cast<CycleKind>(c->kind);
  sp.pre = c->pre;
  sp.post = c->post;
  sp.jacobi_weight = c->jacobi_weight;
  sp.k_inner = c->k_inner;
  return sp;
}
// run f with the solver's cycle spec / Krylov settings temporarily replaced
template <class F>
void with_settings(hz_solver* s, const CycleSpec& sp, bool bicg, int restart, double tol, int max_cycles, F&& f) {
  const CycleSpec sp0 = s->spec;
  const bool b0 = s->bicgstab;
  const hz_options o0 = s->opts;
  s->spec = sp;
  s->bicgstab = bicg;
  s->opts.fgmres_restart = restart;
  s->opts.tol = tol;
  s->opts.max_cycles = max_cycles;
  s->opts.rhs_block = 0;  // one block over all columns, as block_fgmres
  try {
    f();
  } catch (...) {
    s->spec = sp0;
    s->bicgstab = b0;
    s->opts = o0;
    throw;
  }
  s->spec = sp0;
  s->bicgstab = b0;
  s->opts = o0;
}
}  // namespace

extern "C" {

int hz_hierarchy_cycle(hz_solver* s, const hz_cycle_spec* spec, int64_t n, int k, const double* b, double* x,
                       int x_zero) {
  return guarded([&] {
    if (!s || !b || !x) throw HzError(kValidation, "null argument");
    if (s->dense || !s->h64) throw HzError(kState, "solver has no multigrid hierarchy");
    if (s->slabs) throw HzError(kState, "hz_hierarchy_cycle: not in slab mode");
    const CycleSpec sp = spec_from(spec);
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    s->ensure_blocks(k);
    upload_rows(s, k, b, s->dB.get());
    if (x_zero)
      HZ_CUDA(cudaMemsetAsync(s->dX.get(), 0, size_t(n) * k * sizeof(double2), s->stream));
    else
      upload_rows(s, k, x, s->dX.get());
    s->h64->cycle(sp, k, s->dB.get(), s->dX.get(), x_zero != 0, s->stream);
    download_rows(s, k, s->dX.get(), x);
  });
}

int hz_block_krylov(hz_solver* s, int method, const hz_cycle_spec* spec, int restart, double tol, int max_cycles,
                    int64_t n, int k, const double* B, double* X, hz_report* rep) {
  return guarded([&] {
    if (!s || !B || !X) throw HzError(kValidation, "null argument");
    if (s->dense || !s->h64) throw HzError(kState, "solver has no multigrid hierarchy");
    if (method != 0 && method != 1) throw HzError(kValidation, "block_krylov: method 0 (FGMRES) or 1 (BiCGSTAB)");
    if (method == 0 && restart < 1) throw HzError(kValidation, "fgmres: restart must be positive");
    const CycleSpec sp = spec_from(spec);
    check_block(*s->prob, n, k);
    DeviceGuard dg(s->prob->device);
    with_settings(s, sp, method == 1, restart, tol, max_cycles, [&] {
      s->ensure_blocks(k);
      upload_rows(s, k, B, s->dB.get());
      Report r = run_solve(s, k, s->dB.get(), s->dX.get());
      download_rows(s, k, s->dX.get(), X);
      fill_report(r, k, rep);
    });
  });
}

int64_t hz_slab_vmm_chunks(void) { return vmm_chunks_created(); }

}  // extern "C"
