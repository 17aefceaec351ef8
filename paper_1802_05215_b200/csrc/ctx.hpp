// Context: one per host thread / device stream (the reference has no equivalent: it is
// single-threaded host code; this owns what a B200 slice worker needs).
#pragma once

#include <cusolverDn.h>

#include <atomic>
#include <unordered_map>

#include "common.hpp"

namespace se {

struct Ctx {
  int device = 0;
  int num_sms = 148;
  int prio_hi = 0, prio_lo = 0;  // stream/kernel priority range of the device
  cudaStream_t stream = nullptr;   // current launch stream (bulk Lanczos work: low priority)
  cudaStream_t bulk = nullptr;     // the low-priority stream
  cudaStream_t hstream = nullptr;  // high priority: latency-bound host-driven phases
  cusolverDnHandle_t solver = nullptr;
  long launches = 0;  // this library's kernel launches issued on `stream`
  // device bytes the Ritz-candidate evaluation (U = W Y and A U) may hold at once; larger
  // candidate sets are evaluated in column chunks (se_ctx_set_candidate_budget)
  size_t cand_budget = (size_t)8 << 30;

  // Filter-kernel timing (bench roofline): events bracket each filter application.
  bool time_filter = false;
  double filter_ms = 0.0;
  long filter_launches = 0;
  double filter_bytes = 0.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evsync = nullptr;
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;  // profiling of host-driven phases
  cudaEvent_t evx = nullptr;                    // cross-stream ordering of allocations
  double prof_kernel_ms = 0.0;
  double prof_chk[3] = {0, 0, 0};  // stagnation check: h2d, kernel + count, d2h (host seconds)
  void* pinned = nullptr;  // staging for host<->device copies (pageable copies serialise
  size_t pinned_bytes = 0; // across the slice threads sharing a GPU)  // blocking-sync event: host waits sleep instead of spinning
};

// Route this context's launches to the high-priority stream for a scope (projected eigensolves,
// stagnation checks, Ritz extraction): with 8 slices sharing a GPU these short, synchronising
// phases otherwise queue behind other slices' bandwidth-bound reorthogonalisation kernels.
struct HiPrio {  // nests: restores whichever stream was current
  Ctx& c;
  cudaStream_t prev;
  explicit HiPrio(Ctx& cc) : c(cc), prev(cc.stream) { c.stream = c.hstream; }
  ~HiPrio() { c.stream = prev; }
};

// Wait for the work queued on the context's current stream (the host thread blocks instead of
// spin-polling, so the slice threads sharing a GPU leave the host cores to each other).
void ctx_sync(Ctx& c);
// Synchronous host<->device copies through the context's pinned staging buffer.
void h2d(Ctx& c, void* dst, const void* src, size_t bytes);
void* staging(Ctx& c, size_t bytes);  // the pinned staging buffer (>= bytes)
void d2h(Ctx& c, void* dst, const void* src, size_t bytes);

Ctx* ctx_create(int device);
void ctx_destroy(Ctx* c);

// ---- device memory -------------------------------------------------------------------------
// dev_alloc / dev_free are stream-ordered (cudaMallocAsync / cudaFreeAsync from the device's
// memory pool, kept resident) on the calling thread's current context, ordered against both of
// its streams with events: no device-wide synchronisation, so one slice thread's allocations do
// not stall the other slices sharing the GPU (cudaFree waits for the whole device).  Without a
// current context (or inside a stream capture) they fall back to cudaMalloc / cudaFree.
// Memory several contexts read (a CSR matrix) comes from dev_alloc_shared / dev_free_shared.
void set_current_ctx(Ctx* c);
Ctx* current_ctx();
void* dev_alloc_bytes(size_t bytes);
void dev_free(void* p);
void* dev_alloc_shared_bytes(size_t bytes);
void dev_free_shared(void* p);
std::atomic<long>& dev_frees();  // synchronising frees (SE_PROFILE)

template <class T>
T* dev_alloc(size_t count) {
  return static_cast<T*>(dev_alloc_bytes((count ? count : 1) * sizeof(T)));
}
template <class T>
T* dev_alloc_shared(size_t count) {
  return static_cast<T*>(dev_alloc_shared_bytes((count ? count : 1) * sizeof(T)));
}

}  // namespace se
