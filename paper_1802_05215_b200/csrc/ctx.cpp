#include "ctx.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

namespace se {

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(SE_ENOMEM, std::string("CUDA out of memory in ") + what);
  }
  fail(SE_ECUDA, std::string(cudaGetErrorString(e)) + " in " + what + " (" + file + ":" +
                     std::to_string(line) + ")");
}

namespace {
thread_local Ctx* tl_ctx = nullptr;
std::mutex pool_mu;
std::unordered_map<void*, int> pool_ptrs;  // stream-ordered allocations -> device
std::atomic<long> sync_frees{0};
std::unordered_map<const Ctx*, int> live_ctx;  // guarded by pool_mu
bool alive(const Ctx* c) { return c && live_ctx.count(c) != 0; }

[[noreturn]] void oom(size_t bytes, cudaError_t e) {
  cudaGetLastError();
  fail(SE_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
}
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}
cudaStream_t other_stream(const Ctx& c) { return c.stream == c.bulk ? c.hstream : c.bulk; }
}  // namespace

void set_current_ctx(Ctx* c) { tl_ctx = c; }
Ctx* current_ctx() { return tl_ctx; }
std::atomic<long>& dev_frees() { return sync_frees; }

void* dev_alloc_shared_bytes(size_t bytes) {
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) oom(bytes, e);
  return p;
}
void dev_free_shared(void* p) {
  if (!p) return;
  ++sync_frees;
  cudaFree(p);
}

void* dev_alloc_bytes(size_t bytes) {
  Ctx* c = tl_ctx;
  if (!c || capturing(c->stream)) return dev_alloc_shared_bytes(bytes);
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes, c->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // the pool may hold freed-but-pending blocks: wait for this context, retry once
    cudaStreamSynchronize(c->bulk);
    cudaStreamSynchronize(c->hstream);
    e = cudaMallocAsync(&p, bytes, c->stream);
    if (e != cudaSuccess) oom(bytes, e);
  }
  // usable on the context's other stream too
  SE_CUDA(cudaEventRecord(c->evx, c->stream));
  SE_CUDA(cudaStreamWaitEvent(other_stream(*c), c->evx, 0));
  std::lock_guard<std::mutex> lk(pool_mu);
  pool_ptrs.emplace(p, c->device);
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  int dev = -1;
  {
    std::lock_guard<std::mutex> lk(pool_mu);
    auto it = pool_ptrs.find(p);
    if (it != pool_ptrs.end()) {
      dev = it->second;
      pool_ptrs.erase(it);
    }
  }
  Ctx* c = tl_ctx;
  {
    std::lock_guard<std::mutex> lk(pool_mu);
    if (!alive(c)) c = nullptr;  // destroyed by another thread since it was made current
  }
  if (dev >= 0 && c && c->device == dev && !capturing(c->stream)) {
    // after everything queued on either stream of this context
    cudaEventRecord(c->evx, other_stream(*c));
    cudaStreamWaitEvent(c->stream, c->evx, 0);
    cudaFreeAsync(p, c->stream);
    return;
  }
  ++sync_frees;
  cudaFree(p);
}

void ctx_sync(Ctx& c) {
  SE_CUDA(cudaEventRecord(c.evsync, c.stream));
  SE_CUDA(cudaEventSynchronize(c.evsync));
}

void* staging(Ctx& c, size_t bytes) {
  if (bytes > c.pinned_bytes) {
    if (c.pinned) SE_CUDA(cudaFreeHost(c.pinned));
    c.pinned_bytes = std::max(bytes + bytes / 2, (size_t)1 << 20);
    SE_CUDA(cudaMallocHost(&c.pinned, c.pinned_bytes));
  }
  return c.pinned;
}

void h2d(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  void* p = staging(c, bytes);
  std::memcpy(p, src, bytes);
  SE_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, c.stream));
  ctx_sync(c);
}

void d2h(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  void* p = staging(c, bytes);
  SE_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToHost, c.stream));
  ctx_sync(c);
  std::memcpy(dst, p, bytes);
}

Ctx* ctx_create(int device) {
  int count = 0;
  SE_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) fail(SE_EINVAL, "se_ctx_create: no such CUDA device");
  SE_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  SE_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    fail(SE_ECUDA, std::string("libsliceeig_cuda is built for sm_100a (B200); device is ") + prop.name);
  auto* c = new Ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  int least = 0, greatest = 0;
  SE_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  c->prio_hi = greatest;
  c->prio_lo = least;
  SE_CUDA(cudaStreamCreateWithPriority(&c->bulk, cudaStreamNonBlocking, least));
  SE_CUDA(cudaStreamCreateWithPriority(&c->hstream, cudaStreamNonBlocking, greatest));
  c->stream = c->bulk;
  {
    std::lock_guard<std::mutex> lk(pool_mu);
    live_ctx.emplace(c, device);
  }
  {  // keep freed pool memory resident: stream-ordered reuse without returning it to the driver
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      unsigned long long keep = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) fail(SE_ECUDA, "cusolverDnCreate failed");
  cusolverDnSetStream(c->solver, c->hstream);
  SE_CUDA(cudaEventCreateWithFlags(&c->evsync, cudaEventBlockingSync | cudaEventDisableTiming));
  SE_CUDA(cudaEventCreateWithFlags(&c->evx, cudaEventDisableTiming));
  SE_CUDA(cudaEventCreate(&c->evk0));
  SE_CUDA(cudaEventCreate(&c->evk1));
  SE_CUDA(cudaEventCreate(&c->ev0));
  SE_CUDA(cudaEventCreate(&c->ev1));
  return c;
}

void ctx_destroy(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->bulk);
  cudaStreamSynchronize(c->hstream);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->evsync) cudaEventDestroy(c->evsync);
  if (c->evx) cudaEventDestroy(c->evx);
  if (tl_ctx == c) tl_ctx = nullptr;
  {
    std::lock_guard<std::mutex> lk(pool_mu);
    live_ctx.erase(c);
  }
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->bulk) cudaStreamDestroy(c->bulk);
  if (c->hstream) cudaStreamDestroy(c->hstream);
  delete c;
}

void devmat_reserve(Ctx& c, DevMat& m, int n, int cols, bool keep) {
  (void)c;
  if (m.p && m.n == n && m.cap >= cols) return;
  double* p = dev_alloc<double>((size_t)n * std::max(cols, 1));
  if (keep && m.p && m.cap > 0)
    SE_CUDA(cudaMemcpyAsync(p, m.p, sizeof(double) * (size_t)n * m.cap, cudaMemcpyDeviceToDevice,
                            c.stream));
  if (m.p) {
    ctx_sync(c);
    dev_free(m.p);
  }
  m.p = p;
  m.n = n;
  m.cap = cols;
}

void devmat_free(DevMat& m) {
  dev_free(m.p);
  m.p = nullptr;
  m.cap = 0;
}

}  // namespace se
