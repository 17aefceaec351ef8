#include "ctx.hpp"

#include <algorithm>
#include <cstring>
#include <string>

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
  SE_CUDA(cudaStreamCreateWithPriority(&c->bulk, cudaStreamNonBlocking, least));
  SE_CUDA(cudaStreamCreateWithPriority(&c->hstream, cudaStreamNonBlocking, greatest));
  c->stream = c->bulk;
  if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) fail(SE_ECUDA, "cublasCreate failed");
  cublasSetStream(c->blas, c->hstream);
  if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) fail(SE_ECUDA, "cusolverDnCreate failed");
  cusolverDnSetStream(c->solver, c->hstream);
  SE_CUDA(cudaEventCreateWithFlags(&c->evsync, cudaEventBlockingSync | cudaEventDisableTiming));
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
  if (c->blas) cublasDestroy(c->blas);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->evsync) cudaEventDestroy(c->evsync);
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
