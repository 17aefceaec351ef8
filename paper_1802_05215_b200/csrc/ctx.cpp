#include "ctx.hpp"

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
  SE_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) fail(SE_ECUDA, "cublasCreate failed");
  cublasSetStream(c->blas, c->stream);
  if (cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS) fail(SE_ECUDA, "cusolverDnCreate failed");
  cusolverDnSetStream(c->solver, c->stream);
  SE_CUDA(cudaEventCreate(&c->ev0));
  SE_CUDA(cudaEventCreate(&c->ev1));
  return c;
}

void ctx_destroy(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->blas) cublasDestroy(c->blas);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
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
    SE_CUDA(cudaStreamSynchronize(c.stream));
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
