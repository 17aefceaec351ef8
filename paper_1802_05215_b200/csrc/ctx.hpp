// Context: one per host thread / device stream (the reference has no equivalent: it is
// single-threaded host code; this owns what a B200 slice worker needs).
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <atomic>
#include <unordered_map>

#include "common.hpp"

namespace se {

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  long launches = 0;  // this library's kernel launches issued on `stream`

  // Filter-kernel timing (bench roofline): events bracket each filter application.
  bool time_filter = false;
  double filter_ms = 0.0;
  long filter_launches = 0;
  double filter_bytes = 0.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

Ctx* ctx_create(int device);
void ctx_destroy(Ctx* c);

// RAII device allocation on a context's device.
template <class T>
T* dev_alloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(SE_ENOMEM, std::string("device allocation of ") + std::to_string(count * sizeof(T)) +
                        " bytes failed: " + cudaGetErrorString(e));
  }
  return p;
}
inline void dev_free(void* p) {
  if (p) cudaFree(p);
}

}  // namespace se
