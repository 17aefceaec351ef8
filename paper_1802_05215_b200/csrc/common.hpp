// Internal shared declarations of libsliceeig_cuda.so (host + device).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sliceeig_cuda.h"

namespace se {

// Exceptions carrying the C-ABI status code; capi.cpp maps them to SE_* codes.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const char* msg) {
  if (!ok) fail(SE_EINVAL, msg);
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define SE_CUDA(x) ::se::cuda_check((x), #x, __FILE__, __LINE__)

// ---- device matrices -----------------------------------------------------------------------
// CSR in HBM: int32 row_ptr[n+1], int32 col_idx[nnz], f64 vals[nnz] (the reference layout,
// csr.hpp:158-162) plus a per-tile nnz table used by the row-tile SpMV.
// Rows of at most kEllW entries also get a padded copy (ell_c/ell_a, n x kEllW row-major; pad
// col = row, val = 0) that the block KPM kernel reads instead of the CSR arrays.
constexpr int kEllW = 8;

namespace k {
struct ResidentPlan;  // resident.cu: row tiles + neighbour lists of the one-launch filter
}

struct DevCsr {
  int device = 0;
  int n = 0;
  long nnz = 0;
  int* rp = nullptr;
  int* ci = nullptr;
  double* v = nullptr;
  int max_row_nnz = 0;
  int* ell_c = nullptr;     // padded copy (max_row_nnz <= kEllW), else null
  double* ell_a = nullptr;
  // residual weights w (null: none): candidates report ||w .* (A u - lambda u)|| / sqrt(u.u).
  // Set on D A D of a diagonal-B pencil with w = D^-1, which makes the residual the reference's
  // ||A x - lambda B x|| / sqrt(x' B x) for x = D u (eigensolvers.hpp:289-316)
  double* resw = nullptr;
  // plan of the resident (one launch for all degrees) filter; null when the matrix does not fit
  // in the GPU's aggregate shared memory
  k::ResidentPlan* resident = nullptr;
  // vals and col_idx live in ONE allocation (vals first, col_idx right after) so a single L2
  // access-policy window covers the whole matrix stream of the filter SpMV
  void alloc_entries(long count);
  size_t entries_bytes() const { return (((size_t)std::max(nnz, 1L) + 1) & ~(size_t)1) * 12; }
  void free_entries();
  double abytes() const { return 12.0 * (double)nnz + 4.0 * (double)(n + 1); }
};

// A growable device column-major matrix (n rows, capacity `cap` columns, ld = n).
struct DevMat {
  int n = 0;
  int cap = 0;
  double* p = nullptr;
  double* col(int j) const { return p + (size_t)j * n; }
};

void* dev_alloc_shared_bytes(size_t bytes);
void dev_free_shared(void* p);
inline void DevCsr::alloc_entries(long count) {
  const size_t c = ((size_t)std::max(count, 1L) + 1) & ~(size_t)1;  // even: col_idx 16-byte aligned
  v = static_cast<double*>(dev_alloc_shared_bytes(c * (sizeof(double) + sizeof(int)) + 16));
  ci = reinterpret_cast<int*>(v + c);
}
inline void DevCsr::free_entries() {
  dev_free_shared(v);
  v = nullptr;
  ci = nullptr;
}

struct Ctx;
void devmat_reserve(Ctx& c, DevMat& m, int n, int cols, bool keep);
void devmat_free(DevMat& m);

// Scratch allocations tied to a context (freed with it).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
};

}  // namespace se
