// Persistent filter kernel for matrices whose CSR fits in the GPU's aggregate shared memory
// (BASELINE cfg1 and cfg2: A = 0.6 / 22.8 MB): one cooperative CTA per SM owns a contiguous,
// nnz-balanced row range, stages its slice of A into shared memory ONCE, and then runs all k
// degrees of the Chebyshev recurrence (filter_poly.hpp:256-277) with a grid barrier between
// degrees.  Per degree only the vector gathers and row-local streams touch L2 -- A is never
// re-read -- and the k-1 kernel launch gaps disappear.  Row sums, map and recurrence use the
// same individually rounded operations as k_spmv_cheb, so the result is bit-identical.
#include <cooperative_groups.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace se {
namespace k {

namespace {

constexpr int kPThreads = 1024;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

struct PArgs {
  const double* v;
  const Ctl* src_ctl;
  long src_ld;
  const Ctl* halt;
  double* out;
  double* b0;
  double* b1;
  double* b2;
  const double* mu;  // device, k+1 values
  int k;
  double c, invd;
};

__global__ void __launch_bounds__(kPThreads, 1) k_filter_persist(int n, const int* __restrict__ rp,
                                                                 const int* __restrict__ ci,
                                                                 const double* __restrict__ vals,
                                                                 const int* __restrict__ part,
                                                                 PArgs a) {
  if (a.halt && a.halt->halted) return;  // grid-uniform
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  const int R0 = part[blockIdx.x], R1 = part[blockIdx.x + 1];
  const int base = __ldg(rp + R0), end = __ldg(rp + R1);
  const int rows = R1 - R0, nz = end - base;
  // layout: vals (8-aligned, starting at the even-aligned base), cols (4-aligned), row offsets
  const int va = base & ~1, ca = base & ~3;
  const int nv16 = (end - va + 1) >> 1, nc16 = (end - ca + 3) >> 2;
  double* s_v = reinterpret_cast<double*>(smem);
  int* s_c = reinterpret_cast<int*>(smem + sizeof(double) * 2 * nv16);
  int* s_rp = s_c + 4 * nc16;
  for (int q = threadIdx.x; q < nv16; q += kPThreads)
    cp_async16(&s_v[2 * q], vals + va + 2 * q, 8 * min(2, end - (va + 2 * q)));
  for (int q = threadIdx.x; q < nc16; q += kPThreads)
    cp_async16(&s_c[4 * q], ci + ca + 4 * q, 4 * min(4, end - (ca + 4 * q)));
  for (int q = threadIdx.x; q <= rows; q += kPThreads) cp_async4(&s_rp[q], rp + R0 + q);
  cp_async_wait_all();
  __syncthreads();
  (void)nz;
  const double* __restrict__ V = a.v + (a.src_ctl ? (size_t)a.src_ctl->i * a.src_ld : 0);
  double* B[3] = {a.b0, a.b1, a.b2};
  for (int j = 1; j <= a.k; ++j) {
    const double* __restrict__ x = j == 1 ? V : B[(j - 2) % 3];
    const double* __restrict__ prev = j == 2 ? V : B[(j + 0) % 3];  // B[(j-3)%3] for j >= 3
    double* __restrict__ y = B[(j - 1) % 3];
    const double muj = a.mu[j];
    for (int lr = threadIdx.x; lr < rows; lr += kPThreads) {
      const int r = R0 + lr;
      const int s = s_rp[lr] - va, e = s_rp[lr + 1] - va, cs = s_rp[lr] - ca;
      double acc = 0.0;
      for (int p = 0; p < e - s; p += 8) {
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = (p + u < e - s) ? __ldcg(x + s_c[cs + p + u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p + u < e - s) acc = add(acc, mul(s_v[s + p + u], xv[u]));
      }
      const double xr = __ldcg(x + r);
      const double t = mul(sub(acc, mul(a.c, xr)), a.invd);
      if (j == 1) {
        y[r] = t;
        a.out[r] = add(add(0.0, mul(a.mu[0], xr)), mul(muj, t));
      } else {
        const double tj = sub(mul(2.0, t), __ldcg(prev + r));
        y[r] = tj;
        a.out[r] = add(a.out[r], mul(muj, tj));
      }
    }
    if (j < a.k) grid.sync();
  }
}

}  // namespace

size_t persist_smem_bytes(int part_nnz_max, int part_rows_max) {
  return sizeof(double) * (size_t)(part_nnz_max + 4) + sizeof(int) * (size_t)(part_nnz_max + 8) +
         sizeof(int) * (size_t)(part_rows_max + 2);
}

bool persist_eligible(const Ctx& c, const DevCsr& a) {
  return a.part != nullptr && a.nparts == c.num_sms &&
         persist_smem_bytes(a.part_nnz_max, a.part_rows_max) <= (size_t)200 * 1024;
}

void filter_persist(Ctx& c, const DevCsr& a, const double* v, const Ctl* src_ctl, long src_ld,
                    const Ctl* halt, double* out, double* const* bufs, const double* mu_dev,
                    int kdeg, double cc, double invd) {
  PArgs p{v, src_ctl, src_ld, halt, out, bufs[0], bufs[1], bufs[2], mu_dev, kdeg, cc, invd};
  const size_t smem = persist_smem_bytes(a.part_nnz_max, a.part_rows_max);
  static thread_local bool attr = false;
  if (!attr) {
    SE_CUDA(cudaFuncSetAttribute(k_filter_persist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024));
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nparts);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  SE_CUDA(cudaLaunchKernelEx(&cfg, k_filter_persist, a.n, (const int*)a.rp, (const int*)a.ci,
                             (const double*)a.v, (const int*)a.part, p));
  ++c.launches;
}

// nnz-balanced contiguous row partition into c.num_sms parts (host rp)
void build_partition(Ctx& c, DevCsr& a, const int* rp_host) {
  const int P = c.num_sms;
  std::vector<int> part(P + 1, 0);
  const long nnz = rp_host[a.n];
  int r = 0;
  for (int q = 1; q < P; ++q) {
    const long target = nnz * q / P;
    while (r < a.n && rp_host[r] < target) ++r;
    part[q] = r;
  }
  part[P] = a.n;
  int mx_nz = 0, mx_rows = 0;
  for (int q = 0; q < P; ++q) {
    if (part[q + 1] < part[q]) part[q + 1] = part[q];
    mx_nz = std::max(mx_nz, rp_host[part[q + 1]] - rp_host[part[q]]);
    mx_rows = std::max(mx_rows, part[q + 1] - part[q]);
  }
  int t32 = 0;
  for (long r0 = 0; r0 < a.n; r0 += 32) t32 = std::max(t32, rp_host[std::min<long>(r0 + 32, a.n)] - rp_host[r0]);
  a.tile32_nnz_max = t32;
  a.part = dev_alloc_shared<int>(P + 1);
  h2d(c, a.part, part.data(), sizeof(int) * (P + 1));
  a.nparts = P;
  a.part_nnz_max = mx_nz;
  a.part_rows_max = mx_rows;
}

}  // namespace k
}  // namespace se
