// Fused middle of CGS2 (orth.hpp:70-80 with the DGKS re-pass of :77): pass-1 update
// t1 = t - W c1, ||t1|| and the re-pass decision, and the pass-2 coefficients c2 = W^T t1 --
// each row block of W is read from HBM ONCE into shared memory and used for both products
// (the unfused pass reads it twice).  A CGS2 step then reads W three times instead of four:
// T1 (k_gemvt), this kernel, N2 (k_gemvn, skipped when no re-pass is needed).
//
// One 1024-thread CTA per SM owns a contiguous range of R-row blocks (R even, a power of two as
// large as a kStages-deep ring allows for the basis capacity).  Thread 0 stages each block with
// TMA (2-D tensor map over W, boxes of R rows x kBC columns) into a ring of kStages
// shared-memory stages tracked by mbarriers; while block b is reduced, blocks b+1 ..
// b+kStages-1 are in flight.  A stage holds the block as 16-byte units u = j P + p (column j,
// row pair p, P = R/2 pairs) -- the TMA box layout -- and every phase walks units linearly, so
// shared-memory accesses are bank-conflict free.  All sums run in a fixed order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

constexpr int kFT = 1024;                               // threads per CTA (one CTA per SM)
constexpr int kWarps = kFT / 32;
constexpr int kStages = 4;                              // ring depth
constexpr size_t kRing = 200 * 1024;                    // dynamic shared memory (the ring)
constexpr int kMaxR = 32;                               // rows per block cap (P <= 16 < 32)
constexpr int kBC = 64;                                 // columns per TMA box
constexpr int kMaxUnits = (int)(kRing / kStages / 16);  // 16-byte units per stage
constexpr int kOwn = (kMaxUnits + kFT - 1) / kFT;       // c2 partial units per thread

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// rows per block for a basis capacity of cap columns: a kStages ring of R x cap' doubles must
// fit (cap' = cap rounded up to whole TMA boxes)
constexpr int rows_for(int cap) {
  const int capb = (cap + kBC - 1) / kBC * kBC;
  int R = 0;
  for (int r = 2; r <= kMaxR; r *= 2)
    if ((size_t)capb * (size_t)(r / 2) <= (size_t)kMaxUnits) R = r;
  return R;
}

__global__ void __launch_bounds__(kFT, 1) k_cgs_mid(const __grid_constant__ CUtensorMap wmap, int R,
                                                    int n, double* __restrict__ t, Ctl* ctl,
                                                    const double* __restrict__ coef1,
                                                    double* c2part, int ldp, double* npart,
                                                    unsigned* cnt, double* coef2, double* hdiag) {
  if (ctl->halted) return;
  const int ncols = ctl->i + 1;
  const int P = R / 2;  // R: rows_for(capacity), the tensor map's box height
  int lp = 0;
  while ((1 << lp) < P) ++lp;
  const int units = ncols << lp;  // 16-byte units per block
  const int nbox = (ncols + kBC - 1) / kBC;
  const unsigned stage_tx = (unsigned)(nbox * kBC * R * (int)sizeof(double));
  extern __shared__ __align__(128) double2 ring[];  // [kStages][kMaxUnits]
  __shared__ __align__(8) unsigned long long full[kStages];
  __shared__ __align__(16) double2 tst[kStages][kMaxR / 2];  // the block's rows of t
  __shared__ double2 s_red[kWarps * (kMaxR / 2)];
  __shared__ double2 t1s[kMaxR / 2];
  __shared__ double s_w[kWarps];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  double acc[kOwn];
#pragma unroll
  for (int q = 0; q < kOwn; ++q) acc[q] = 0.0;
  // this thread's t1-phase coefficients (its columns are the same in every block)
  const int pme = tid & (P - 1), G = kFT >> lp;
  double cf[kOwn];
#pragma unroll
  for (int m = 0; m < kOwn; ++m) {
    const int j = (tid >> lp) + m * G;
    cf[m] = j < ncols ? __ldg(coef1 + j) : 0.0;
  }
  double nacc = 0.0;
  const int nrb = (n + R - 1) / R;
  const int b0 = (int)((long)blockIdx.x * nrb / gridDim.x);
  const int b1 = (int)((long)(blockIdx.x + 1) * nrb / gridDim.x);
  auto issue = [&](int b) {  // thread 0: stage block b with TMA (rows past n are zero-filled)
    if (b < b1) {
      const int s = (b - b0) % kStages;
      double2* st = ring + (size_t)s * kMaxUnits;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // after generic reads
      const unsigned tb = (unsigned)(min(R, n - b * R) * (int)sizeof(double));
      mbar_expect_tx(&full[s], stage_tx + tb);
      bulk_load(&tst[s][0], t + (size_t)b * R, tb, &full[s]);
      for (int c = 0; c < nbox; ++c) tma_load_2d(st + (size_t)c * kBC * P, &wmap, b * R, c * kBC, &full[s]);
    }
  };
  if (tid == 0)
    for (int s = 0; s < kStages - 1; ++s) issue(b0 + s);
  for (int b = b0; b < b1; ++b) {
    const int r0 = b * R, pn = min(R, n - r0) >> 1;  // n even -> whole pairs
    const int it = b - b0;
    __syncthreads();  // everyone is done with block b - 1 (its stage may be refilled)
    if (tid == 0) issue(b + kStages - 1);
    mbar_wait(&full[it % kStages], (unsigned)(it / kStages) & 1u);
    const double2* st = ring + (size_t)(it % kStages) * kMaxUnits;
    // t1 = t - W c1 on the block rows: thread (pair p, group g) sums columns g, g + G, ...
    {
      const int p = pme;
      double p0 = 0.0, p1 = 0.0;
      if (p < pn) {
#pragma unroll
        for (int m = 0; m < kOwn; ++m) {
          const int j = (tid >> lp) + m * G;
          if (j < ncols) {
            const double2 w = st[(j << lp) + p];
            p0 = add(p0, mul(cf[m], w.x));
            p1 = add(p1, mul(cf[m], w.y));
          }
        }
      }
      for (int o = 16; o >= P; o >>= 1) {  // lanes sharing p
        p0 = add(p0, __shfl_xor_sync(0xffffffffu, p0, o));
        p1 = add(p1, __shfl_xor_sync(0xffffffffu, p1, o));
      }
      if (lane < P) s_red[warp * P + lane] = make_double2(p0, p1);
    }
    __syncthreads();
    if (warp < pn) {  // warp p combines the kWarps partials of pair p
      const double2 v = s_red[lane * P + warp];
      const double s0 = warp_sum(v.x), s1 = warp_sum(v.y);
      if (lane == 0) {
        double2* tp = reinterpret_cast<double2*>(t + r0) + warp;
        const double2 tv = tst[it % kStages][warp];
        const double2 x = make_double2(sub(tv.x, s0), sub(tv.y, s1));
        *tp = x;
        t1s[warp] = x;
        nacc = add(nacc, mul(x.x, x.x));
        nacc = add(nacc, mul(x.y, x.y));
      }
    }
    __syncthreads();
    // c2 partials per unit (column j, pair p): thread owns units tid + q kFT
#pragma unroll
    for (int q = 0; q < kOwn; ++q) {
      const int u = tid + q * kFT;
      if (u < units && (u & (P - 1)) < pn) {
        const double2 w = st[u], y = t1s[u & (P - 1)];
        acc[q] = add(add(acc[q], mul(w.x, y.x)), mul(w.y, y.y));
      }
    }
  }
  __syncthreads();
  // per-CTA c2 partials: combine the P pair partials of each column in pair order
  double* su = reinterpret_cast<double*>(ring);
#pragma unroll
  for (int q = 0; q < kOwn; ++q) {
    const int u = tid + q * kFT;
    if (u < units) su[u] = acc[q];
  }
  __syncthreads();
  for (int j = tid; j < ncols; j += kFT) {
    double a = 0.0;
    for (int p = 0; p < P; ++p) a = add(a, su[(j << lp) + p]);
    c2part[(size_t)blockIdx.x * ldp + j] = a;
  }
  {
    const double v = warp_sum(nacc);
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
      const double u = warp_sum(s_w[lane]);
      if (lane == 0) npart[blockIdx.x] = u;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: c2 = sum of partials in CTA order; ||t1||; DGKS decision (orth.hpp:76-78)
  __shared__ int s_repass;
  if (warp == 0) {
    double u = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) u = add(u, __ldcg(npart + b));
    u = warp_sum(u);
    if (lane == 0) {
      const double after = sqrt(u);
      const int rep = after > 0.70710678118654752 * ctl->before ? 0 : 1;
      s_repass = rep;
      ctl->npass += 1;
      ctl->passes_total += 1;
      ctl->repass = rep;
      ctl->before = after;
      ctl->after = after;
      *cnt = 0u;
    }
  }
  __syncthreads();
  const int hcol = hdiag ? ctl->i : -1;
  for (int j = tid; j < ncols; j += kFT) {
    double u = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) u = add(u, __ldcg(c2part + (size_t)b * ldp + j));
    coef2[j] = u;
    if (j == hcol && s_repass) hdiag[j] = add(hdiag[j], u);  // h[i] += c2_i (orth.hpp:30)
  }
}

// L2 two-read variant (SE_CGS_FUSED=2): no shared-memory staging of W.  A CTA (32 warps) walks
// its contiguous range of 32-row blocks; per block, phase 1 streams W[rows, :] from HBM (warp w
// takes columns w, w + 32, ...; lane = row, so every load is one 256-byte column segment) and
// forms t1 = t - W c1; phase 2 re-reads the same block -- still in L2: the blocks in flight across
// the grid are grid x 32 x ncols x 8 bytes -- and adds W[rows, j]^T t1[rows] to the CTA's c2
// accumulator of column j (owned by one warp, summed in block order).  Same tail as k_cgs_mid.
constexpr int kL2Rows = 32;
constexpr int kL2Warps = 32;
constexpr int kL2Unroll = 8;

__global__ void __launch_bounds__(kL2Warps * 32) k_cgs_mid_l2(int n, const double* __restrict__ Q,
                                                                double* __restrict__ t, Ctl* ctl,
                                                                const double* __restrict__ coef1,
                                                                double* c2part, int ldp, double* npart,
                                                                unsigned* cnt, double* coef2, double* hdiag) {
  if (ctl->halted) return;
  const int ncols = ctl->i + 1;
  extern __shared__ double smem_l2[];
  double* s_c1 = smem_l2;                 // ncols
  double* s_acc = smem_l2 + ldp;          // ncols: this CTA's c2 partials
  __shared__ double s_red[kL2Warps][kL2Rows + 1];
  __shared__ double s_t1[kL2Rows];
  __shared__ double s_w[kL2Warps];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = (int)(blockDim.x >> 5);  // warps (column stride)
  for (int j = tid; j < ncols; j += blockDim.x) {
    s_c1[j] = __ldg(coef1 + j);
    s_acc[j] = 0.0;
  }
  __syncthreads();
  double nacc = 0.0;
  const int nrb = (n + kL2Rows - 1) / kL2Rows;
  const int b0 = (int)((long)blockIdx.x * nrb / gridDim.x);
  const int b1 = (int)((long)(blockIdx.x + 1) * nrb / gridDim.x);
  for (int b = b0; b < b1; ++b) {
    const int r = b * kL2Rows + lane;
    const bool live = r < n;
    const double* __restrict__ qr = Q + r;
    // phase 1: partial (W c1)[r] over this warp's columns
    double p = 0.0;
    {
      int j = warp;
      for (; j + (kL2Unroll - 1) * NW < ncols; j += kL2Unroll * NW) {
        double w[kL2Unroll];
#pragma unroll
        for (int u = 0; u < kL2Unroll; ++u) w[u] = live ? __ldg(qr + (size_t)(j + u * NW) * n) : 0.0;
#pragma unroll
        for (int u = 0; u < kL2Unroll; ++u) p = add(p, mul(s_c1[j + u * NW], w[u]));
      }
      for (; j < ncols; j += NW) p = add(p, mul(s_c1[j], live ? __ldg(qr + (size_t)j * n) : 0.0));
    }
    s_red[warp][lane] = p;
    __syncthreads();
    if (warp == 0) {
      double sum = 0.0;
      for (int q = 0; q < NW; ++q) sum = add(sum, s_red[q][lane]);
      double x = 0.0;
      if (live) {
        x = sub(t[r], sum);
        t[r] = x;
      }
      s_t1[lane] = x;
      nacc = add(nacc, mul(x, x));
    }
    __syncthreads();
    // phase 2: c2[j] += W[rows, j] . t1[rows]  (L2 re-read)
    const double tv = s_t1[lane];
    int j = warp;
    for (; j + (kL2Unroll - 1) * NW < ncols; j += kL2Unroll * NW) {
      double v[kL2Unroll];
#pragma unroll
      for (int u = 0; u < kL2Unroll; ++u) v[u] = live ? mul(__ldg(qr + (size_t)(j + u * NW) * n), tv) : 0.0;
      // butterfly multi-reduction of the 32 x 8 products: at lane bits 4 / 3 / 2 each lane keeps
      // half of its columns and receives its partner's other half (4 + 2 + 1 exchanges), then
      // two plain xor steps; lane L ends with the full sum of column 4 b4 + 2 b3 + b2
      const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double send = h4 ? v[k] : v[k + 4];
        const double keep = h4 ? v[k + 4] : v[k];
        v[k] = add(keep, __shfl_xor_sync(0xffffffffu, send, 16));
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double send = h3 ? v[k] : v[k + 2];
        const double keep = h3 ? v[k + 2] : v[k];
        v[k] = add(keep, __shfl_xor_sync(0xffffffffu, send, 8));
      }
      {
        const double send = h2 ? v[0] : v[1];
        const double keep = h2 ? v[1] : v[0];
        v[0] = add(keep, __shfl_xor_sync(0xffffffffu, send, 4));
      }
      v[0] = add(v[0], __shfl_xor_sync(0xffffffffu, v[0], 2));
      v[0] = add(v[0], __shfl_xor_sync(0xffffffffu, v[0], 1));
      if ((lane & 3) == 0) {
        const int col = j + ((h4 ? 4 : 0) + (h3 ? 2 : 0) + (h2 ? 1 : 0)) * NW;
        s_acc[col] = add(s_acc[col], v[0]);
      }
    }
    for (; j < ncols; j += NW) {
      double v = live ? mul(__ldg(qr + (size_t)j * n), tv) : 0.0;
      for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) s_acc[j] = add(s_acc[j], v);
    }
  }
  __syncthreads();
  for (int j = tid; j < ncols; j += blockDim.x) c2part[(size_t)blockIdx.x * ldp + j] = s_acc[j];
  if (warp == 0) {
    const double v = warp_sum(nacc);
    if (lane == 0) npart[blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ int s_repass;
  if (warp == 0) {
    double u = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) u = add(u, __ldcg(npart + b));
    u = warp_sum(u);
    if (lane == 0) {
      const double after = sqrt(u);
      const int rep = after > 0.70710678118654752 * ctl->before ? 0 : 1;
      s_repass = rep;
      ctl->npass += 1;
      ctl->passes_total += 1;
      ctl->cols_total += ncols;
      ctl->repass = rep;
      ctl->before = after;
      ctl->after = after;
      *cnt = 0u;
    }
  }
  (void)s_w;
  __syncthreads();
  const int hcol = hdiag ? ctl->i : -1;
  for (int j = tid; j < ncols; j += blockDim.x) {
    double u = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) u = add(u, __ldcg(c2part + (size_t)b * ldp + j));
    coef2[j] = u;
    if (j == hcol && s_repass) hdiag[j] = add(hdiag[j], u);  // h[i] += c2_i (orth.hpp:30)
  }
}

}  // namespace

size_t cgs_mid_scratch_doubles(const Ctx& c, int cap_cols) {
  const size_t grid = (size_t)c.num_sms * 4;
  return grid * (size_t)std::max(cap_cols, 1) + grid + 64;
}

bool cgs_mid_l2();
bool cgs_mid_supported(int n, int cap_cols) {
  if (cgs_mid_l2()) return cap_cols <= 12800;
  return n % 2 == 0 && cap_cols <= kMaxFusedCols && rows_for(cap_cols) >= 2;
}

namespace {
PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    SE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(SE_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}
}  // namespace

bool cgs_mid_l2() {
  static const bool v = [] {
    const char* e = std::getenv("SE_CGS_FUSED");
    return e && std::atoi(e) == 2;
  }();
  return v;
}

void cgs_mid(Ctx& c, int n, double* t, const double* Q, Ctl* ctl, const double* coef1,
             double* coef2, double* hdiag, int cap, double* scratch, unsigned* cnt) {
  if (cgs_mid_l2()) {
    const size_t smem = sizeof(double) * 2 * (size_t)std::max(cap, 1);
    static thread_local bool attr2 = false;
    if (!attr2) {
      SE_CUDA(cudaFuncSetAttribute(k_cgs_mid_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr2 = true;
    }
    if (smem > 200 * 1024) fail(SE_EINVAL, "cgs_mid: basis too wide for the fused path");
    static const int cps = [] {  // CTAs per SM (SE_MID_CPS): 1 x 1024, 2 x 512, 4 x 256 threads
      const char* e = std::getenv("SE_MID_CPS");
      const int v = e ? std::atoi(e) : 1;
      return v == 2 || v == 4 ? v : 1;
    }();
    const int grid = c.num_sms * cps;
    k_cgs_mid_l2<<<grid, kL2Warps * 32 / cps, smem, c.stream>>>(n, Q, t, ctl, coef1, scratch, cap,
                                                          scratch + (size_t)grid * cap, cnt, coef2, hdiag);
    ++c.launches;
    SE_CUDA(cudaGetLastError());
    return;
  }
  static thread_local bool attr = false;
  if (!attr) {
    SE_CUDA(cudaFuncSetAttribute(k_cgs_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRing));
    attr = true;
  }
  if (!cgs_mid_supported(n, cap)) fail(SE_EINVAL, "cgs_mid: basis too wide for the fused path");
  const int R = rows_for(cap);
  // W as a 2-D tensor: dim 0 = rows (n, contiguous), dim 1 = columns (cap, stride n doubles)
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)cap};
  const cuuint64_t strides[1] = {(cuuint64_t)n * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)kBC};
  const cuuint32_t estr[2] = {1, 1};
  static const CUtensorMapL2promotion promo = [] {
    const char* e = std::getenv("SE_MID_L2PROMO");
    const int v = e ? std::atoi(e) : 3;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
           : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                    : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(Q), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SE_ECUDA, "cgs_mid: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  const int grid = c.num_sms;
  double* c2part = scratch;
  double* npart = scratch + (size_t)grid * cap;
  k_cgs_mid<<<grid, kFT, kRing, c.stream>>>(map, R, n, t, ctl, coef1, c2part, cap, npart, cnt, coef2,
                                            hdiag);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

}  // namespace k
}  // namespace se
