// Resident Chebyshev filter: all k degrees of apply_pol (filter_poly.hpp:256-277) in ONE launch,
// for matrices whose CSR arrays fit in the GPU's aggregate shared memory (148 x ~190 KB = 28 MB:
// BASELINE cfg1 and cfg2; n <= ~300k rows).
//
// Why: on such a matrix one filter degree moves ~33 MB that is L2-resident, and a chain of k
// dependent launches costs 4.2-4.5 us per degree however the launches are issued -- a third of
// the cfg2 solve.  Here the matrix is read ONCE per filter application: every CTA copies the CSR
// rows of its own row tile into shared memory and keeps them there for all k degrees, together
// with its tile of the current Chebyshev vector (double-buffered), while the previous vector, the
// current vector and the running sum out = sum_j mu_j T_j v of its own rows live in registers.
// Per degree a CTA only exchanges vector entries with the tiles its columns reach: it writes its
// new tile to a global (L2) buffer, publishes its degree counter with a release store, and polls
// the counters of its neighbour tiles with acquire loads before gathering their entries -- a
// dataflow hand-off between neighbouring tiles (2 of a 7-point stencil's 7 gathers leave the
// tile) instead of a grid-wide barrier or a kernel boundary.
//
// Safety: the launch is cooperative (all CTAs co-resident by construction), the wait is bounded
// (a stuck neighbour traps instead of hanging the device), and the write-after-read hazard of
// the three rotating exchange buffers is covered by the same wait because the neighbour relation
// is symmetrised when the plan is built.
//
// Numerics: per row exactly the arithmetic of k_spmv_cheb (storage-order sums of individually
// rounded products, the same map and recurrence), so the result is bit-identical to the
// per-degree kernels and to the reference's scalar loops.
#include <algorithm>
#include <atomic>
#include <vector>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ long long ld_acquire(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

struct ResArgs {
  int n, tile_rows, kdeg;
  const int* rp;
  const int* ci;
  const double* v;
  const int* nbr_ptr;
  const int* nbr;
  const double* x;    // input vector (contiguous)
  double* out;        // sum_j mu_j T_j x
  double* buf[3];     // exchange buffers (n doubles each)
  const double* mu;   // k + 1 coefficients (device)
  double c, invd;
  long long* flags;   // one degree counter per tile (monotone across launches)
  const Ctl* halt;
  int cap_nnz;        // shared-memory capacity of a tile's entries
};

constexpr long long kSpinLimit = 1ll << 24;

// RPT rows per thread; T threads per CTA (blockDim.x).
template <int RPT>
__global__ void __launch_bounds__(1024, 1) k_cheb_resident(ResArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = blockDim.x, tid = threadIdx.x;
  const int b = blockIdx.x;
  const int r0 = b * a.tile_rows;
  const int rows = min(a.tile_rows, a.n - r0);
  double* s_val = reinterpret_cast<double*>(smem_raw);
  double* s_x = s_val + a.cap_nnz;                         // [2][tile_rows]
  int* s_col = reinterpret_cast<int*>(s_x + 2 * a.tile_rows);
  int* s_rp = s_col + a.cap_nnz;                           // tile_rows + 1, rebased
  // the tile's matrix rows: independent of the previous kernel (fetched before the PDL wait)
  const int base = __ldg(a.rp + r0);
  const int nnzt = __ldg(a.rp + r0 + rows) - base;
  for (int p = tid; p < nnzt; p += T) {
    s_val[p] = __ldg(a.v + base + p);
    s_col[p] = __ldg(a.ci + base + p);
  }
  for (int q = tid; q <= rows; q += T) s_rp[q] = __ldg(a.rp + r0 + q) - base;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (a.halt && a.halt->halted) return;
  const long long f0 = ld_acquire(a.flags + b);  // every tile ended the last launch at this value
  const int nb0 = a.nbr_ptr[b], nb1 = a.nbr_ptr[b + 1];

  double prev[RPT], cur[RPT], acc_out[RPT];
  int ps[RPT], pe[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = tid + q * T;
    const bool live = lr < rows;
    prev[q] = live ? __ldg(a.x + r0 + lr) : 0.0;
    cur[q] = 0.0;
    acc_out[q] = 0.0;
    if (live) s_x[lr] = prev[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = tid + q * T;
    ps[q] = lr < rows ? s_rp[lr] : 0;
    pe[q] = lr < rows ? s_rp[lr + 1] : 0;
  }

  // row sum of A times the vector whose own tile is sx (shared) and whose other entries are in
  // g (global: the input vector through the read-only path, exchange buffers through L2)
  auto row_sum = [&](int q, const double* sx, const double* g, bool readonly) {
    double acc = 0.0;
    for (int p = ps[q]; p < pe[q]; p += 8) {
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = 0.0;
        if (p + u < pe[q]) {
          const int col = s_col[p + u];
          const unsigned off = (unsigned)(col - r0);
          xv[u] = off < (unsigned)rows ? sx[off] : (readonly ? __ldg(g + col) : __ldcg(g + col));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < pe[q]) acc = add(acc, mul(s_val[p + u], xv[u]));
    }
    return acc;
  };
  auto publish = [&](long long value) {
    __syncthreads();  // every thread's exchange stores are issued; s_x hand-over
    if (tid == 0) {
      __threadfence();
      st_release(a.flags + b, value);
    }
  };
  auto wait_neighbours = [&](long long value) {
    if (tid < 32) {
      for (int q = nb0 + tid; q < nb1; q += 32) {
        const long long* f = a.flags + a.nbr[q];
        long long spins = 0;
        while (ld_acquire(f) < value)
          if (++spins > kSpinLimit) __trap();  // a neighbour never arrived: fail, do not hang
      }
    }
    __syncthreads();
  };

  // degree 1: T_1 = Ahat x; out = mu0 x + mu1 T_1   (filter_poly.hpp:260-269)
  {
    const double mu0 = __ldg(a.mu), mu1 = __ldg(a.mu + 1);
    double* dst = a.buf[1];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(q, s_x, a.x, true), mul(a.c, prev[q])), a.invd);
      cur[q] = t;
      acc_out[q] = add(add(0.0, mul(mu0, prev[q])), mul(mu1, t));
      if (a.kdeg > 1) {
        __stcg(dst + r0 + lr, t);
        s_x[a.tile_rows + lr] = t;
      }
    }
    publish(f0 + 1);
  }
  // degrees 2..k: T_j = 2 Ahat T_{j-1} - T_{j-2}; out += mu_j T_j   (filter_poly.hpp:270-276)
  for (int j = 2; j <= a.kdeg; ++j) {
    wait_neighbours(f0 + j - 1);
    const double muj = __ldg(a.mu + j);
    const double* src = a.buf[(j - 1) % 3];
    double* dst = a.buf[j % 3];
    const double* sx = s_x + ((j - 1) & 1) * a.tile_rows;
    double* sxn = s_x + (j & 1) * a.tile_rows;
    const bool more = j < a.kdeg;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(q, sx, src, false), mul(a.c, cur[q])), a.invd);
      const double tj = sub(mul(2.0, t), prev[q]);
      acc_out[q] = add(acc_out[q], mul(muj, tj));
      prev[q] = cur[q];
      cur[q] = tj;
      if (more) {
        __stcg(dst + r0 + lr, tj);
        sxn[lr] = tj;
      }
    }
    publish(f0 + j);
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = tid + q * T;
    if (lr < rows) a.out[r0 + lr] = acc_out[q];
  }
}

// per tile: smallest and largest column index of its rows
__global__ void k_tile_col_span(int n, int tile_rows, const int* __restrict__ rp,
                                const int* __restrict__ ci, int* __restrict__ span) {
  const int b = blockIdx.x;
  const int r0 = b * tile_rows, r1 = min(n, r0 + tile_rows);
  int lo = n, hi = -1;
  for (int p = rp[r0] + threadIdx.x; p < rp[r1]; p += blockDim.x) {
    const int c = ci[p];
    lo = min(lo, c);
    hi = max(hi, c);
  }
  __shared__ int s_lo[256], s_hi[256];
  s_lo[threadIdx.x] = lo;
  s_hi[threadIdx.x] = hi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s_lo[threadIdx.x] = min(s_lo[threadIdx.x], s_lo[threadIdx.x + o]);
      s_hi[threadIdx.x] = max(s_hi[threadIdx.x], s_hi[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    span[2 * b] = s_lo[0];
    span[2 * b + 1] = s_hi[0];
  }
}

size_t res_smem_bytes(int tile_rows, int cap_nnz) {
  return (size_t)cap_nnz * 12 + (size_t)tile_rows * 16 + (size_t)(tile_rows + 1) * 4 + 16;
}

}  // namespace

// The plan of a matrix: row tiles (one per CTA), per-tile entry capacity, neighbour lists.
struct ResidentPlan {
  int nct = 0, tile_rows = 0, threads = 0, rpt = 0, cap_nnz = 0;
  size_t smem = 0;
  int* nbr_ptr = nullptr;  // device
  int* nbr = nullptr;      // device
};

void resident_free(DevCsr& a) {
  if (!a.resident) return;
  dev_free_shared(a.resident->nbr_ptr);
  dev_free_shared(a.resident->nbr);
  delete a.resident;
  a.resident = nullptr;
}

// Build (or rebuild) the plan after the pattern is in place; leaves a.resident null when the
// matrix does not fit (the per-degree kernels then run).
void resident_build(Ctx& c, DevCsr& a) {
  resident_free(a);
  if (a.n <= 0 || a.nnz <= 0) return;
  int dev = 0, max_optin = 0, coop = 0;
  SE_CUDA(cudaGetDevice(&dev));
  SE_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  SE_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return;
  int tile_rows = std::max((a.n + c.num_sms - 1) / c.num_sms, 128);
  tile_rows = (tile_rows + 31) / 32 * 32;
  if (tile_rows > 2048) return;
  const int nct = (a.n + tile_rows - 1) / tile_rows;
  const int threads = tile_rows > 512 ? 1024 : (tile_rows > 256 ? 512 : 256);
  const int rpt = (tile_rows + threads - 1) / threads;
  // per-tile entry counts and column spans
  std::vector<int> rp_tiles(nct + 1);
  for (int b = 0; b <= nct; ++b)
    SE_CUDA(cudaMemcpyAsync(&rp_tiles[b], a.rp + std::min(a.n, b * tile_rows), sizeof(int),
                            cudaMemcpyDeviceToHost, c.stream));
  int* dspan = dev_alloc<int>(2 * (size_t)nct);
  k_tile_col_span<<<nct, 256, 0, c.stream>>>(a.n, tile_rows, a.rp, a.ci, dspan);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
  std::vector<int> span(2 * (size_t)nct);
  SE_CUDA(cudaMemcpyAsync(span.data(), dspan, sizeof(int) * span.size(), cudaMemcpyDeviceToHost,
                          c.stream));
  ctx_sync(c);
  dev_free(dspan);
  int cap = 0;
  for (int b = 0; b < nct; ++b) cap = std::max(cap, rp_tiles[b + 1] - rp_tiles[b]);
  cap = (cap + 1) & ~1;
  const size_t smem = res_smem_bytes(tile_rows, cap);
  if (smem > (size_t)max_optin) return;
  // neighbour tiles: every tile whose rows my columns reach, symmetrised (the write-after-read
  // hazard of the exchange buffers is covered by waiting on the tiles that read mine)
  std::vector<std::vector<char>> adj(nct, std::vector<char>(nct, 0));
  for (int b = 0; b < nct; ++b) {
    if (span[2 * b + 1] < 0) continue;
    const int t0 = span[2 * b] / tile_rows, t1 = span[2 * b + 1] / tile_rows;
    for (int t = t0; t <= t1; ++t)
      if (t != b) adj[b][t] = adj[t][b] = 1;
  }
  std::vector<int> nptr(nct + 1, 0), nlist;
  for (int b = 0; b < nct; ++b) {
    for (int t = 0; t < nct; ++t)
      if (adj[b][t]) nlist.push_back(t);
    nptr[b + 1] = (int)nlist.size();
  }
  auto* p = new ResidentPlan;
  p->nct = nct;
  p->tile_rows = tile_rows;
  p->threads = threads;
  p->rpt = rpt;
  p->cap_nnz = cap;
  p->smem = smem;
  p->nbr_ptr = dev_alloc_shared<int>(nptr.size());
  p->nbr = dev_alloc_shared<int>(std::max<size_t>(nlist.size(), 1));
  SE_CUDA(cudaMemcpyAsync(p->nbr_ptr, nptr.data(), sizeof(int) * nptr.size(), cudaMemcpyHostToDevice,
                          c.stream));
  if (!nlist.empty())
    SE_CUDA(cudaMemcpyAsync(p->nbr, nlist.data(), sizeof(int) * nlist.size(),
                            cudaMemcpyHostToDevice, c.stream));
  ctx_sync(c);
  // the launch must be able to hold every CTA at once
  auto fits = [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return (long)per_sm * c.num_sms >= nct;
  };
  const bool ok = rpt == 1 ? fits(k_cheb_resident<1>) : rpt == 2 ? fits(k_cheb_resident<2>) : false;
  a.resident = p;
  if (!ok) resident_free(a);
}

namespace {
std::atomic<bool> g_resident_on{true};
}
void resident_enable(bool on) { g_resident_on.store(on); }
bool resident_enabled() { return g_resident_on.load(); }
int resident_tiles(const DevCsr& a) { return a.resident && resident_enabled() ? a.resident->nct : 0; }

void cheb_resident(Ctx& c, const DevCsr& a, int kdeg, const double* mu_dev, double cc, double invd,
                   const double* x, double* out, double* const* buf, long long* flags,
                   const Ctl* halt) {
  const ResidentPlan& p = *a.resident;
  ResArgs g{};
  g.n = a.n;
  g.tile_rows = p.tile_rows;
  g.kdeg = kdeg;
  g.rp = a.rp;
  g.ci = a.ci;
  g.v = a.v;
  g.nbr_ptr = p.nbr_ptr;
  g.nbr = p.nbr;
  g.x = x;
  g.out = out;
  for (int q = 0; q < 3; ++q) g.buf[q] = buf[q];
  g.mu = mu_dev;
  g.c = cc;
  g.invd = invd;
  g.flags = flags;
  g.halt = halt;
  g.cap_nnz = p.cap_nnz;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.nct);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = c.prio_hi;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (p.rpt == 1)
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident<1>, g));
  else
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident<2>, g));
  ++c.launches;
}

}  // namespace k
}  // namespace se
