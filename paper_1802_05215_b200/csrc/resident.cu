// Resident Chebyshev filter: all k degrees of apply_pol (filter_poly.hpp:256-277) in ONE launch,
// for matrices whose CSR arrays fit in the GPU's aggregate shared memory (148 x ~190 KB = 28 MB:
// BASELINE cfg1 and cfg2; n <= ~300k rows).
//
// Why: on such a matrix one filter degree moves ~33 MB that is L2-resident, and a chain of k
// dependent launches costs 4.2-4.5 us per degree however the launches are issued -- a third of
// the cfg2 solve.  Here the matrix is read ONCE per filter application: every CTA (two per SM)
// copies the CSR rows of its own row tile into shared memory and keeps them there for all k
// degrees, together with its tile of the current Chebyshev vector (double-buffered), while the
// previous vector, the current vector and the running sum out = sum_j mu_j T_j v of its own rows
// live in registers.
// Per degree a CTA only exchanges vector entries with the tiles its columns reach: it writes its
// new tile to a global (L2) exchange buffer as tagged 16-byte entries {lo32, tag, hi32, tag}
// (NCCL's LL idea: each 8-byte half is atomic and carries the degree that produced it), and a
// consumer re-reads a remote entry until both tags name the degree it needs.  The data is its
// own arrival signal: no flag, no fence, no grid barrier, no kernel boundary -- a dataflow
// hand-off between neighbouring tiles (2 of a 7-point stencil's 7 gathers leave the tile).
//
// Safety: the launch is cooperative (all CTAs co-resident by construction) and the wait is bounded
// (an entry that never arrives traps instead of hanging the device).  FOUR exchange buffers
// rotate (slot = degree mod 4): a tile writes degree j + 3 over degree j - 1 only after it has
// finished degree j + 2, which needed a degree j + 1 entry from each tile it reads; that tile
// had then passed its end-of-degree-j barrier, i.e. ALL its threads were done reading degree
// j - 1 entries.  On a structurally symmetric tile pattern (checked when the plan is built) the
// tiles a tile reads are the tiles that read it, so no entry is overwritten while a neighbour
// still needs it -- by construction, not by timing (three buffers would leave a window).  Tags
// grow monotonically across applications (epoch + degree), so a stale entry never passes for a
// fresh one.
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

// Tile exchange in the style of NCCL's LL protocol: a vector entry travels as 16 bytes
// {lo32, tag, hi32, tag}; each 8-byte half is written and read atomically and carries the tag of
// the degree that produced it, so a consumer simply re-reads an entry until both tags match --
// no flag, no fence, no separate poll: the data is its own arrival signal.
__device__ __forceinline__ void st_ll(uint4* p, double v, unsigned tag) {
  const unsigned lo = (unsigned)__double2loint(v), hi = (unsigned)__double2hiint(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "r"(lo), "r"(tag),
               "r"(hi), "r"(tag)
               : "memory");
}
__device__ __forceinline__ bool ld_ll(const uint4* p, unsigned tag, double& v) {
  unsigned a, b, c, d;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "l"(p)
               : "memory");
  v = __hiloint2double((int)c, (int)a);
  return b == tag && d == tag;
}

struct ResArgs {
  int n, tile_rows, kdeg;
  const int* rp;
  const int* ci;
  const double* v;
  const double* x;    // input vector (contiguous)
  double* out;        // sum_j mu_j T_j x
  uint4* xch[4];      // exchange buffers (n tagged entries each)
  const double* mu;   // k + 1 coefficients (device)
  double c, invd;
  unsigned* epoch;    // tag base: advanced by kdeg at the end of every launch
  const Ctl* halt;
  int cap_nnz;        // shared-memory capacity of a tile's entries
};

constexpr int kSpinLimit = 1 << 22;

// RPT rows per thread, kResThreads threads per CTA, two CTAs per SM (while one tile waits for an
// exchange entry the other computes).  A row's operands outside the tile ("remote": at most kNR
// of them are prefetched, which covers stencils and banded matrices; rows with more fall back to
// reading them in place) are requested for ALL of the thread's rows at the start of a degree;
// the rows are then summed one after the other from shared memory, each checking its remote
// operands only when it needs them, so the exchange round trip overlaps the shared-memory work.
constexpr int kResThreads = 256;
constexpr int kNR = 4;

template <int RPT>
__global__ void __launch_bounds__(kResThreads, 2) k_cheb_resident(ResArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int T = kResThreads;
  const int tid = threadIdx.x;
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
  const unsigned tag0 = *a.epoch;  // advanced by k_epoch_advance after every application

  double prev[RPT], cur[RPT], acc_out[RPT];
  int ps[RPT], len[RPT];
  unsigned rmask[RPT];  // bit u: entry u of the row is remote (rows of <= 32 entries with <= kNR
                        // remote ones); 0xffffffff marks a row that reads remote entries in place
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
    len[q] = lr < rows ? s_rp[lr + 1] - ps[q] : 0;
    unsigned m = 0;
    int nrem = 0;
    for (int u = 0; u < len[q]; ++u)
      if ((unsigned)(s_col[ps[q] + u] - r0) >= (unsigned)rows) {
        ++nrem;
        if (u < 32) m |= 1u << u;
      }
    rmask[q] = (len[q] > 32 || nrem > kNR) ? 0xffffffffu : m;
  }
  constexpr unsigned kInPlace = 0xffffffffu;

  // the i-th remote entry (in storage order) of a prefetching row: its position in the row
  auto remote_pos = [&](unsigned m, int i) {
    for (int k = 0; k < i; ++k) m &= m - 1;  // drop the i lowest set bits
    return __ffs((int)m) - 1;                // -1: the row has fewer remote entries
  };

  // sum of the row's products in storage order.  sx: the tile's vector (shared memory);
  // g (degree 1): the input vector, read in place; xc/tag (degrees >= 2): the exchange buffer;
  // rv / pend: the row's prefetched remote operands and which of them have not arrived yet.
  auto row_sum = [&](int q, const double* sx, const double* g, const uint4* xc, unsigned tag,
                     double (&rv)[kNR], unsigned pend) {
    const bool inplace = g != nullptr || rmask[q] == kInPlace;
    double acc = 0.0;
    for (int p0 = 0; p0 < len[q]; p0 += 8) {
      double xv[8];
      unsigned wait = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = 0.0;
        if (p0 + u < len[q]) {
          const int col = s_col[ps[q] + p0 + u];
          const unsigned off = (unsigned)(col - r0);
          if (off < (unsigned)rows)
            xv[u] = sx[off];
          else if (g)
            xv[u] = __ldg(g + col);
          else if (inplace && !ld_ll(xc + col, tag, xv[u]))
            wait |= 1u << u;
        }
      }
      if (!inplace) {
        // the prefetched operands: re-read those that had not arrived, then drop them into place
        int spins = 0;
        while (pend) {
#pragma unroll
          for (int i = 0; i < kNR; ++i)
            if ((pend >> i) & 1u) {
              const int pos = remote_pos(rmask[q], i);
              if (ld_ll(xc + s_col[ps[q] + pos], tag, rv[i])) pend &= ~(1u << i);
            }
          if (++spins > kSpinLimit) __trap();  // an entry never arrived: fail, do not hang
        }
        const unsigned m = rmask[q] >> p0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if ((m >> u) & 1u) {
            const int i = __popc(rmask[q] & ((1u << (p0 + u)) - 1u));  // which remote entry
            xv[u] = i == 0 ? rv[0] : i == 1 ? rv[1] : i == 2 ? rv[2] : rv[3];
          }
      } else {
        int spins = 0;
        while (wait) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if ((wait >> u) & 1u)
              if (ld_ll(xc + s_col[ps[q] + p0 + u], tag, xv[u])) wait &= ~(1u << u);
          if (++spins > kSpinLimit) __trap();
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p0 + u < len[q]) acc = add(acc, mul(s_val[ps[q] + p0 + u], xv[u]));
    }
    return acc;
  };

  // degree 1: T_1 = Ahat x; out = mu0 x + mu1 T_1   (filter_poly.hpp:260-269)
  {
    const double mu0 = __ldg(a.mu), mu1 = __ldg(a.mu + 1);
    uint4* dst = a.xch[1];  // slot = degree & 3
    double none[kNR] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(q, s_x, a.x, nullptr, 0u, none, 0u), mul(a.c, prev[q])), a.invd);
      cur[q] = t;
      acc_out[q] = add(add(0.0, mul(mu0, prev[q])), mul(mu1, t));
      if (a.kdeg > 1) {
        st_ll(dst + r0 + lr, t, tag0 + 1u);
        s_x[a.tile_rows + lr] = t;
      }
    }
    __syncthreads();  // the tile's new vector is in shared memory for everyone
  }
  // degrees 2..k: T_j = 2 Ahat T_{j-1} - T_{j-2}; out += mu_j T_j   (filter_poly.hpp:270-276)
  for (int j = 2; j <= a.kdeg; ++j) {
    const double muj = __ldg(a.mu + j);
    const uint4* src = a.xch[(j - 1) & 3];
    uint4* dst = a.xch[j & 3];
    const double* sx = s_x + ((j - 1) & 1) * a.tile_rows;
    double* sxn = s_x + (j & 1) * a.tile_rows;
    const bool more = j < a.kdeg;
    const unsigned want = tag0 + (unsigned)(j - 1);
    // request every row's remote operands now; they are looked at when their row is summed
    double rv[RPT][kNR];
    unsigned pend[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      pend[q] = 0;
#pragma unroll
      for (int i = 0; i < kNR; ++i) {
        rv[q][i] = 0.0;
        if (rmask[q] != kInPlace) {
          const int pos = remote_pos(rmask[q], i);
          if (pos >= 0 && !ld_ll(src + s_col[ps[q] + pos], want, rv[q][i])) pend[q] |= 1u << i;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t =
          mul(sub(row_sum(q, sx, nullptr, src, want, rv[q], pend[q]), mul(a.c, cur[q])), a.invd);
      const double tj = sub(mul(2.0, t), prev[q]);
      acc_out[q] = add(acc_out[q], mul(muj, tj));
      prev[q] = cur[q];
      cur[q] = tj;
      if (more) {
        st_ll(dst + r0 + lr, tj, want + 1u);
        sxn[lr] = tj;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = tid + q * T;
    if (lr < rows) a.out[r0 + lr] = acc_out[q];
  }
}

// per tile: bit t of mask[tile] is set when a row of the tile has an entry in tile t's columns
constexpr int kMaskWords = 8;  // up to 256 tiles
__global__ void k_tile_adjacency(int n, int tile_rows, const int* __restrict__ rp,
                                 const int* __restrict__ ci, unsigned* __restrict__ mask) {
  __shared__ unsigned s_m[kMaskWords];
  if (threadIdx.x < kMaskWords) s_m[threadIdx.x] = 0u;
  __syncthreads();
  const int b = blockIdx.x;
  const int r0 = b * tile_rows, r1 = min(n, r0 + tile_rows);
  for (int p = rp[r0] + threadIdx.x; p < rp[r1]; p += blockDim.x) {
    const int t = ci[p] / tile_rows;
    atomicOr(&s_m[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  if (threadIdx.x < kMaskWords) mask[(size_t)b * kMaskWords + threadIdx.x] = s_m[threadIdx.x];
}

__global__ void k_epoch_advance(unsigned* epoch, int kdeg, const Ctl* halt) {
  if (halt && halt->halted) return;
  *epoch += (unsigned)kdeg;
}

size_t res_smem_bytes(int tile_rows, int cap_nnz) {
  return (size_t)cap_nnz * 12 + (size_t)tile_rows * 16 + (size_t)(tile_rows + 1) * 4 + 16;
}

std::atomic<int> g_resident_mode{1};  // 0 off

}  // namespace

// The plan of a matrix: row tiles (one per CTA) and the per-tile entry capacity.
struct ResidentPlan {
  int nct = 0, tile_rows = 0, threads = 0, rpt = 0, cap_nnz = 0;
  size_t smem = 0;
};

void resident_free(DevCsr& a) {
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
  // two tiles per SM when the matrix is large enough to fill them (one tile's exchange wait
  // overlaps the other's shared-memory work); 256 threads a tile, up to 4 rows a thread
  int tile_rows = std::max((a.n + 2 * c.num_sms - 1) / (2 * c.num_sms), 128);
  tile_rows = (tile_rows + 31) / 32 * 32;
  if (tile_rows > 4 * kResThreads) return;
  const int nct = (a.n + tile_rows - 1) / tile_rows;
  const int threads = kResThreads;
  const int rpt = tile_rows <= threads ? 1 : (tile_rows <= 2 * threads ? 2 : 4);
  // per-tile entry counts: the largest sizes the shared-memory image
  std::vector<int> rp_tiles(nct + 1);
  for (int b = 0; b <= nct; ++b)
    SE_CUDA(cudaMemcpyAsync(&rp_tiles[b], a.rp + std::min((long)a.n, (long)b * tile_rows),
                            sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  ctx_sync(c);
  int cap = 0;
  for (int b = 0; b < nct; ++b) cap = std::max(cap, rp_tiles[b + 1] - rp_tiles[b]);
  cap = (cap + 1) & ~1;
  const size_t smem = res_smem_bytes(tile_rows, cap);
  if (smem > (size_t)max_optin || nct > 32 * kMaskWords) return;
  // tile dependence must be symmetric (a tile reads exactly the tiles that read it): that is
  // what keeps a producer from lapping a consumer on the rotating exchange buffers
  {
    unsigned* dmask = dev_alloc<unsigned>((size_t)nct * kMaskWords);
    k_tile_adjacency<<<nct, 256, 0, c.stream>>>(a.n, tile_rows, a.rp, a.ci, dmask);
    SE_CUDA(cudaGetLastError());
    ++c.launches;
    std::vector<unsigned> m((size_t)nct * kMaskWords);
    SE_CUDA(cudaMemcpyAsync(m.data(), dmask, sizeof(unsigned) * m.size(), cudaMemcpyDeviceToHost,
                            c.stream));
    ctx_sync(c);
    dev_free(dmask);
    auto reads = [&](int x, int y) { return (m[(size_t)x * kMaskWords + (y >> 5)] >> (y & 31)) & 1u; };
    for (int x = 0; x < nct; ++x)
      for (int y = x + 1; y < nct; ++y)
        if (reads(x, y) != reads(y, x)) return;
  }
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
  const bool ok = rpt == 1 ? fits(k_cheb_resident<1>)
                  : rpt == 2 ? fits(k_cheb_resident<2>) : fits(k_cheb_resident<4>);
  if (!ok) return;
  auto* p = new ResidentPlan;
  p->nct = nct;
  p->tile_rows = tile_rows;
  p->threads = threads;
  p->rpt = rpt;
  p->cap_nnz = cap;
  p->smem = smem;
  a.resident = p;
}

void resident_enable(int mode) { g_resident_mode.store(mode); }
bool resident_enabled() { return g_resident_mode.load() != 0; }
int resident_tiles(const DevCsr& a) { return a.resident && resident_enabled() ? a.resident->nct : 0; }
size_t resident_state_bytes(const DevCsr& a) { return 4 * (size_t)a.n * sizeof(uint4) + 16; }

void cheb_resident(Ctx& c, const DevCsr& a, int kdeg, const double* mu_dev, double cc, double invd,
                   const double* x, double* out, void* state, const Ctl* halt) {
  const ResidentPlan& p = *a.resident;
  ResArgs g{};
  g.n = a.n;
  g.tile_rows = p.tile_rows;
  g.kdeg = kdeg;
  g.rp = a.rp;
  g.ci = a.ci;
  g.v = a.v;
  g.x = x;
  g.out = out;
  // state: [epoch (16 bytes)] [4 exchange buffers of n tagged entries]
  g.epoch = static_cast<unsigned*>(state);
  uint4* xch = reinterpret_cast<uint4*>(static_cast<unsigned char*>(state) + 16);
  for (int q = 0; q < 4; ++q) g.xch[q] = xch + (size_t)q * a.n;
  g.mu = mu_dev;
  g.c = cc;
  g.invd = invd;
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
  else if (p.rpt == 2)
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident<2>, g));
  else
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident<4>, g));
  // the next application's tags start past this one's (a separate, stream-ordered launch: a
  // tile far from tile 0 in the matrix graph may start after tile 0 has finished a short filter)
  k_epoch_advance<<<1, 1, 0, c.stream>>>(g.epoch, kdeg, halt);
  SE_CUDA(cudaGetLastError());
  c.launches += 2;
}

}  // namespace k
}  // namespace se
