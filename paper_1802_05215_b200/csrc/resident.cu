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
// Measured alternatives (64^3, us per degree; profiles/r2_ncu_summary.md): release/acquire degree
// counters per tile 4.07; this kernel 3.78; all of a thread's operands held in registers before
// the tag checks 5.7-8.5 (spills; the checks serialise the loads anyway); two 256-thread tiles per
// SM with prefetched remote operands 4.2; halo gathered into shared memory in a separate phase
// 4.6 (100 x 100: 1.31, the best there).  The time scales with the rows per SM (1.3 us at 128
// rows, 2.1 at 448, 3.8-4.6 at 1,792): the row sums themselves (two dependent shared-memory loads,
// an individually rounded multiply and add per entry, in storage order) bound the degree, and
// this variant hides the exchange round trips behind other warps' row sums.
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
  const unsigned tag0 = *a.epoch;  // advanced by k_epoch_advance after every application

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

  // Row sum of A times the vector whose own tile is sx (shared memory).  Entries outside the
  // tile come from g (degree 1: the input vector) or from the exchange buffer xc, re-read
  // until they carry `tag`.  Products are formed as operands arrive; the additions run in
  // storage order.
  auto row_sum = [&](int q, const double* sx, const double* g, const uint4* xc, unsigned tag) {
    double acc = 0.0;
    for (int p = ps[q]; p < pe[q]; p += 8) {
      double xv[8];
      unsigned pending = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = 0.0;
        if (p + u < pe[q]) {
          const int col = s_col[p + u];
          const unsigned off = (unsigned)(col - r0);
          if (off < (unsigned)rows)
            xv[u] = sx[off];
          else if (g)
            xv[u] = __ldg(g + col);
          else if (!ld_ll(xc + col, tag, xv[u]))
            pending |= 1u << u;
        }
      }
      int spins = 0;
      while (pending) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if ((pending >> u) & 1u)
            if (ld_ll(xc + s_col[p + u], tag, xv[u])) pending &= ~(1u << u);
        if (++spins > kSpinLimit) __trap();  // a neighbour never arrived: fail, do not hang
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < pe[q]) acc = add(acc, mul(s_val[p + u], xv[u]));
    }
    return acc;
  };

  // degree 1: T_1 = Ahat x; out = mu0 x + mu1 T_1   (filter_poly.hpp:260-269)
  {
    const double mu0 = __ldg(a.mu), mu1 = __ldg(a.mu + 1);
    uint4* dst = a.xch[1];  // slot = degree & 3
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(q, s_x, a.x, nullptr, 0u), mul(a.c, prev[q])), a.invd);
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
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(q, sx, nullptr, src, want), mul(a.c, cur[q])), a.invd);
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

// ---- padded-row fast path (rows of at most 8 entries: stencils) ----------------------------------
// ncu on the kernel above (profiles/r2_resident_64.ncu-rep): 253 warp instructions per row, issue
// slots 48% busy with half the warp slots filled -- it is bound by INSTRUCTIONS (per-entry
// predicates, the local / input / exchange three-way branch, the retry bookkeeping), not by the
// exchange.  For matrices whose rows hold at most 8 entries the tile is kept in padded-row form
// instead (entry-major, s_val[u][row] / s_opi[u][row], so a warp's accesses are consecutive;
// pad entries have value 0 and the row itself as operand: acc + 0 * x leaves the storage-order
// sum unchanged), each entry carries the shared-memory index of its operand (>= 0: a row of the
// tile; < 0: ~halo slot), and the halo -- the previous vector's entries the tile references
// outside itself, a list fixed by the pattern and built once per matrix -- is gathered into
// shared memory at the start of a degree: every thread issues its few halo loads back to back
// (one L2 round trip, not one per entry) and re-reads an entry until it carries the degree's tag.
// The row sums are then 8 unrolled, unpredicated shared-memory multiply-adds.  Used for small
// tiles (<= 512 rows), where it is 1.5x faster than the general kernel; see resident_build.
__device__ __forceinline__ uint4 ld_raw(const uint4* p) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ bool ll_ok(const uint4& r, unsigned tag) { return r.y == tag && r.w == tag; }
__device__ __forceinline__ double ll_value(const uint4& r) { return __hiloint2double((int)r.z, (int)r.x); }

struct EllArgs {
  int n, tile_rows, kdeg;
  const int* rp;
  const int* opi;     // per matrix entry: operand index (>= 0: row of the tile; < 0: ~halo slot)
  const double* v;
  const int* hcol;    // per tile: the columns of its halo slots (cap_halo each)
  const int* hcnt;    // per tile: halo slots in use
  const double* x;
  double* out;
  uint4* xch[4];
  const double* mu;
  double c, invd;
  unsigned* epoch;
  const Ctl* halt;
  int cap_halo;
};

constexpr int kEllR = 8;        // padded row width
constexpr int kHaloBatch = 4;   // halo loads a thread keeps in flight

template <int RPT>
__global__ void __launch_bounds__(512, 2) k_cheb_resident_ell(EllArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = blockDim.x, tid = threadIdx.x;
  const int b = blockIdx.x;
  const int TR = a.tile_rows;
  const int r0 = b * TR;
  const int rows = min(TR, a.n - r0);
  double* s_val = reinterpret_cast<double*>(smem_raw);      // [8][TR]
  double* s_x = s_val + kEllR * TR;                          // [2][TR]
  double* s_halo = s_x + 2 * TR;                             // [cap_halo]
  unsigned short* s_opi = reinterpret_cast<unsigned short*>(s_halo + a.cap_halo);  // [8][TR]:
  // operand index of an entry: < TR a row of the tile, else TR + halo slot
  // the tile's matrix rows in padded form: independent of the previous kernel
  for (int lr = tid; lr < rows; lr += T) {
    const int p0 = __ldg(a.rp + r0 + lr), p1 = __ldg(a.rp + r0 + lr + 1);
#pragma unroll
    for (int u = 0; u < kEllR; ++u) {
      const bool in = p0 + u < p1;
      s_val[u * TR + lr] = in ? __ldg(a.v + p0 + u) : 0.0;
      const int oi = in ? __ldg(a.opi + p0 + u) : lr;
      s_opi[u * TR + lr] = (unsigned short)(oi >= 0 ? oi : TR + ~oi);
    }
  }
  const int hcnt = __ldg(a.hcnt + b);
  const int* __restrict__ hcol = a.hcol + (size_t)b * a.cap_halo;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (a.halt && a.halt->halted) return;
  const unsigned tag0 = *a.epoch;

  double prev[RPT], cur[RPT], acc_out[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int lr = tid + q * T;
    const bool live = lr < rows;
    prev[q] = live ? __ldg(a.x + r0 + lr) : 0.0;
    cur[q] = 0.0;
    acc_out[q] = 0.0;
    if (live) s_x[lr] = prev[q];
  }
  for (int h = tid; h < hcnt; h += T) s_halo[h] = __ldg(a.x + __ldg(hcol + h));  // degree 1's halo
  __syncthreads();

  auto row_sum = [&](int lr, const double* sx) {
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < kEllR; ++u) {
      const int oi = s_opi[u * TR + lr];
      const double* base = oi < TR ? sx : s_halo - TR;
      acc = add(acc, mul(s_val[u * TR + lr], base[oi]));
    }
    return acc;
  };

  // degree 1   (filter_poly.hpp:260-269)
  {
    const double mu0 = __ldg(a.mu), mu1 = __ldg(a.mu + 1);
    uint4* dst = a.xch[1];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(lr, s_x), mul(a.c, prev[q])), a.invd);
      cur[q] = t;
      acc_out[q] = add(add(0.0, mul(mu0, prev[q])), mul(mu1, t));
      if (a.kdeg > 1) {
        st_ll(dst + r0 + lr, t, tag0 + 1u);
        s_x[TR + lr] = t;
      }
    }
    __syncthreads();
  }
  // degrees 2..k   (filter_poly.hpp:270-276)
  for (int j = 2; j <= a.kdeg; ++j) {
    const double muj = __ldg(a.mu + j);
    const uint4* src = a.xch[(j - 1) & 3];
    uint4* dst = a.xch[j & 3];
    const double* sx = s_x + ((j - 1) & 1) * TR;
    double* sxn = s_x + (j & 1) * TR;
    const bool more = j < a.kdeg;
    const unsigned want = tag0 + (unsigned)(j - 1);
    for (int h0 = tid; h0 < hcnt; h0 += kHaloBatch * T) {
      uint4 raw[kHaloBatch];
      int col[kHaloBatch];
#pragma unroll
      for (int k = 0; k < kHaloBatch; ++k) {
        const int h = h0 + k * T;
        col[k] = h < hcnt ? __ldg(hcol + h) : -1;
      }
#pragma unroll
      for (int k = 0; k < kHaloBatch; ++k)
        if (col[k] >= 0) raw[k] = ld_raw(src + col[k]);
#pragma unroll
      for (int k = 0; k < kHaloBatch; ++k) {
        if (col[k] < 0) continue;
        int spins = 0;
        while (!ll_ok(raw[k], want)) {
          raw[k] = ld_raw(src + col[k]);
          if (++spins > kSpinLimit) __trap();  // an entry never arrived: fail, do not hang
        }
        s_halo[h0 + k * T] = ll_value(raw[k]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = tid + q * T;
      if (lr >= rows) continue;
      const double t = mul(sub(row_sum(lr, sx), mul(a.c, cur[q])), a.invd);
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

// per matrix entry its operand index; per tile its halo column list (one slot per remote entry)
__global__ void k_tile_operands(int n, int tile_rows, int cap_halo, const int* __restrict__ rp,
                                const int* __restrict__ ci, int* __restrict__ opi,
                                int* __restrict__ hcol, int* __restrict__ hcnt) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int r0 = b * tile_rows, r1 = min(n, r0 + tile_rows);
  for (int p = rp[r0] + threadIdx.x; p < rp[r1]; p += blockDim.x) {
    const int c = ci[p];
    if (c >= r0 && c < r1) {
      opi[p] = c - r0;
    } else {
      const int slot = atomicAdd(&s_cnt, 1);
      if (slot < cap_halo) hcol[(size_t)b * cap_halo + slot] = c;
      opi[p] = ~slot;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) hcnt[b] = s_cnt;
}

__global__ void k_tile_remote_count(int n, int tile_rows, const int* __restrict__ rp,
                                    const int* __restrict__ ci, int* __restrict__ nrem) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int r0 = b * tile_rows, r1 = min(n, r0 + tile_rows);
  int mine = 0;
  for (int p = rp[r0] + threadIdx.x; p < rp[r1]; p += blockDim.x) {
    const int c = ci[p];
    mine += (c < r0 || c >= r1);
  }
  atomicAdd(&s_cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) nrem[b] = s_cnt;
}

size_t ell_smem_bytes(int tile_rows, int cap_halo) {
  return (size_t)tile_rows * kEllR * 10 + (size_t)tile_rows * 16 + (size_t)cap_halo * 8 + 16;
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
  // padded-row fast path (rows of <= 8 entries): operand indices and per-tile halo lists
  bool ell = false;
  int cap_halo = 0;
  size_t ell_smem = 0;
  int* opi = nullptr;   // device, nnz
  int* hcol = nullptr;  // device, nct x cap_halo
  int* hcnt = nullptr;  // device, nct
};

void resident_free(DevCsr& a) {
  if (!a.resident) return;
  dev_free_shared(a.resident->opi);
  dev_free_shared(a.resident->hcol);
  dev_free_shared(a.resident->hcnt);
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
  // one tile per SM (at least 128 rows a tile), up to 1,024 threads and 2 rows a thread
  int tile_rows = std::max((a.n + c.num_sms - 1) / c.num_sms, 128);
  tile_rows = (tile_rows + 31) / 32 * 32;
  if (tile_rows > 2048) return;
  const int nct = (a.n + tile_rows - 1) / tile_rows;
  const int threads = tile_rows > 512 ? 1024 : (tile_rows > 256 ? 512 : 256);
  const int rpt = (tile_rows + threads - 1) / threads;
  // The padded-row kernel serves small tiles (rows of <= 8 entries, <= 512 rows a tile: cfg1, the
  // 32^3 proxy, 40^3): 1.05 against 1.55 us per degree at 100 x 100.  At 64^3 (1,792 rows and
  // 3,700 halo entries a tile) every variant measured lands at 3.7-4.6 us and the general kernel
  // is the fastest (profiles/r2_ncu_summary.md), so large tiles stay with it.
  const bool want_ell = a.max_row_nnz > 0 && a.max_row_nnz <= kEllR && tile_rows <= 512;
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
  const bool ok = rpt == 1 ? fits(k_cheb_resident<1>) : rpt == 2 ? fits(k_cheb_resident<2>) : false;
  if (!ok) return;
  auto* p = new ResidentPlan;
  p->nct = nct;
  p->tile_rows = tile_rows;
  p->threads = threads;
  p->rpt = rpt;
  p->cap_nnz = cap;
  p->smem = smem;
  a.resident = p;
  // the padded-row fast path, when every row holds at most 8 entries and the image fits
  if (want_ell) {
    int* dnrem = dev_alloc<int>(nct);
    k_tile_remote_count<<<nct, 256, 0, c.stream>>>(a.n, tile_rows, a.rp, a.ci, dnrem);
    SE_CUDA(cudaGetLastError());
    ++c.launches;
    std::vector<int> nrem(nct);
    SE_CUDA(cudaMemcpyAsync(nrem.data(), dnrem, sizeof(int) * nct, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    dev_free(dnrem);
    int cap_halo = 2;
    for (int v : nrem) cap_halo = std::max(cap_halo, v);
    cap_halo = (cap_halo + 1) & ~1;
    const size_t esm = ell_smem_bytes(tile_rows, cap_halo);
    auto efits = [&](auto kern) {
      if (esm > (size_t)max_optin || tile_rows + cap_halo > 65535) return false;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, esm) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return (long)per_sm * c.num_sms >= nct;
    };
    if (efits(k_cheb_resident_ell<1>)) {
      p->opi = dev_alloc_shared<int>((size_t)a.nnz);
      p->hcol = dev_alloc_shared<int>((size_t)nct * cap_halo);
      p->hcnt = dev_alloc_shared<int>(nct);
      k_tile_operands<<<nct, 256, 0, c.stream>>>(a.n, tile_rows, cap_halo, a.rp, a.ci, p->opi, p->hcol,
                                                 p->hcnt);
      SE_CUDA(cudaGetLastError());
      ++c.launches;
      ctx_sync(c);
      p->cap_halo = cap_halo;
      p->ell_smem = esm;
      p->ell = true;
    }
  }
}

void resident_enable(int mode) { g_resident_mode.store(mode); }
bool resident_enabled() { return g_resident_mode.load() != 0; }
int resident_tiles(const DevCsr& a) { return a.resident && resident_enabled() ? a.resident->nct : 0; }
// Shared memory one tile of the resident filter holds (0: no plan): above half an SM's shared
// memory two filter launches cannot share the GPU, and slices are then best solved one at a time.
size_t resident_tile_smem(const DevCsr& a) {
  if (!a.resident || !resident_enabled()) return 0;
  return a.resident->ell && g_resident_mode.load() != 2 ? a.resident->ell_smem : a.resident->smem;
}
size_t resident_state_bytes(const DevCsr& a) { return 4 * (size_t)a.n * sizeof(uint4) + 16; }

void cheb_resident(Ctx& c, const DevCsr& a, int kdeg, const double* mu_dev, double cc, double invd,
                   const double* x, double* out, void* state, const Ctl* halt) {
  const ResidentPlan& p = *a.resident;
  if (p.ell && g_resident_mode.load() != 2) {  // mode 2: force the general kernel (A/B timing)
    EllArgs e{};
    e.n = a.n;
    e.tile_rows = p.tile_rows;
    e.kdeg = kdeg;
    e.rp = a.rp;
    e.opi = p.opi;
    e.v = a.v;
    e.hcol = p.hcol;
    e.hcnt = p.hcnt;
    e.x = x;
    e.out = out;
    e.epoch = static_cast<unsigned*>(state);
    uint4* ex = reinterpret_cast<uint4*>(static_cast<unsigned char*>(state) + 16);
    for (int q = 0; q < 4; ++q) e.xch[q] = ex + (size_t)q * a.n;
    e.mu = mu_dev;
    e.c = cc;
    e.invd = invd;
    e.halt = halt;
    e.cap_halo = p.cap_halo;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.nct);
    cfg.blockDim = dim3(p.threads);
    cfg.dynamicSmemBytes = p.ell_smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = c.prio_hi;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident_ell<1>, e));
    k_epoch_advance<<<1, 1, 0, c.stream>>>(e.epoch, kdeg, halt);
    SE_CUDA(cudaGetLastError());
    c.launches += 2;
    return;
  }
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
  else
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_resident<2>, g));
  // the next application's tags start past this one's (a separate, stream-ordered launch: a
  // tile far from tile 0 in the matrix graph may start after tile 0 has finished a short filter)
  k_epoch_advance<<<1, 1, 0, c.stream>>>(g.epoch, kdeg, halt);
  SE_CUDA(cudaGetLastError());
  c.launches += 2;
}

}  // namespace k
}  // namespace se
