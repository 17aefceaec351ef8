// Sparse kernels for sm_100a: the fused Chebyshev-filter SpMV (K1 of SURVEY.md §2.1), the block
// KPM moment step (K3), and the device stencil generator (K8).
//
// Numerics: every product and sum is rounded individually (__dmul_rn / __dadd_rn, no FMA
// contraction) and each row is summed in storage order, exactly like the reference's scalar loops
// (CsrMatrix::matvec csr.hpp:98-105, apply_pol filter_poly.hpp:256-277, kpm_dos dos.hpp:96-108),
// which are compiled for baseline x86-64 without FMA.  The filter application is therefore
// bit-identical to the reference's on the same input vector.
#include <cub/cub.cuh>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

constexpr int kRows = 256;    // rows per CTA tile, one per thread
constexpr int kChunk = 2048;  // nnz staged per pass: 16 KB vals + 8 KB cols of shared memory

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

struct KArgs {
  const double* x;
  const double* prev;
  double* y;
  double* out;
  double c, invd, mu0, muj;
  const Ctl* src_ctl;
  long src_ld;
  int x_indirect, prev_indirect;
  const Ctl* halt;
};

// One CTA = one tile of kRows consecutive rows.  The tile's nnz range [rp[r0], rp[r0+kRows]) is
// contiguous in CSR, so it is staged into shared memory with fully coalesced 16-byte loads; each
// thread then sums its own row sequentially (reference order) gathering x through L1/L2.  Rows
// longer than the stage are handled by carrying the accumulator across stage passes.
// Latency structure (the kernel is latency-bound when A is L2-resident): one round trip for the
// row pointers and every row-local operand (x[r], prev[r], out[r]), one for the staged tile,
// one for the x gathers (8 in flight per thread).
// Programmatic dependent launch: everything that does not depend on the previous kernel (row
// pointers, the tile's A entries) is fetched BEFORE griddepcontrol.wait, so in a chain of filter
// degrees the next launch's A staging overlaps the previous degree's tail; x, prev, out, and the
// Ctl words are read after it.  Without the launch attribute the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// One tile of kRows rows (see k_spmv_cheb).  `wait` = this is the CTA's first tile: the PDL wait
// and the halt check happen once, after the first tile's A staging has been issued.
template <int MODE>
__device__ __forceinline__ bool spmv_cheb_tile(int n, int tile, bool wait, const int* __restrict__ rp,
                                               const int* __restrict__ ci,
                                               const double* __restrict__ v, const KArgs& a,
                                               double* s_v, int* s_c) {
  const size_t coff = (size_t)blockIdx.y * n;  // column of a column-major batch (kPlain)
  const int r0 = tile * kRows;
  const int r = r0 + threadIdx.x;
  const bool live = r < n;
  const int rend = min(r0 + kRows, n);
  // independent of the previous kernel: tile bounds, own row bounds, first chunk of A
  const int base = __ldg(rp + r0), end = __ldg(rp + rend);
  int rs = end, re = end;
  if (live) {
    rs = __ldg(rp + r);
    re = __ldg(rp + r + 1);
  }
  auto stage = [&](int c0) {  // cp.async (LDGSTS, 16-byte, zero-filled tails)
    const int cend = c0 + min(kChunk, end - c0);
    const int va = c0 & ~1, ca = c0 & ~3;
    const int nv16 = (cend - va + 1) >> 1, nc16 = (cend - ca + 3) >> 2;
    for (int q = threadIdx.x; q < nv16; q += kRows) {
      const int valid = min(2, cend - (va + 2 * q));
      cp_async16(&s_v[2 * q], v + va + 2 * q, 8 * valid);
    }
    for (int q = threadIdx.x; q < nc16; q += kRows) {
      const int valid = min(4, cend - (ca + 4 * q));
      cp_async16(&s_c[4 * q], ci + ca + 4 * q, 4 * valid);
    }
  };
  if (base < end) stage(base);
  if (wait) {
    pdl_wait();
    pdl_trigger();
    if (a.halt && a.halt->halted) {
      cp_async_wait_all();
      return false;
    }
  }
  const size_t ioff = a.src_ctl ? (size_t)a.src_ctl->i * a.src_ld : 0;
  const double* __restrict__ x = a.x + coff + (a.x_indirect ? ioff : 0);
  double xr = 0.0, pv = 0.0, ov = 0.0;
  if (live) {
    if (MODE != kPlain) xr = __ldg(x + r);
    if (MODE == kNext) {
      const double* __restrict__ prev = a.prev + (a.prev_indirect ? ioff : 0);
      pv = __ldg(prev + r);
      ov = a.out[r];
    }
  }
  double acc = 0.0;
  for (int c0 = base; c0 < end; c0 += kChunk) {
    const int cn = min(kChunk, end - c0);
    const int va = c0 & ~1, ca = c0 & ~3;
    const int cend = c0 + cn;
    if (c0 != base) stage(c0);
    cp_async_wait_all();
    __syncthreads();
    // gathers, 8 in flight; sums stay in storage order
    const int p0 = max(rs, c0), pend = min(re, cend);
    const int dv = va, dc = ca;  // smem index = global index - chunk origin (per array)
    for (int p = p0; p < pend; p += 8) {
      double xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = (p + u < pend) ? __ldg(x + s_c[p + u - dc]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (p + u < pend) acc = add(acc, mul(s_v[p + u - dv], xv[u]));
    }
    __syncthreads();
  }
  if (!live) return true;
  double* __restrict__ y = a.y + coff;
  if (MODE == kPlain) {
    y[r] = acc;
    return true;
  }
  // Ahat x = (A x - c x) * (1/d)   (filter_poly.hpp:265)
  const double t = mul(sub(acc, mul(a.c, xr)), a.invd);
  if (MODE == kFirst) {
    y[r] = t;
    // out = 0 + mu0 v ; out += mu1 T_1 v   (filter_poly.hpp:261-262, 269)
    a.out[r] = add(add(0.0, mul(a.mu0, xr)), mul(a.muj, t));
  } else {
    // T_j = 2 Ahat T_{j-1} - T_{j-2} ; out += mu_j T_j   (filter_poly.hpp:272-275)
    const double tj = sub(mul(2.0, t), pv);
    y[r] = tj;
    a.out[r] = add(ov, mul(a.muj, tj));
  }
  return true;
}

// Grid: one CTA per tile by default; a capped grid (SE_FILTER_CTAS) walks the tiles with a
// stride, so a filter degree occupies fewer SM slots next to other slices' GEMV CTAs.
template <int MODE>
__global__ void __launch_bounds__(kRows) k_spmv_cheb(int n, const int* __restrict__ rp,
                                                      const int* __restrict__ ci,
                                                      const double* __restrict__ v, KArgs a) {
  __shared__ __align__(16) double s_v[kChunk + 8];
  __shared__ __align__(16) int s_c[kChunk + 8];
  const int ntiles = (n + kRows - 1) / kRows;
  bool first = true;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (!first) __syncthreads();  // the previous tile's readers of s_v / s_c are done
    if (!spmv_cheb_tile<MODE>(n, tile, first, rp, ci, v, a, s_v, s_c)) return;
    first = false;
  }
}


// ---- multi-vector filter degree (one A tile staging for up to kMV independent recurrences) ------
// Used to batch the filter degree j of several slices solved on the same GPU: the tile of A is
// staged once and every live vector's row sum is formed from it (storage order, rounded exactly
// as in k_spmv_cheb, so each vector's result is bit-identical to its single-vector filter).
constexpr int kMV = 8;

constexpr int kMRows = 64;  // rows per tile; one warp-pair per vector: 64 x kMV threads

// CTA = 64-row tile x nv vectors (thread = (vector, row)); the tile's A entries are staged once
// with cp.async and shared by every vector's row sums (each warp: 32 consecutive rows of one
// vector, so gathers coalesce exactly as in the single-vector kernel).
__global__ void __launch_bounds__(kMRows * kMV) k_spmv_cheb_multi(int n, const int* __restrict__ rp,
                                                                  const int* __restrict__ ci,
                                                                  const double* __restrict__ v,
                                                                  MultiArgs a) {
  __shared__ __align__(16) double s_v[kMRows * 16 + 8];
  __shared__ __align__(16) int s_c[kMRows * 16 + 8];
  constexpr int kStage = kMRows * 16;
  const int q = threadIdx.x / kMRows;  // vector
  const int lr = threadIdx.x - q * kMRows;
  const int r0 = blockIdx.x * kMRows;
  const int r = r0 + lr;
  const int rend = min(r0 + kMRows, n);
  const int base = __ldg(rp + r0), end = __ldg(rp + rend);
  int rs = end, re = end;
  if (r < n) {
    rs = __ldg(rp + r);
    re = __ldg(rp + r + 1);
  }
  auto stage = [&](int c0) {  // independent of the previous kernel: issued before the PDL wait
    const int cend = c0 + min(kStage, end - c0);
    const int va = c0 & ~1, ca = c0 & ~3;
    const int nv16 = (cend - va + 1) >> 1, nc16 = (cend - ca + 3) >> 2;
    for (int t = threadIdx.x; t < nv16; t += kMRows * kMV)
      cp_async16(&s_v[2 * t], v + va + 2 * t, 8 * min(2, cend - (va + 2 * t)));
    for (int t = threadIdx.x; t < nc16; t += kMRows * kMV)
      cp_async16(&s_c[4 * t], ci + ca + 4 * t, 4 * min(4, cend - (ca + 4 * t)));
  };
  if (base < end) stage(base);
  pdl_wait();
  pdl_trigger();
  const bool on = q < a.nv && !(a.ctl[q] && a.ctl[q]->halted);
  const bool live = on && r < n;
  size_t ioff = 0;
  const double* __restrict__ x = nullptr;
  double xr = 0.0, pv = 0.0, ov = 0.0;
  if (live) {
    ioff = a.ctl[q] ? (size_t)a.ctl[q]->i * a.ld : 0;
    x = a.x[q] + (a.x_ind[q] ? ioff : 0);
    xr = __ldg(x + r);
    if (!a.first[q]) {
      pv = __ldg(a.prev[q] + (a.prev_ind[q] ? ioff : 0) + r);
      ov = a.out[q][r];
    }
  }
  double acc = 0.0;
  for (int c0 = base; c0 < end; c0 += kStage) {
    const int cn = min(kStage, end - c0), cend = c0 + cn;
    const int va = c0 & ~1, ca = c0 & ~3;
    if (c0 != base) {
      __syncthreads();  // the previous chunk's readers are done
      stage(c0);
    }
    cp_async_wait_all();
    __syncthreads();
    if (live) {
      const int p0 = max(rs, c0), pend = min(re, cend);
      for (int p = p0; p < pend; p += 8) {
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = (p + u < pend) ? __ldg(x + s_c[p + u - ca]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p + u < pend) acc = add(acc, mul(s_v[p + u - va], xv[u]));
      }
    }
  }
  if (!live) return;
  const double t = mul(sub(acc, mul(a.c, xr)), a.invd);
  if (a.first[q]) {
    a.y[q][r] = t;
    a.out[q][r] = add(add(0.0, mul(a.mu0[q], xr)), mul(a.muj[q], t));
  } else {
    const double tj = sub(mul(2.0, t), pv);
    a.y[q][r] = tj;
    a.out[q][r] = add(ov, mul(a.muj[q], tj));
  }
}

// ---- block KPM step --------------------------------------------------------------------------
// Probes stored row-major (n x kB, kB = 16 lanes; b <= 16 live).  A half-warp owns one row; lane
// j owns probe j and sums that row in storage order (bitwise the reference's per-probe matvec).
// The moment dot v_j . T_k v_j is reduced deterministically: per-CTA partials + last-CTA sum.
constexpr int kB = 16;
constexpr int kKpmFirst = 1, kKpmDoubling = 2;  // 0: direct recurrence
constexpr int kKpmThreads = 256;
constexpr int kEllMinB = 3;  // resident CTAs per SM the ELL kernel is register-capped for
constexpr int kKpmPD = 1;    // default L2 prefetch distance (batches) of the ELL kernel


// x / d from the correctly rounded reciprocal with one FMA correction (Markstein): the
// correctly rounded quotient for finite, non-extreme operands, at 3 instructions instead of the
// ~12 of the IEEE division routine.
__device__ __forceinline__ double div_by(double x, double d, double dinv) {
  const double q = __dmul_rn(x, dinv);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, dinv, q);
}

// Deterministic reduction of the per-thread dot partials: per-CTA sums over the 16 half-warps
// (fixed order), then the last CTA sums the CTA partials in CTA order into zeta.
__device__ __forceinline__ void kpm_finish(double acc0, double acc1, int b, bool first, bool dbl,
                                           double* __restrict__ partial, unsigned* counter,
                                           double* __restrict__ zeta, int kmom) {
  __shared__ double s0[kKpmThreads], s1[kKpmThreads];
  __shared__ bool s_last;
  s0[threadIdx.x] = acc0;
  s1[threadIdx.x] = acc1;
  __syncthreads();
  if (threadIdx.x < kB) {
    double q0 = 0.0, q1 = 0.0;
    for (int h = 0; h < kKpmThreads / kB; ++h) {
      q0 = add(q0, s0[h * kB + threadIdx.x]);
      q1 = add(q1, s1[h * kB + threadIdx.x]);
    }
    partial[(size_t)blockIdx.x * 2 * kB + threadIdx.x] = q0;
    partial[(size_t)blockIdx.x * 2 * kB + kB + threadIdx.x] = q1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Last CTA: columns x {acc0, acc1}, each summed over CTAs in index order by 8 lanes + shuffle.
  const int col = threadIdx.x >> 3;  // 32 (column, which) pairs, 8 threads each
  const int sub8 = threadIdx.x & 7;
  double q = 0.0;
  for (int blk = sub8; blk < (int)gridDim.x; blk += 8) q = add(q, __ldcg(partial + (size_t)blk * 2 * kB + col));
  for (int o = 4; o > 0; o >>= 1) q = add(q, __shfl_down_sync(0xffffffffu, q, o, 8));
  if (sub8 == 0) {
    const int which = col / kB, j = col % kB;
    if (j < b) {
      if (first)
        zeta[(size_t)which * b + j] = q;  // v.v and v.w1, probe j
      else if (dbl)
        zeta[(size_t)(2 * kmom + which) * b + j] = q;  // w_k.w_k, w_k.w_{k+1}
      else if (which == 0)
        zeta[(size_t)kmom * b + j] = q;
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Pipelined direct-gather block step (default for even probe counts): no shared-memory staging;
// a warp sweeps 4 rows at a time, 8 lanes per row, each lane owning a probe pair (16-byte loads
// and stores).  The three dependent fetches of a row batch are software-pipelined across batches: the row pointers of batch k+2 and the
// (col, val) entries of batch k+1 -- loaded cooperatively, one coalesced load per warp, since
// the 4 rows' entries are contiguous -- are in flight while batch k's probe rows are gathered
// and reduced.  Entries reach their row's lanes by warp shuffles.  Batches whose rows exceed U
// entries (or 32 together) take the plain per-lane loop.  Same storage-order sums.
template <int U, int BC>
__global__ void __launch_bounds__(kKpmThreads, 3) k_kpm_stream(
    int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ vals,
    int b_rt, int mode, const double* __restrict__ v, const double* __restrict__ w0,
    const double* __restrict__ w1, double* __restrict__ t, double cc, double d,
    double* __restrict__ partial, unsigned* counter, double* __restrict__ zeta, int kmom) {
  const int b = BC > 0 ? BC : b_rt;  // compile-time probe count for the common block widths
  const double dinv = 1.0 / d;        // correctly rounded; div_by corrects each quotient
  const bool first = mode == kKpmFirst;
  const bool dbl = mode == kKpmDoubling;
  const int lane = threadIdx.x & 31, g = lane >> 3, l8 = lane & 7;
  const bool live = 2 * l8 < b;  // b even
  const double* __restrict__ src = first ? w0 : w1;
  const int warps = (int)(gridDim.x * (kKpmThreads / 32));
  const int nb = (n + 3) / 4;
  auto load_rp = [&](int rb) -> int {  // lane i (<= 4): rp[4 rb + i] (clamped to n)
    return rb < nb ? __ldg(rp + min(4 * rb + min(lane, 4), n)) : 0;
  };
  auto load_ent = [&](int rb, int rpv, int& c, double& a) {  // lane i: entry base + i
    const int base = __shfl_sync(0xffffffffu, rpv, 0), end = __shfl_sync(0xffffffffu, rpv, 4);
    c = 0;
    a = 0.0;
    if (rb < nb && lane < end - base) {
      c = __ldg(ci + base + lane);
      a = __ldg(vals + base + lane);
    }
  };
  auto prefetch_rows = [&](int rb1, int rpv, int c) {  // batch rb1's probe rows -> L2
    if (rb1 >= nb) return;
    const int base = __shfl_sync(0xffffffffu, rpv, 0), end = __shfl_sync(0xffffffffu, rpv, 4);
    if (lane < end - base) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (size_t)c * b));
    const int r1 = 4 * rb1 + (lane & 3);
    if (r1 < n) {
      if (lane >= 28 && !first) asm volatile("prefetch.global.L2 [%0];" ::"l"(w0 + (size_t)r1 * b));
      if (lane >= 24 && lane < 28 && !dbl) asm volatile("prefetch.global.L2 [%0];" ::"l"(v + (size_t)r1 * b));
    }
  };
  int rb = (int)(blockIdx.x * (kKpmThreads / 32) + (threadIdx.x >> 5));
  // pipeline: row pointers two batches ahead, entries one batch ahead, probe rows of the next
  // batch prefetched into L2
  int rp_cur = load_rp(rb), rp_nxt = load_rp(rb + warps), c_cur, c_nxt;
  double a_cur, a_nxt;
  load_ent(rb, rp_cur, c_cur, a_cur);
  load_ent(rb + warps, rp_nxt, c_nxt, a_nxt);
  int rp_nn = load_rp(rb + 2 * warps);
  double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
  for (; rb < nb; rb += warps) {
    int c_nn;
    double a_nn;
    load_ent(rb + 2 * warps, rp_nn, c_nn, a_nn);
    const int rp_n3 = load_rp(rb + 3 * warps);
    prefetch_rows(rb + warps, rp_nxt, c_nxt);
    const int base = __shfl_sync(0xffffffffu, rp_cur, 0);
    const int cnt = __shfl_sync(0xffffffffu, rp_cur, 4) - base;
    const int rs = __shfl_sync(0xffffffffu, rp_cur, g), re = __shfl_sync(0xffffffffu, rp_cur, g + 1);
    const int r = 4 * rb + g;
    const bool on = r < n && live;
    const size_t o = (size_t)r * b + 2 * l8;
    double2 xr = make_double2(0.0, 0.0), vr = xr, pr = xr;
    if (on) {
      xr = __ldg(reinterpret_cast<const double2*>(src + o));
      if (!dbl) vr = __ldg(reinterpret_cast<const double2*>(v + o));
      if (!first) pr = __ldg(reinterpret_cast<const double2*>(w0 + o));
    }
    double2 acc = make_double2(0.0, 0.0);
    const int len = on ? re - rs : 0;  // off lanes (rows past n, probes past b) gather nothing
    if (cnt <= 32 && __all_sync(0xffffffffu, len <= U)) {
      double2 x[U];
      double av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sl = min(rs - base + u, 31);
        const int cu = __shfl_sync(0xffffffffu, c_cur, sl);
        av[u] = __shfl_sync(0xffffffffu, a_cur, sl);
        x[u] = make_double2(0.0, 0.0);
        if (u < len) x[u] = __ldg(reinterpret_cast<const double2*>(src + (size_t)cu * b + 2 * l8));
      }
      // past the row's end x[u] = 0: acc + av * 0 leaves acc unchanged (no select needed)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x = add(acc.x, mul(av[u], x[u].x));
        acc.y = add(acc.y, mul(av[u], x[u].y));
      }
    } else if (on) {
      for (int p = rs; p < re; ++p) {
        const double a = __ldg(vals + p);
        const double2 xv = __ldg(reinterpret_cast<const double2*>(src + (size_t)__ldg(ci + p) * b + 2 * l8));
        acc.x = add(acc.x, mul(a, xv.x));
        acc.y = add(acc.y, mul(a, xv.y));
      }
    }
    if (on) {
      // (A w - c w) / d   (dos.hpp:99)
      const double2 m = make_double2(div_by(sub(acc.x, mul(cc, xr.x)), d, dinv),
                                     div_by(sub(acc.y, mul(cc, xr.y)), d, dinv));
      double2* to = reinterpret_cast<double2*>(t + o);
      if (first) {
        *to = m;
        a0.x = add(a0.x, mul(vr.x, xr.x));
        a0.y = add(a0.y, mul(vr.y, xr.y));
        a1.x = add(a1.x, mul(vr.x, m.x));
        a1.y = add(a1.y, mul(vr.y, m.y));
      } else {
        const double2 tk = make_double2(sub(mul(2.0, m.x), pr.x), sub(mul(2.0, m.y), pr.y));
        *to = tk;
        if (dbl) {
          a0.x = add(a0.x, mul(xr.x, xr.x));
          a0.y = add(a0.y, mul(xr.y, xr.y));
          a1.x = add(a1.x, mul(xr.x, tk.x));
          a1.y = add(a1.y, mul(xr.y, tk.y));
        } else {
          a0.x = add(a0.x, mul(vr.x, tk.x));
          a0.y = add(a0.y, mul(vr.y, tk.y));
        }
      }
    }
    rp_cur = rp_nxt;
    rp_nxt = rp_nn;
    rp_nn = rp_n3;
    c_cur = c_nxt;
    a_cur = a_nxt;
    c_nxt = c_nn;
    a_nxt = a_nn;
  }
  __shared__ double s_a0[kKpmThreads / 8][kB], s_a1[kKpmThreads / 8][kB];
  const int grp = threadIdx.x >> 3;
  s_a0[grp][2 * l8] = a0.x;
  s_a0[grp][2 * l8 + 1] = a0.y;
  s_a1[grp][2 * l8] = a1.x;
  s_a1[grp][2 * l8 + 1] = a1.y;
  __syncthreads();
  const int h = threadIdx.x / kB, j = threadIdx.x % kB;
  const double f0 = add(s_a0[2 * h][j], s_a0[2 * h + 1][j]);
  const double f1 = add(s_a1[2 * h][j], s_a1[2 * h + 1][j]);
  __syncthreads();
  kpm_finish(f0, f1, b, first, dbl, partial, counter, zeta, kmom);
}

// Padded-row (ELL) block step: the default for matrices whose rows hold at most kEllW entries
// (stencils).  The matrix is kept a second time as ec/ea[n][kEllW] (rows padded with col = row,
// val = 0: acc + 0 * x leaves the storage-order sum unchanged), so a row's entries are two
// 16-byte column loads and four 16-byte value loads that the 8 lanes of the row share (L1
// broadcast): no row pointers, no shuffles, no per-entry predicates.  Column indices are loaded
// one batch ahead; separately each lane loads one column of the batch PD ahead (a coalesced
// load) and prefetches that probe row into L2, so a batch's gathers are (mostly) L2 hits.  The mode is a template argument (no runtime branches in the loop).
// Same lane mapping as k_kpm_stream (8 lanes x 2 probes per row, 4 rows per warp), same sums.
template <int MODE, int BC, int PD>
__global__ void __launch_bounds__(kKpmThreads, kEllMinB) k_kpm_ell(
    int n, const int* __restrict__ ec, const double* __restrict__ ea, int b_rt,
    const double* __restrict__ v, const double* __restrict__ w0, const double* __restrict__ w1,
    double* __restrict__ t, double cc, double d, double* __restrict__ partial, unsigned* counter,
    double* __restrict__ zeta, int kmom) {
  constexpr bool first = MODE == kKpmFirst, dbl = MODE == kKpmDoubling;
  const int b = BC > 0 ? BC : b_rt;
  const double dinv = 1.0 / d;
  const int lane = threadIdx.x & 31, g = lane >> 3, l8 = lane & 7;
  const bool live = 2 * l8 < b;
  const double* __restrict__ src = first ? w0 : w1;
  const int warps = (int)(gridDim.x * (kKpmThreads / 32));
  const int nb = (n + 3) / 4;
  int rb = (int)(blockIdx.x * (kKpmThreads / 32) + (threadIdx.x >> 5));
  auto load_cols = [&](int rbq, int4& lo, int4& hi) {
    const int r = 4 * rbq + g;
    lo = make_int4(0, 0, 0, 0);
    hi = lo;
    if (rbq < nb && r < n) {
      lo = __ldg(reinterpret_cast<const int4*>(ec + (size_t)r * kEllW));
      hi = __ldg(reinterpret_cast<const int4*>(ec + (size_t)r * kEllW + 4));
    }
  };
  // prefetch path: lane (g, l8) loads entry l8 of row g of batch rb + PD warps (one coalesced
  // 128-byte load per warp), and one iteration later prefetches that probe row into L2
  auto pf_col = [&](int rbq) -> int {
    return (rbq < nb && 4 * rbq + g < n) ? __ldg(ec + (size_t)rbq * 32 + lane) : -1;
  };
  int4 cl, ch;
  load_cols(rb, cl, ch);
  int pc = pf_col(rb + (PD - 1) * warps);
  double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
  for (; rb < nb; rb += warps) {
    int4 nl, nh;
    load_cols(rb + warps, nl, nh);
    const int pn = pf_col(rb + PD * warps);
    if (pc >= 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src + (size_t)pc * b));
      if (!first && l8 == 0)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(w0 + (size_t)(4 * (rb + (PD - 1) * warps) + g) * b));
    }
    pc = pn;
    const int r = 4 * rb + g;
    if (r < n && live) {
      const size_t o = (size_t)r * b + 2 * l8;
      const int cs[kEllW] = {cl.x, cl.y, cl.z, cl.w, ch.x, ch.y, ch.z, ch.w};
      double2 x[kEllW];
#pragma unroll
      for (int u = 0; u < kEllW; ++u)
        x[u] = __ldg(reinterpret_cast<const double2*>(src + (size_t)cs[u] * b + 2 * l8));
      // the row's own probe row: the pad slot (col = row) when the row is not full
      const double2 xr = cs[kEllW - 1] == r ? x[kEllW - 1]
                                            : __ldg(reinterpret_cast<const double2*>(src + o));
      double2 vr = make_double2(0.0, 0.0), pr = vr;
      if (!dbl) vr = __ldg(reinterpret_cast<const double2*>(v + o));
      if (!first) pr = __ldg(reinterpret_cast<const double2*>(w0 + o));
      const double2* ap = reinterpret_cast<const double2*>(ea + (size_t)r * kEllW);
      double av[kEllW];
#pragma unroll
      for (int q = 0; q < kEllW / 2; ++q) {
        const double2 e = __ldg(ap + q);
        av[2 * q] = e.x;
        av[2 * q + 1] = e.y;
      }
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < kEllW; ++u) {
        acc.x = add(acc.x, mul(av[u], x[u].x));
        acc.y = add(acc.y, mul(av[u], x[u].y));
      }
      // (A w - c w) / d   (dos.hpp:99)
      const double2 m = make_double2(div_by(sub(acc.x, mul(cc, xr.x)), d, dinv),
                                     div_by(sub(acc.y, mul(cc, xr.y)), d, dinv));
      double2* to = reinterpret_cast<double2*>(t + o);
      if (first) {
        *to = m;
        a0.x = add(a0.x, mul(vr.x, xr.x));
        a0.y = add(a0.y, mul(vr.y, xr.y));
        a1.x = add(a1.x, mul(vr.x, m.x));
        a1.y = add(a1.y, mul(vr.y, m.y));
      } else {
        const double2 tk = make_double2(sub(mul(2.0, m.x), pr.x), sub(mul(2.0, m.y), pr.y));
        *to = tk;
        if (dbl) {
          a0.x = add(a0.x, mul(xr.x, xr.x));
          a0.y = add(a0.y, mul(xr.y, xr.y));
          a1.x = add(a1.x, mul(xr.x, tk.x));
          a1.y = add(a1.y, mul(xr.y, tk.y));
        } else {
          a0.x = add(a0.x, mul(vr.x, tk.x));
          a0.y = add(a0.y, mul(vr.y, tk.y));
        }
      }
    }
    cl = nl;
    ch = nh;
  }
  __shared__ double s_a0[kKpmThreads / 8][kB], s_a1[kKpmThreads / 8][kB];
  const int grp = threadIdx.x >> 3;
  s_a0[grp][2 * l8] = a0.x;
  s_a0[grp][2 * l8 + 1] = a0.y;
  s_a1[grp][2 * l8] = a1.x;
  s_a1[grp][2 * l8 + 1] = a1.y;
  __syncthreads();
  const int h = threadIdx.x / kB, j = threadIdx.x % kB;
  const double f0 = add(s_a0[2 * h][j], s_a0[2 * h + 1][j]);
  const double f1 = add(s_a1[2 * h][j], s_a1[2 * h + 1][j]);
  __syncthreads();
  kpm_finish(f0, f1, b, first, dbl, partial, counter, zeta, kmom);
}

// ---- block filter degree on a row-major vector block (K2, padded-row matrices) ------------------
// The block filter of cheb_si / the block apply_pol for matrices with <= kEllW entries per row
// (stencils): kBV = 8 vectors stored row-major (n x 8, one 64-byte line per row), 4 lanes x 2
// vectors per row, 8 rows per warp and sweep.  A row's entries are read once for all 8 vectors
// (two 16-byte column loads and four 16-byte value loads shared by the row's 4 lanes), every
// gather is a 16-byte piece of a 64-byte line, column indices are loaded one sweep ahead and the
// next sweep's gather rows are prefetched into L2 -- the structure of k_kpm_ell, with the
// filter's update (filter_poly.hpp:260-276) instead of the moment dots.  Row sums run in storage
// order with individually rounded products; the pad entries add 0 * x, so each vector's result is
// the single-vector kernel's (and the reference's) bit for bit.
constexpr int kBV = 8;
constexpr int kBlkThreads = 256;

template <bool FIRST>
__global__ void __launch_bounds__(kBlkThreads, 3) k_cheb_ell_block(
    int n, const int* __restrict__ ec, const double* __restrict__ ea,
    const double* __restrict__ X,     // T_{j-1} (FIRST: the input block v)
    const double* __restrict__ P,     // T_{j-2} (unused when FIRST)
    double* __restrict__ Y,           // T_j
    double* __restrict__ O,           // running sum (FIRST: written, else updated)
    double cc, double invd, double mu0, double muj) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, g = lane >> 2, l4 = lane & 3;
  const int warps = (int)(gridDim.x * (kBlkThreads / 32));
  const int nb = (n + 7) / 8;
  int rb = (int)(blockIdx.x * (kBlkThreads / 32) + (threadIdx.x >> 5));
  auto load_cols = [&](int rbq, int4& lo, int4& hi) {
    const int r = 8 * rbq + g;
    lo = make_int4(0, 0, 0, 0);
    hi = lo;
    if (rbq < nb && r < n) {
      lo = __ldg(reinterpret_cast<const int4*>(ec + (size_t)r * kEllW));
      hi = __ldg(reinterpret_cast<const int4*>(ec + (size_t)r * kEllW + 4));
    }
  };
  // prefetch: the 8 rows x 8 entries of the sweep one stride ahead are 64 column indices; lane
  // (g, l4) prefetches the rows named by entries l4 and l4 + 4 of row g
  int4 cl, ch;
  load_cols(rb, cl, ch);
  for (; rb < nb; rb += warps) {
    int4 nl, nh;
    load_cols(rb + warps, nl, nh);
    {
      const int c0 = l4 == 0 ? nl.x : l4 == 1 ? nl.y : l4 == 2 ? nl.z : nl.w;
      const int c1 = l4 == 0 ? nh.x : l4 == 1 ? nh.y : l4 == 2 ? nh.z : nh.w;
      if (rb + warps < nb && 8 * (rb + warps) + g < n) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (size_t)c0 * kBV));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (size_t)c1 * kBV));
      }
    }
    const int r = 8 * rb + g;
    if (r < n) {
      const size_t o = (size_t)r * kBV + 2 * l4;
      const int cs[kEllW] = {cl.x, cl.y, cl.z, cl.w, ch.x, ch.y, ch.z, ch.w};
      double2 x[kEllW];
#pragma unroll
      for (int u = 0; u < kEllW; ++u)
        x[u] = __ldg(reinterpret_cast<const double2*>(X + (size_t)cs[u] * kBV + 2 * l4));
      const double2 xr = cs[kEllW - 1] == r ? x[kEllW - 1]
                                            : __ldg(reinterpret_cast<const double2*>(X + o));
      double2 pr = make_double2(0.0, 0.0), ov = pr;
      if (!FIRST) {
        pr = __ldg(reinterpret_cast<const double2*>(P + o));
        ov = *reinterpret_cast<const double2*>(O + o);
      }
      const double2* ap = reinterpret_cast<const double2*>(ea + (size_t)r * kEllW);
      double av[kEllW];
#pragma unroll
      for (int q = 0; q < kEllW / 2; ++q) {
        const double2 e = __ldg(ap + q);
        av[2 * q] = e.x;
        av[2 * q + 1] = e.y;
      }
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < kEllW; ++u) {
        acc.x = add(acc.x, mul(av[u], x[u].x));
        acc.y = add(acc.y, mul(av[u], x[u].y));
      }
      // Ahat x = (A x - c x) * (1/d)   (filter_poly.hpp:265)
      const double2 t = make_double2(mul(sub(acc.x, mul(cc, xr.x)), invd),
                                     mul(sub(acc.y, mul(cc, xr.y)), invd));
      if (FIRST) {
        *reinterpret_cast<double2*>(Y + o) = t;
        *reinterpret_cast<double2*>(O + o) =
            make_double2(add(add(0.0, mul(mu0, xr.x)), mul(muj, t.x)),
                         add(add(0.0, mul(mu0, xr.y)), mul(muj, t.y)));
      } else {
        const double2 tj = make_double2(sub(mul(2.0, t.x), pr.x), sub(mul(2.0, t.y), pr.y));
        *reinterpret_cast<double2*>(Y + o) = tj;
        *reinterpret_cast<double2*>(O + o) =
            make_double2(add(ov.x, mul(muj, tj.x)), add(ov.y, mul(muj, tj.y)));
      }
    }
    cl = nl;
    ch = nh;
  }
}

// column-major (nv columns, ld n) -> row-major n x 8 (columns nv..7 zero), and back
__global__ void __launch_bounds__(256) k_block_pack(const double* __restrict__ cm, double* __restrict__ rm,
                                                    int n, int nv) {
  __shared__ double tile[kBV][33];
  const int i0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * kBV; e += 256) {
    const int l = e >> 5, i = e & 31;
    tile[l][i] = (l < nv && i0 + i < n) ? cm[(size_t)l * n + i0 + i] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kBV; e += 256) {
    const int i = e >> 3, l = e & 7;
    if (i0 + i < n) rm[(size_t)(i0 + i) * kBV + l] = tile[l][i];
  }
}
__global__ void __launch_bounds__(256) k_block_unpack(const double* __restrict__ rm, double* __restrict__ cm,
                                                      int n, int nv) {
  __shared__ double tile[kBV][33];
  const int i0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * kBV; e += 256) {
    const int i = e >> 3, l = e & 7;
    if (i0 + i < n) tile[l][i] = rm[(size_t)(i0 + i) * kBV + l];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kBV; e += 256) {
    const int l = e >> 5, i = e & 31;
    if (l < nv && i0 + i < n) cm[(size_t)l * n + i0 + i] = tile[l][i];
  }
}

// CSR -> padded rows (kEllW per row; pad col = row, val = 0), one thread per row
__global__ void k_build_ell(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, int* __restrict__ ec, double* __restrict__ ea) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int p = rp[r], e = rp[r + 1];
#pragma unroll
  for (int u = 0; u < kEllW; ++u) {
    const bool in = p + u < e;
    ec[(size_t)r * kEllW + u] = in ? ci[p + u] : r;
    ea[(size_t)r * kEllW + u] = in ? v[p + u] : 0.0;
  }
}

// Rademacher sign bits (probe-major, W words per probe) -> row-major n x bk doubles (+1 / -1;
// columns b .. bk-1 zero)
__global__ void k_expand_rademacher(const unsigned long long* __restrict__ bits, long W,
                                    double* __restrict__ rm, int n, int b, int bk) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long)n * bk) return;
  const int i = (int)(e / bk), l = (int)(e - (long)i * bk);
  double v = 0.0;
  if (l < b) v = ((__ldg(bits + l * W + (i >> 6)) >> (i & 63)) & 1ull) ? 1.0 : -1.0;
  rm[e] = v;
}

// probe-major (b x n) -> row-major (n x b), 32 rows per CTA through shared memory
__global__ void __launch_bounds__(256) k_transpose_probes(const double* __restrict__ pm,
                                                          double* __restrict__ rm, int n, int b) {
  __shared__ double tile[kB][33];
  const int i0 = blockIdx.x * 32;
  for (int e = threadIdx.x; e < 32 * b; e += 256) {
    const int l = e >> 5, i = e & 31;
    if (i0 + i < n) tile[l][i] = pm[(size_t)l * n + i0 + i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * b; e += 256) {
    const int i = e / b, l = e - i * b;
    if (i0 + i < n) rm[(size_t)(i0 + i) * b + l] = tile[l][i];
  }
}

// ---- device Laplacian generator (laplacian.hpp:19-48) -------------------------------------------
struct Grid {
  int nx, ny, nz, ndims;
};

__device__ __forceinline__ int lap_row_nnz(const Grid& g, int row) {
  const int i = row % g.nx, j = (row / g.nx) % g.ny, kk = row / (g.nx * g.ny);
  int c = 1 + (i > 0) + (i < g.nx - 1);
  if (g.ny > 1) c += (j > 0) + (j < g.ny - 1);
  if (g.nz > 1) c += (kk > 0) + (kk < g.nz - 1);
  return c;
}

__global__ void k_lap_count(Grid g, int n, int* cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) cnt[r] = lap_row_nnz(g, r);
  if (r == n) cnt[r] = 0;
}

// Entries in ascending column order: -nx*ny, -nx, -1, diag, +1, +nx, +nx*ny.
__global__ void k_lap_fill(Grid g, int n, const int* __restrict__ rp, int* __restrict__ ci,
                           double* __restrict__ v) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int i = r % g.nx, j = (r / g.nx) % g.ny, kk = r / (g.nx * g.ny);
  const int plane = g.nx * g.ny;
  int p = rp[r];
  if (g.nz > 1 && kk > 0) { ci[p] = r - plane; v[p++] = -1.0; }
  if (g.ny > 1 && j > 0) { ci[p] = r - g.nx; v[p++] = -1.0; }
  if (i > 0) { ci[p] = r - 1; v[p++] = -1.0; }
  ci[p] = r;
  v[p++] = 2.0 * (double)g.ndims;
  if (i < g.nx - 1) { ci[p] = r + 1; v[p++] = -1.0; }
  if (g.ny > 1 && j < g.ny - 1) { ci[p] = r + g.nx; v[p++] = -1.0; }
  if (g.nz > 1 && kk < g.nz - 1) { ci[p] = r + plane; v[p++] = -1.0; }
}

__global__ void k_scale_sym(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            double* __restrict__ v, const double* __restrict__ d) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double dr = d[r];
  for (int p = rp[r]; p < rp[r + 1]; ++p) v[p] = mul(mul(v[p], dr), d[ci[p]]);
}

__global__ void k_row_len_max(int n, const int* __restrict__ rp, int* out) {
  int m = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    m = max(m, rp[r + 1] - rp[r]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

void spmv_cheb(Ctx& c, const DevCsr& a, int mode, const ChebArgs& args) {
  if (a.n == 0) return;
  KArgs k{args.x, args.prev, args.y, args.out, args.c, args.invd, args.mu0, args.muj,
          args.src_ctl, args.src_ld, 0, 0, args.halt};
  // src_ctl indirection applies to the vector that is W[:, i]: x on the first degree, prev on
  // the second (filter_poly.hpp:260,268-272: prev = v until the first rotation).
  if (args.src_ctl) {
    k.x_indirect = (mode == kFirst || mode == kPlain);
    k.prev_indirect = (mode == kNext);
  }
  const int ntiles = (a.n + kRows - 1) / kRows;
  dim3 grid(ntiles, mode == kPlain ? args.ncols : 1);
  // The filter chain is latency-bound (k dependent launches per Lanczos step) while the slices'
  // reorthogonalisation passes sharing the GPU are bandwidth-bound: filter launches (and their
  // graph nodes) get the device's highest priority so their CTAs are scheduled ahead of queued
  // GEMV CTAs of other slices.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kRows);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  attr[na].id = cudaLaunchAttributePriority;
  attr[na].val.priority = c.prio_hi;
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  switch (mode) {
    case kPlain:
      SE_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_cheb<kPlain>, a.n, (const int*)a.rp, (const int*)a.ci,
                                 (const double*)a.v, k));
      break;
    case kFirst:
      SE_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_cheb<kFirst>, a.n, (const int*)a.rp, (const int*)a.ci,
                                 (const double*)a.v, k));
      break;
    default:
      SE_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_cheb<kNext>, a.n, (const int*)a.rp, (const int*)a.ci,
                                 (const double*)a.v, k));
  }
  ++c.launches;
}

size_t kpm_scratch_doubles(const Ctx& c, int n) {
  (void)n;
  return (size_t)2 * kB * c.num_sms * 8;  // per-CTA partials of the (<= 8 per SM) resident grid
}

void spmv_cheb_multi(Ctx& c, const DevCsr& a, const MultiArgs& args) {
  if (a.n == 0 || args.nv == 0) return;
  if (args.nv > kMV) fail(SE_EINVAL, "spmv_cheb_multi: too many vectors");
  // programmatic dependent launch (the A staging overlaps the previous degree's tail) and the
  // filter launches' high priority, as for k_spmv_cheb
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((a.n + kMRows - 1) / kMRows);
  cfg.blockDim = dim3(kMRows * kMV);
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = c.prio_hi;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  SE_CUDA(cudaLaunchKernelEx(&cfg, k_spmv_cheb_multi, a.n, (const int*)a.rp, (const int*)a.ci,
                             (const double*)a.v, args));
  ++c.launches;
}

bool cheb_block_available(const DevCsr& a) { return a.ell_c != nullptr && a.n > 0; }

void cheb_block_pack(Ctx& c, const double* cm, double* rm, int n, int nv) {
  k_block_pack<<<(n + 31) / 32, 256, 0, c.stream>>>(cm, rm, n, nv);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}
void cheb_block_unpack(Ctx& c, const double* rm, double* cm, int n, int nv) {
  k_block_unpack<<<(n + 31) / 32, 256, 0, c.stream>>>(rm, cm, n, nv);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}

void cheb_block_step(Ctx& c, const DevCsr& a, bool first, const double* X, const double* P,
                     double* Y, double* O, double cc, double invd, double mu0, double muj) {
  if (!a.ell_c) fail(SE_EINVAL, "internal: block filter needs the padded-row copy");
  // one contiguous sweep window: the grid is exactly the resident CTAs
  static int per_sm[2] = {0, 0};
  int& occ = per_sm[first ? 1 : 0];
  if (occ == 0) {
    if (first)
      SE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cheb_ell_block<true>, kBlkThreads, 0));
    else
      SE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cheb_ell_block<false>, kBlkThreads, 0));
    occ = std::max(occ, 1);
  }
  const int nb = (a.n + 7) / 8;
  const int want = (nb + kBlkThreads / 32 - 1) / (kBlkThreads / 32);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::max(1, std::min(want, occ * c.num_sms)));
  cfg.blockDim = dim3(kBlkThreads);
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = c.prio_hi;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (first)
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_ell_block<true>, a.n, (const int*)a.ell_c,
                               (const double*)a.ell_a, X, P, Y, O, cc, invd, mu0, muj));
  else
    SE_CUDA(cudaLaunchKernelEx(&cfg, k_cheb_ell_block<false>, a.n, (const int*)a.ell_c,
                               (const double*)a.ell_a, X, P, Y, O, cc, invd, mu0, muj));
  ++c.launches;
}

void expand_rademacher(Ctx& c, const std::uint64_t* bits, double* rm, int n, int b, int bk) {
  if (n == 0 || bk == 0) return;
  if (bk > kB || b > bk) fail(SE_EINVAL, "expand_rademacher: block too wide");
  const long tot = (long)n * bk;
  k_expand_rademacher<<<(unsigned)((tot + 255) / 256), 256, 0, c.stream>>>(
      reinterpret_cast<const unsigned long long*>(bits), ((long)n + 63) / 64, rm, n, b, bk);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void transpose_probes(Ctx& c, const double* pm, double* rm, int n, int b) {
  if (n == 0 || b == 0) return;
  if (b > kB) fail(SE_EINVAL, "transpose_probes: block too wide");
  k_transpose_probes<<<(n + 31) / 32, 256, 0, c.stream>>>(pm, rm, n, b);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void kpm_step(Ctx& c, const Scratch& s, const DevCsr& a, int b, int mode, const double* v,
              const double* w0, const double* w1, double* t, double cc, double d, double* zeta_dev,
              int kmom) {
  if (kpm_scratch_doubles(c, a.n) > s.cap || s.ncnt < 1) fail(SE_EINVAL, "internal: kpm scratch");
  if (b % 2 != 0) fail(SE_EINVAL, "internal: kpm blocks carry an even probe count");
  // Matrices with <= kEllW entries per row (stencils) keep a padded-row copy: the ELL kernel.
  // Longer rows (random sparse, cfg4) stream the CSR entries.
  if (a.ell_c) {
    using EFn = decltype(&k_kpm_ell<0, 16, kKpmPD>);
    auto pick = [&](auto md) -> EFn {
      constexpr int M = decltype(md)::value;
      return b == 16 ? k_kpm_ell<M, 16, kKpmPD> : b == 8 ? k_kpm_ell<M, 8, kKpmPD> : k_kpm_ell<M, 0, kKpmPD>;
    };
    const EFn kern = mode == kKpmFirst      ? pick(std::integral_constant<int, kKpmFirst>{})
                     : mode == kKpmDoubling ? pick(std::integral_constant<int, kKpmDoubling>{})
                                            : pick(std::integral_constant<int, 0>{});
    static const int per_sm = [] {
      int v = 0;
      SE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_kpm_ell<kKpmDoubling, 16, kKpmPD>, kKpmThreads, 0));
      return std::max(1, std::min(v, 8));
    }();
    const int grid = std::max(1, std::min(c.num_sms * per_sm, (a.n + 31) / 32));
    kern<<<grid, kKpmThreads, 0, c.stream>>>(a.n, a.ell_c, a.ell_a, b, v, w0, w1, t, cc, d, s.buf, s.cnt,
                                             zeta_dev, kmom);
    ++c.launches;
    SE_CUDA(cudaGetLastError());
    return;
  }
  static const int per_sm = [] {
    int v = 0;
    SE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_kpm_stream<8, 0>, kKpmThreads, 0));
    return std::max(1, std::min(v, 8));
  }();
  const int grid = std::max(1, std::min(c.num_sms * per_sm, (a.n + 31) / 32));
  // U = entries gathered per row in one round: the matrix's row length (stencils: 5 or 7)
  using KFn = decltype(&k_kpm_stream<8, 0>);
  auto pick = [&](auto u) -> KFn {
    constexpr int U = decltype(u)::value;
    return b == 16 ? k_kpm_stream<U, 16> : b == 8 ? k_kpm_stream<U, 8> : k_kpm_stream<U, 0>;
  };
  const KFn kern = a.max_row_nnz <= 5 ? pick(std::integral_constant<int, 5>{})
                   : a.max_row_nnz <= 7 ? pick(std::integral_constant<int, 7>{})
                                        : pick(std::integral_constant<int, 8>{});
  kern<<<grid, kKpmThreads, 0, c.stream>>>(a.n, a.rp, a.ci, a.v, b, mode, v, w0, w1, t, cc, d, s.buf,
                                           s.cnt, zeta_dev, kmom);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void build_ell(Ctx& c, DevCsr& a) {
  if (!a.resident) resident_build(c, a);  // the pattern is in place: plan the resident filter
  if (a.n == 0 || a.max_row_nnz > kEllW) return;
  if (!a.ell_c) {
    a.ell_c = dev_alloc_shared<int>((size_t)a.n * kEllW);
    a.ell_a = dev_alloc_shared<double>((size_t)a.n * kEllW);
  }
  k_build_ell<<<(a.n + 255) / 256, 256, 0, c.stream>>>(a.n, a.rp, a.ci, a.v, a.ell_c, a.ell_a);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void gen_laplacian(Ctx& c, int ndims, const int* dims, DevCsr& a) {
  Grid g{dims[0], ndims > 1 ? dims[1] : 1, ndims > 2 ? dims[2] : 1, ndims};
  const long nl = (long)g.nx * g.ny * g.nz;
  const int n = (int)nl;
  a.n = n;
  a.rp = dev_alloc_shared<int>(n + 1);
  const int tb = 256;
  k_lap_count<<<(n + 1 + tb - 1) / tb, tb, 0, c.stream>>>(g, n, a.rp);
  ++c.launches;
  size_t tmp_bytes = 0;
  SE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, a.rp, a.rp, n + 1, c.stream));
  void* tmp = dev_alloc<char>(tmp_bytes);
  SE_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, a.rp, a.rp, n + 1, c.stream));
  ctx_sync(c);
  dev_free(tmp);
  int nnz = 0;
  SE_CUDA(cudaMemcpyAsync(&nnz, a.rp + n, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  ctx_sync(c);
  a.nnz = nnz;
  a.alloc_entries(nnz);
  k_lap_fill<<<(n + tb - 1) / tb, tb, 0, c.stream>>>(g, n, a.rp, a.ci, a.v);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
  a.max_row_nnz = 1 + 2 * ndims;
  build_ell(c, a);
}

void csr_scale_sym(Ctx& c, DevCsr& a, const double* d_dev) {
  if (a.n == 0) return;
  k_scale_sym<<<(a.n + 255) / 256, 256, 0, c.stream>>>(a.n, a.rp, a.ci, a.v, d_dev);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
  build_ell(c, a);  // the padded copy follows the scaled values
}

int csr_max_row_nnz(Ctx& c, const DevCsr& a) {
  if (a.n == 0) return 0;
  int* d = dev_alloc<int>(1);
  SE_CUDA(cudaMemsetAsync(d, 0, sizeof(int), c.stream));
  k_row_len_max<<<std::min(c.num_sms * 4, (a.n + 255) / 256), 256, 0, c.stream>>>(a.n, a.rp, d);
  ++c.launches;
  int h = 0;
  SE_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  ctx_sync(c);
  dev_free(d);
  return h;
}

}  // namespace k
}  // namespace se
