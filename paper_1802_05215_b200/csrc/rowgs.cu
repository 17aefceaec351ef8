// Row-major Krylov basis and the three-read CGS2 step (K4 of SURVEY.md §2.1; reference
// orth.hpp:19-80 cgs_pass / paired_cgs2, eigensolvers.hpp:406-433 / 524-556 for the step).
//
// Layout: the Lanczos basis W is stored ROW-major, W[r * ldw + j] (ldw = column capacity, even),
// so one row of the active basis (columns 0..i) is a single contiguous run of 8 (i+1) bytes and
// a block of rows can be held by a CTA in registers.  That lets the middle of CGS2 use each row
// block twice from ONE read:
//
//   T1  : coef1 = W^T t                    (and ||t|| for the TR step)          one read of W
//   MID : t1 = t - W coef1, ||t1||, coef2 = W^T t1   (same rows, registers)     one read of W
//   N2  : t2 = t1 - W coef2, ||t2||        (only when the DGKS test asks, orth.hpp:76-78)
//
// i.e. three reads of W per re-passed CGS2 step instead of the four of two column-major passes,
// and two when no re-pass is needed (coef2 is then simply discarded).  A TMA-staged variant
// (cp.async.bulk row copies into a shared-memory mbarrier ring) was measured first and lost to
// the register-direct kernel at every basis width (profiles/r2_ncu_summary.md).
//
// The basis is written one column at a time (k_rw_normalize: W[:, i+1] = t / beta) and read one
// column at a time by the filter (k_rw_col_get): strided 8-byte accesses, ~4 n sectors per step,
// negligible next to the 8 n (i+1) bytes of each pass.
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

constexpr double kEta = 0.70710678118654752;  // DGKS threshold, orth.hpp:13
constexpr int kRT = 256;                      // threads per streaming CTA
constexpr int kRW = kRT / 32;
constexpr int kRwPerSm = 2;                   // resident streaming CTAs per SM (persistent grid)
constexpr int kFinCols = 32;                  // columns per finishing CTA (8 threads each)

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

enum RwPhase { kT = 0, kMid = 1, kN = 2 };

// The streaming pass.  PH = kT: part[g][j] = sum over this CTA's rows of W[r, j] t[r];
// npart[g] = sum t[r]^2.  PH = kMid: t[r] -= W[r, :] coef (written back), npart = sum t1^2,
// part = W^T t1 partials.  PH = kN (only when ctl->repass): t[r] -= W[r, :] coef, npart.
//
// Row blocks of R rows are dealt round-robin over a persistent grid (2 CTAs per SM).  Every
// thread owns the column PAIRS j2 = tid + 256 q (q < QP) and loads them for the block's R rows
// straight into registers -- R x QP independent 16-byte streaming loads in flight per thread,
// ~100 KB per SM -- then uses the same registers for the row dots W[r, :] coef (MID / N) and for
// the W^T x partial sums (T / MID): one read of the row block serves both halves of the fused
// step.  Coefficients and partials live in registers; the row dots are reduced by the warp xor
// tree and then over the warps in order, so the sums are deterministic.
template <int PH, int QP, int R>
__global__ void __launch_bounds__(kRT, 2) k_rw_stream(int n, const double* __restrict__ W, int ldw,
                                                      double* __restrict__ t, const Ctl* ctl,
                                                      const double* __restrict__ coef,
                                                      double* __restrict__ part,
                                                      double* __restrict__ npart, int) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  if (PH == kN && !ctl->repass) return;
  const int ncols = ctl->i + 1;
  const int np = (ncols + 1) >> 1;
  const int nblk = (n + R - 1) / R;
  __shared__ double s_red[2][kRW][R];  // double-buffered: one barrier per row block
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2 cr[QP], acc[QP];
#pragma unroll
  for (int q = 0; q < QP; ++q) {
    const int j2 = tid + kRT * q;
    cr[q] = make_double2(0.0, 0.0);
    if (PH != kT && j2 < np) {
      cr[q].x = coef[2 * j2];
      cr[q].y = 2 * j2 + 1 < ncols ? coef[2 * j2 + 1] : 0.0;
    }
    acc[q] = make_double2(0.0, 0.0);
  }
  double nrm = 0.0;
  int it = 0;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x, ++it) {
    const int r0 = b * R, rows = min(R, n - r0);
    double2 w[R][QP];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < QP; ++q) {
        const int j2 = tid + kRT * q;
        w[r][q] = (r < rows && j2 < np)
                      ? __ldcs(reinterpret_cast<const double2*>(W + (size_t)(r0 + r) * ldw) + j2)
                      : make_double2(0.0, 0.0);
      }
    // the block's t rows, read by every thread before anything is written back
    double x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = r < rows ? t[r0 + r] : 0.0;
    if (PH != kT) {
      // row dots W[r, :] coef: own pairs, warp xor tree, then the warps in order (every thread
      // forms the same sums from the shared partials)
      double (*red)[R] = s_red[it & 1];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < QP; ++q) p = fma(w[r][q].y, cr[q].y, fma(w[r][q].x, cr[q].x, p));
        p = warp_sum(p);
        if (lane == 0) red[warp][r] = p;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double sum = 0.0;
#pragma unroll
        for (int v = 0; v < kRW; ++v) sum = add(sum, red[v][r]);
        x[r] = r < rows ? sub(x[r], sum) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (tid == r && r < rows) t[r0 + r] = x[r];
    }
    if (tid == 0)
      for (int r = 0; r < rows; ++r) nrm = fma(x[r], x[r], nrm);
    if (PH != kN) {
#pragma unroll
      for (int q = 0; q < QP; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[q].x = fma(w[r][q].x, x[r], acc[q].x);
          acc[q].y = fma(w[r][q].y, x[r], acc[q].y);
        }
    }
  }
  if (PH != kN) {
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const int j2 = tid + kRT * q;
      if (2 * j2 < ncols) part[(size_t)blockIdx.x * ldw + 2 * j2] = acc[q].x;
      if (2 * j2 + 1 < ncols) part[(size_t)blockIdx.x * ldw + 2 * j2 + 1] = acc[q].y;
    }
  }
  if (tid == 0) npart[blockIdx.x] = nrm;
}

// Narrow bases (<= 512 columns): a warp owns whole rows (lane = column pairs j2 = lane + 32 q),
// so the row dots need only the warp's xor tree -- no CTA barrier in the loop -- and each warp
// streams RW rows per iteration on its own.  Partial sums are per warp and combined over the
// CTA's warps in order at the end, so the result is again deterministic.
template <int PH, int Q, int RW>
__global__ void __launch_bounds__(kRT, 2) k_rw_warp(int n, const double* __restrict__ W, int ldw,
                                                    double* __restrict__ t, const Ctl* ctl,
                                                    const double* __restrict__ coef,
                                                    double* __restrict__ part,
                                                    double* __restrict__ npart, int) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  if (PH == kN && !ctl->repass) return;
  const int ncols = ctl->i + 1;
  const int np = (ncols + 1) >> 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kRW + warp, nw = gridDim.x * kRW;  // global warp id / count
  const int nblk = (n + RW - 1) / RW;
  __shared__ double2 s_acc[kRW][Q * 32];
  __shared__ double s_nrm[kRW];
  double2 cr[Q], acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int j2 = lane + 32 * q;
    cr[q] = make_double2(0.0, 0.0);
    if (PH != kT && j2 < np) {
      cr[q].x = coef[2 * j2];
      cr[q].y = 2 * j2 + 1 < ncols ? coef[2 * j2 + 1] : 0.0;
    }
    acc[q] = make_double2(0.0, 0.0);
  }
  double nrm = 0.0;  // lane 0: this warp's sum of squares, in row order
  for (int b = gw; b < nblk; b += nw) {
    const int r0 = b * RW, rows = min(RW, n - r0);
    double2 w[RW][Q];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j2 = lane + 32 * q;
        w[r][q] = (r < rows && j2 < np)
                      ? __ldcs(reinterpret_cast<const double2*>(W + (size_t)(r0 + r) * ldw) + j2)
                      : make_double2(0.0, 0.0);
      }
    double x[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) x[r] = r < rows ? t[r0 + r] : 0.0;
    if (PH != kT) {
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) p = fma(w[r][q].y, cr[q].y, fma(w[r][q].x, cr[q].x, p));
        p = warp_sum(p);
        x[r] = r < rows ? sub(x[r], p) : 0.0;
      }
      if (lane < rows) {
#pragma unroll
        for (int r = 0; r < RW; ++r)
          if (lane == r) t[r0 + r] = x[r];
      }
    }
    if (lane == 0)
      for (int r = 0; r < rows; ++r) nrm = fma(x[r], x[r], nrm);
    if (PH != kN) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          acc[q].x = fma(w[r][q].x, x[r], acc[q].x);
          acc[q].y = fma(w[r][q].y, x[r], acc[q].y);
        }
    }
  }
  // combine the CTA's warps in order
  if (PH != kN)
#pragma unroll
    for (int q = 0; q < Q; ++q) s_acc[warp][lane + 32 * q] = acc[q];
  if (lane == 0) s_nrm[warp] = nrm;
  __syncthreads();
  if (PH != kN)
    for (int j2 = threadIdx.x; j2 < np; j2 += kRT) {
      double2 a = make_double2(0.0, 0.0);
#pragma unroll
      for (int v = 0; v < kRW; ++v) {
        a.x = add(a.x, s_acc[v][j2].x);
        a.y = add(a.y, s_acc[v][j2].y);
      }
      if (2 * j2 < ncols) part[(size_t)blockIdx.x * ldw + 2 * j2] = a.x;
      if (2 * j2 + 1 < ncols) part[(size_t)blockIdx.x * ldw + 2 * j2 + 1] = a.y;
    }
  if (threadIdx.x == 0) {
    double q = 0.0;
    for (int v = 0; v < kRW; ++v) q = add(q, s_nrm[v]);
    npart[blockIdx.x] = q;
  }
}

// sum of the G per-CTA squares, identical in every CTA (fixed thread assignment + tree)
__device__ double grid_norm2(const double* npart, int G) {
  __shared__ double s_w[kRW];
  __shared__ double s_tot;
  double v = 0.0;
  for (int g = threadIdx.x; g < G; g += kRT) v = add(v, __ldcg(npart + g));
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double q = 0.0;
    for (int w = 0; w < kRW; ++w) q = add(q, s_w[w]);
    s_tot = q;
  }
  __syncthreads();
  return s_tot;
}

// Finish a pass: coefficients (8 threads per column over the CTA partials, fixed order), the
// norm, the DGKS bookkeeping (orth.hpp:72-78) and TR's H(i,i) += h[i] (eigensolvers.hpp:534).
//   kT  : coef = sum part; hdiag[i] += coef[i]; want_before: before = after = ||t||, flags reset
//   kMid: after = ||t1||; repass = !(after > eta before); coef = sum part (coef2);
//         hdiag[i] += coef2[i] when the re-pass runs; pass statistics
//   kN  : (grid 1, only when re-passed) before = after = ||t2||; pass statistics
template <int PH>
__global__ void __launch_bounds__(kRT) k_rw_finish(int G, int ldw, const double* part,
                                                   const double* npart, Ctl* ctl, double* coef,
                                                   double* hdiag, int want_before) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  if (PH == kN && !ctl->repass) return;
  const int ncols = ctl->i + 1, icol = ctl->i;
  const double nrm = sqrt(grid_norm2(npart, G));
  if (PH == kN) {
    if (threadIdx.x == 0) {
      ctl->before = nrm;
      ctl->after = nrm;
      ctl->npass += 1;
      ctl->passes_total += 1;
      ctl->cols_total += ncols;
      ctl->reads_cols += ncols;
    }
    return;
  }
  // every CTA reads ctl->before, which only CTA 0 of the T finish writes (before the MID kernel)
  const bool repass = PH == kMid ? !(nrm > kEta * ctl->before) : false;
  const int jj = threadIdx.x >> 3, sub8 = threadIdx.x & 7;
  const int j = blockIdx.x * kFinCols + jj;
  double q = 0.0;
  if (j < ncols)
    for (int g = sub8; g < G; g += 8) q = add(q, __ldcg(part + (size_t)g * ldw + j));
  for (int o = 4; o > 0; o >>= 1) q = add(q, __shfl_down_sync(0xffffffffu, q, o, 8));
  if (sub8 == 0 && j < ncols) {
    coef[j] = q;
    if (hdiag && j == icol && (PH == kT || repass)) hdiag[j] = add(hdiag[j], q);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->reads_cols += ncols;
    if (PH == kT) {
      if (want_before) {
        ctl->before = nrm;
        ctl->after = nrm;
        ctl->repass = 0;
        ctl->npass = 0;
      }
    } else {
      ctl->after = nrm;  // `before` stays the pre-pass norm (other CTAs of this grid read it)
      ctl->repass = repass ? 1 : 0;
      ctl->npass += 1;
      ctl->passes_total += 1;
      ctl->cols_total += ncols;
    }
  }
}

// dst = W[:, ctl->i + off] (the filter's source column, contiguous)
__global__ void k_rw_col_get(int n, const double* __restrict__ W, int ldw, const Ctl* ctl, int off,
                             double* __restrict__ dst) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const int col = ctl->i + off;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    dst[r] = W[(size_t)r * ldw + col];
}

// beta = after; breakdown (beta <= 1e-14, orth.hpp:14) halts the recurrence; otherwise
// W[:, i+1] = t * (1/beta) (eigensolvers.hpp:431), beta_arr[i] = beta, i += 1.
__global__ void k_rw_normalize(int n, const double* __restrict__ t, double* __restrict__ W, int ldw,
                               Ctl* ctl, double* beta_arr, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const double beta = ctl->after;
  const int i = ctl->i;
  const bool brk = beta <= 1e-14;
  if (!brk) {
    const double inv = 1.0 / beta;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
      W[(size_t)r * ldw + i + 1] = mul(t[r], inv);
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    beta_arr[i] = beta;
    if (brk)
      ctl->halted = 1;
    else
      ctl->i = i + 1;
    *cnt = 0u;
  }
}

// Block sum, valid in thread 0 (deterministic tree).
__device__ double block_sum0(double v) {
  __shared__ double s_w[32];
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = add(r, s_w[w]);
  return r;
}

// last-CTA reduction of per-CTA sums in CTA order (valid in thread 0 of the last CTA)
__device__ bool grid_total(double mine, double* partial, unsigned* counter, double* total) {
  __shared__ bool s_last;
  const double bs = block_sum0(mine);
  if (threadIdx.x == 0) partial[blockIdx.x] = bs;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double q = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) q = add(q, __ldcg(partial + b));
  q = block_sum0(q);
  if (threadIdx.x == 0) {
    *total = q;
    *counter = 0u;
  }
  return true;
}

// NR (eigensolvers.hpp:408-409): t -= beta W[:, i-1] (beta != 0), alpha = t . W[:, i]
__global__ void __launch_bounds__(kRT) k_rw_nr_beta_alpha(int n, double* __restrict__ t,
                                                          const double* __restrict__ W, int ldw,
                                                          Ctl* ctl, double* alpha_arr,
                                                          const double* beta_arr, double* partial,
                                                          unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const int i = ctl->i;
  const double beta = i > 0 ? beta_arr[i - 1] : 0.0;
  const int ip = i > 0 ? i - 1 : 0;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double* row = W + (size_t)r * ldw;
    double tr = t[r];
    if (beta != 0.0) {
      tr = add(tr, mul(-beta, row[ip]));
      t[r] = tr;
    }
    s = add(s, mul(tr, row[i]));
  }
  double tot;
  if (grid_total(s, partial, cnt, &tot) && threadIdx.x == 0) {
    ctl->alpha = tot;
    alpha_arr[i] = tot;
  }
}

// NR (eigensolvers.hpp:410): t -= alpha W[:, i]; before = ||t|| for CGS2 (orth.hpp:72)
__global__ void __launch_bounds__(kRT) k_rw_nr_sub_alpha(int n, double* __restrict__ t,
                                                         const double* __restrict__ W, int ldw,
                                                         Ctl* ctl, double* partial, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const double alpha = ctl->alpha;
  const int i = ctl->i;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double tr = add(t[r], mul(-alpha, W[(size_t)r * ldw + i]));
    t[r] = tr;
    s = add(s, mul(tr, tr));
  }
  double tot;
  if (grid_total(s, partial, cnt, &tot) && threadIdx.x == 0) {
    ctl->before = sqrt(tot);
    ctl->after = ctl->before;
    ctl->repass = 0;
    ctl->npass = 0;
  }
}

// W[:, col0 + q] = src_q for q < cnt, src_q = U + idx[q] * ldu (column-major sources), through
// a 32 x 32 shared tile so both sides are coalesced
__global__ void k_rw_put_cols(int n, double* __restrict__ W, int ldw, int col0, int cnt,
                              const double* __restrict__ U, long ldu, const int* __restrict__ idx) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.x * 32, q0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int q = q0 + k, r = r0 + tx;
    if (q < cnt && r < n) tile[k][tx] = U[(size_t)(idx ? idx[q] : q) * ldu + r];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, q = q0 + tx;
    if (q < cnt && r < n) W[(size_t)r * ldw + col0 + q] = tile[tx][k];
  }
}

// dst (column-major, ld n) = W[:, col0 .. col0+cnt)
__global__ void k_rw_get_cols(int n, const double* __restrict__ W, int ldw, int col0, int cnt,
                              double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.x * 32, q0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, q = q0 + tx;
    if (q < cnt && r < n) tile[k][tx] = W[(size_t)r * ldw + col0 + q];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int q = q0 + k, r = r0 + tx;
    if (q < cnt && r < n) dst[(size_t)q * n + r] = tile[tx][k];
  }
}

__global__ void k_rw_col_move(int n, double* __restrict__ W, int ldw, int from, int to) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    W[(size_t)r * ldw + to] = W[(size_t)r * ldw + from];
}

template <class K, class... Args>
void launch_pdl(const Ctx& c, K kern, dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SE_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

int grid_small(const Ctx& c, int n) { return std::max(1, std::min(c.num_sms * 4, (n + kRT - 1) / kRT)); }

// Geometry per basis capacity (ldw): rows per block R and column pairs per thread QP, so a
// thread keeps ~16 pairs (R x QP) in flight whatever the width.
struct Geometry {
  int R = 1, QP = 1;
};
// Geometry classes by the active column count (padded to even): class g serves ncols <=
// kClassLim[g] with R rows per block and QP column pairs per thread, so a thread keeps ~8-16
// pairs in flight whatever the width.  The Lanczos step graph is captured once per class.
constexpr int kNumClasses = 13;
// classes 0-3: warp-per-row kernel (Q pairs per lane, RW rows per warp iteration); 4-: CTA rows
constexpr int kClassLim[kNumClasses] = {64, 128, 256, 512, 832, 1024, 1664, 2048, 3072, 3328, 4096, 6144, 8192};
constexpr int kClassR[kNumClasses] = {8, 8, 4, 1, 8, 4, 4, 2, 2, 2, 1, 1, 1};
constexpr int kClassQP[kNumClasses] = {1, 2, 4, 8, 2, 2, 4, 4, 6, 8, 8, 12, 16};
constexpr int kNumWarpClasses = 4;

Geometry geometry_of_class(int g) { return {kClassR[g], kClassQP[g]}; }

template <int PH, int QP, int R>
void stream_one(Ctx& c, const RowScratch& s, int n, const double* W, int ldw, double* t,
                const Ctl* ctl, const double* coef) {
  launch_pdl(c, k_rw_stream<PH, QP, R>, dim3(s.grid), dim3(kRT), 0, n, W, ldw, t, ctl, coef,
             s.part, s.npart, 0);
  ++c.launches;
}

template <int PH, int Q, int RW>
void warp_one(Ctx& c, const RowScratch& s, int n, const double* W, int ldw, double* t,
              const Ctl* ctl, const double* coef) {
  launch_pdl(c, k_rw_warp<PH, Q, RW>, dim3(s.grid), dim3(kRT), 0, n, W, ldw, t, ctl, coef, s.part,
             s.npart, 0);
  ++c.launches;
}

template <int PH>
void stream_launch(Ctx& c, const RowScratch& s, int n, const double* W, int ldw, double* t,
                   const Ctl* ctl, const double* coef, int cls) {
  switch (cls) {
    case 0: return warp_one<PH, 1, 8>(c, s, n, W, ldw, t, ctl, coef);
    case 1: return warp_one<PH, 2, 8>(c, s, n, W, ldw, t, ctl, coef);
    case 2: return warp_one<PH, 4, 4>(c, s, n, W, ldw, t, ctl, coef);
    case 3: return warp_one<PH, 8, 1>(c, s, n, W, ldw, t, ctl, coef);
    default: break;
  }
  const Geometry g = geometry_of_class(cls);
  switch (g.QP * 100 + g.R) {
    case 208: return stream_one<PH, 2, 8>(c, s, n, W, ldw, t, ctl, coef);
    case 204: return stream_one<PH, 2, 4>(c, s, n, W, ldw, t, ctl, coef);
    case 404: return stream_one<PH, 4, 4>(c, s, n, W, ldw, t, ctl, coef);
    case 402: return stream_one<PH, 4, 2>(c, s, n, W, ldw, t, ctl, coef);
    case 602: return stream_one<PH, 6, 2>(c, s, n, W, ldw, t, ctl, coef);
    case 802: return stream_one<PH, 8, 2>(c, s, n, W, ldw, t, ctl, coef);
    case 801: return stream_one<PH, 8, 1>(c, s, n, W, ldw, t, ctl, coef);
    case 1201: return stream_one<PH, 12, 1>(c, s, n, W, ldw, t, ctl, coef);
    default: return stream_one<PH, 16, 1>(c, s, n, W, ldw, t, ctl, coef);
  }
}

template <int PH>
void finish_launch(Ctx& c, const RowScratch& s, int ldw, Ctl* ctl, double* coef, double* hdiag,
                   int want_before) {
  const dim3 grid(PH == kN ? 1 : (ldw + kFinCols - 1) / kFinCols);
  launch_pdl(c, k_rw_finish<PH>, grid, dim3(kRT), 0, s.grid, ldw, (const double*)s.part,
             (const double*)s.npart, ctl, coef, hdiag, want_before);
  ++c.launches;
}

}  // namespace

int rw_ldw(int cols) { return std::max(2, (cols + 1) & ~1); }

RowScratch rw_scratch(const Ctx& c, int ldw) {
  RowScratch s;
  if (ldw > kClassLim[kNumClasses - 1])
    fail(SE_EINVAL, "row-major Krylov basis: capacity beyond 8192 columns");
  s.grid = c.num_sms * kRwPerSm;
  s.ldw = ldw;
  return s;
}
size_t rw_scratch_doubles(const RowScratch& s) { return (size_t)s.grid * s.ldw + s.grid; }
void rw_bind(RowScratch& s, double* buf) {
  s.part = buf;
  s.npart = buf + (size_t)s.grid * s.ldw;
}

int rw_class(int ncols) {
  const int pad = (ncols + 1) & ~1;
  for (int g = 0; g < kNumClasses; ++g)
    if (pad <= kClassLim[g]) return g;
  fail(SE_EINVAL, "row-major Krylov basis: more than 8192 columns");
}

void rw_cgs2(Ctx& c, const RowScratch& s, int n, double* t, const double* W, int ldw, Ctl* ctl,
             double* hdiag, double* coef1, double* coef2, bool want_before, int cls) {
  if (cls < 0) cls = rw_class(ldw);
  stream_launch<kT>(c, s, n, W, ldw, t, ctl, nullptr, cls);
  finish_launch<kT>(c, s, ldw, ctl, coef1, hdiag, want_before ? 1 : 0);
  stream_launch<kMid>(c, s, n, W, ldw, t, ctl, coef1, cls);
  finish_launch<kMid>(c, s, ldw, ctl, coef2, hdiag, 0);
  stream_launch<kN>(c, s, n, W, ldw, t, ctl, coef2, cls);
  finish_launch<kN>(c, s, ldw, ctl, nullptr, nullptr, 0);
}

void rw_col_get(Ctx& c, int n, const double* W, int ldw, const Ctl* ctl, int off, double* dst) {
  launch_pdl(c, k_rw_col_get, dim3(grid_small(c, n)), dim3(kRT), 0, n, W, ldw, ctl, off, dst);
  ++c.launches;
}

void rw_normalize(Ctx& c, unsigned* cnt, int n, const double* t, double* W, int ldw, Ctl* ctl,
                  double* beta_arr) {
  launch_pdl(c, k_rw_normalize, dim3(grid_small(c, n)), dim3(kRT), 0, n, t, W, ldw, ctl, beta_arr,
             cnt);
  ++c.launches;
}

void rw_nr_beta_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, int ldw,
                      Ctl* ctl, double* alpha_arr, const double* beta_arr) {
  launch_pdl(c, k_rw_nr_beta_alpha, dim3(grid_small(c, n)), dim3(kRT), 0, n, t, W, ldw, ctl,
             alpha_arr, beta_arr, s.buf, s.cnt);
  ++c.launches;
}

void rw_nr_sub_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, int ldw, Ctl* ctl) {
  launch_pdl(c, k_rw_nr_sub_alpha, dim3(grid_small(c, n)), dim3(kRT), 0, n, t, W, ldw, ctl, s.buf,
             s.cnt);
  ++c.launches;
}

void rw_put_cols(Ctx& c, int n, double* W, int ldw, int col0, int cnt, const double* U, long ldu,
                 const int* idx_dev) {
  if (cnt <= 0) return;
  k_rw_put_cols<<<dim3((n + 31) / 32, (cnt + 31) / 32), 256, 0, c.stream>>>(n, W, ldw, col0, cnt,
                                                                            U, ldu, idx_dev);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}

void rw_get_cols(Ctx& c, int n, const double* W, int ldw, int col0, int cnt, double* dst) {
  if (cnt <= 0) return;
  k_rw_get_cols<<<dim3((n + 31) / 32, (cnt + 31) / 32), 256, 0, c.stream>>>(n, W, ldw, col0, cnt, dst);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}

void rw_col_move(Ctx& c, int n, double* W, int ldw, int from, int to) {
  if (from == to) return;
  k_rw_col_move<<<grid_small(c, n), kRT, 0, c.stream>>>(n, W, ldw, from, to);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}

}  // namespace k
}  // namespace se
