// Krylov kernels for sm_100a: full reorthogonalisation (K4/K5 of SURVEY.md §2.1), the Lanczos
// recurrence scalars, normalisation, and candidate (Ritz pair) statistics (K6).
//
// All reductions are deterministic: fixed per-CTA partials combined in index order by the
// last CTA to finish (threadfence + counter), so a rerun on the same GPU is bitwise identical
// (the reference's determinism contract, SPEC.md:248 / test_dos.cpp:117-140).
// Every kernel reads the column count / halt flag from the device control block (Ctl) so a
// whole Lanczos step is replayable as one CUDA graph.
#include <cmath>

#include <cstdlib>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

constexpr double kDgksEta = 0.70710678118654752;  // orth.hpp:13
constexpr int kThreads = 256;
constexpr int kCW = 32;        // columns per GEMV-T work item
constexpr int kMaxRch = 4096;  // rows per GEMV-T work item (t chunk in shared memory)
constexpr int kNW = 256;  // columns per GEMV-N chunk

// Counter slot layout inside Ctx::counters.
constexpr int kSlotNorm = 0;
constexpr int kSlotMisc = 1;
constexpr int kSlotGroups = 64;  // + group index (GEMV-T per-column-group completion)

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v = add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block sum (deterministic): warp xor-trees then warp 0 over the warp sums in order.
__device__ double block_sum(double v) {
  __shared__ double s_w[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) s_w[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in warp 0
}

// Last-CTA pattern: every CTA publishes partial[blockIdx.x]; returns true (block-uniform) in the
// CTA that completes last, after which `total` (valid in thread 0) is the index-ordered sum.
__device__ bool grid_sum(double mine, double* partial, unsigned* counter, double* total) {
  __shared__ bool s_last;
  const double bs = block_sum(mine);
  if (threadIdx.x == 0) partial[blockIdx.x] = bs;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double q = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) q = add(q, __ldcg(partial + b));
  q = block_sum(q);
  if (threadIdx.x == 0) {
    *total = q;
    *counter = 0u;
  }
  return true;
}

int grid_for(const Ctx& c, int n) {
  return std::max(1, std::min(c.num_sms * 4, (n + kThreads - 1) / kThreads));
}

// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_norm_before(int n, const double* __restrict__ t,
                                                          Ctl* ctl, double* partial, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    s = add(s, mul(t[r], t[r]));
  double tot;
  if (grid_sum(s, partial, cnt, &tot) && threadIdx.x == 0) {
    ctl->before = sqrt(tot);
    ctl->after = ctl->before;
    ctl->repass = 0;
    ctl->npass = 0;
  }
}

// NR (eigensolvers.hpp:408-409): t -= beta W[:, i-1] (when beta != 0), alpha = t . W[:, i].
__global__ void __launch_bounds__(kThreads) k_nr_beta_alpha(int n, double* __restrict__ t,
                                                            const double* __restrict__ W, Ctl* ctl,
                                                            double* alpha_arr, const double* beta_arr,
                                                            double* partial, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const int i = ctl->i;
  const double beta = i > 0 ? beta_arr[i - 1] : 0.0;
  const double* __restrict__ w = W + (size_t)i * n;
  const double* __restrict__ wp = W + (size_t)(i > 0 ? i - 1 : 0) * n;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double tr = t[r];
    if (beta != 0.0) {
      tr = add(tr, mul(-beta, wp[r]));
      t[r] = tr;
    }
    s = add(s, mul(tr, w[r]));
  }
  double tot;
  if (grid_sum(s, partial, cnt, &tot) && threadIdx.x == 0) {
    ctl->alpha = tot;
    alpha_arr[i] = tot;
  }
}

// NR (eigensolvers.hpp:410): t -= alpha w ; then before = ||t|| for CGS2 (orth.hpp:72).
__global__ void __launch_bounds__(kThreads) k_nr_sub_alpha(int n, double* __restrict__ t,
                                                           const double* __restrict__ W, Ctl* ctl,
                                                           double* partial, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const double alpha = ctl->alpha;
  const double* __restrict__ w = W + (size_t)ctl->i * n;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double tr = add(t[r], mul(-alpha, w[r]));
    t[r] = tr;
    s = add(s, mul(tr, tr));
  }
  double tot;
  if (grid_sum(s, partial, cnt, &tot) && threadIdx.x == 0) {
    ctl->before = sqrt(tot);
    ctl->after = ctl->before;
    ctl->repass = 0;
    ctl->npass = 0;
  }
}

// ---- CGS pass, part 1: coef = Q^T t (cgs_pass orth.hpp:23-25) --------------------------------
// Work item = (row chunk of `rch` rows, group of kCW columns).  The t chunk is staged in shared
// memory; each warp owns kCW/8 columns and streams its column segment with 8 loads in flight
// per lane.  Per-(row chunk, column) partials are combined, in row-chunk order, by whichever CTA
// finishes a column group last.
__device__ __forceinline__ int pass_ncols(const Ctl* ctl, int mode, int fixed) {
  return fixed >= 0 ? fixed : (mode == 1 ? ctl->nlock : ctl->i + 1);
}

__device__ __forceinline__ bool pass_skip(const Ctl* ctl, int pass2) {
  return ctl->halted || (pass2 && !ctl->repass);
}

__global__ void __launch_bounds__(kThreads) k_gemvt(int n, int rch, const double* __restrict__ Q,
                                                    const double* __restrict__ t, Ctl* ctl, int mode,
                                                    int pass2, int fixed, double* partial, int ldp,
                                                    unsigned* grp_cnt, double* coef, double* hdiag) {
  // One work item per CTA (short-lived CTAs keep SM slots turning over, so the latency-bound
  // kernels of other slices sharing the GPU are scheduled promptly).  Items beyond the current
  // column count exit at once.  Programmatic dependent launch: the CTA is resident before the
  // previous kernel ends and waits here.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl && pass_skip(ctl, pass2)) return;
  const int ncols = pass_ncols(ctl, mode, fixed);
  const int nrb = (n + rch - 1) / rch;
  const int g = blockIdx.x / nrb, rb = blockIdx.x - g * nrb;
  if (ncols <= 0 || g * kCW >= ncols) return;
  const int hcol = (hdiag && ctl) ? ctl->i : -1;
  extern __shared__ double s_t[];  // rch doubles (dynamic: small items leave room for other CTAs)
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = rb * rch, rn = min(rch, n - r0);
  for (int q = threadIdx.x; q < rch; q += kThreads) s_t[q] = q < rn ? t[r0 + q] : 0.0;
  __syncthreads();
  for (int jj = warp; jj < kCW; jj += kThreads / 32) {
    const int j = g * kCW + jj;
    if (j >= ncols) break;
    const double* __restrict__ qc = Q + (size_t)j * n + r0;
    double acc = 0.0;
    int q = lane;
    for (; q + 7 * 32 < rn; q += 8 * 32) {
      double w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = __ldcs(qc + q + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = add(acc, mul(w[u], s_t[q + 32 * u]));
    }
    for (; q < rn; q += 32) acc = add(acc, mul(__ldcs(qc + q), s_t[q]));
    acc = warp_sum(acc);
    if (lane == 0) partial[(size_t)rb * ldp + j] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&grp_cnt[g], 1u) == (unsigned)(nrb - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // 8 threads per column, strided over row chunks, shuffle-combined in fixed order.
  const int jj = threadIdx.x >> 3, sub8 = threadIdx.x & 7;
  const int j = g * kCW + jj;
  double q = 0.0;
  if (j < ncols)
    for (int b = sub8; b < nrb; b += 8) q = add(q, __ldcg(partial + (size_t)b * ldp + j));
  for (int o = 4; o > 0; o >>= 1) q = add(q, __shfl_down_sync(0xffffffffu, q, o, 8));
  if (sub8 == 0 && j < ncols) {
    coef[j] = q;
    if (j == hcol) hdiag[j] = add(hdiag[j], q);  // h[j] += c_j (orth.hpp:30), H(i,i) += h[i]
  }
  if (threadIdx.x == 0) grp_cnt[g] = 0u;
}

// ---- CGS pass, part 2: t -= Q coef (orth.hpp:26-29) + ||t|| + DGKS decision (orth.hpp:76-78).
// CTA (row block of 256 rows, chunk of kNW columns): each thread sums its row over the chunk
// (column order, 16 loads in flight) into P[chunk][row]; the last chunk CTA of a row block
// subtracts the chunk partials in chunk order and adds the block's ||t||^2; the last row block
// finishes the norm and the re-pass decision.  mode 0: Krylov basis (norm + flags); 1: locked
// set; 2: plain (no norm).
__global__ void __launch_bounds__(kThreads) k_gemvn(int n, const double* __restrict__ Q,
                                                    double* __restrict__ t, Ctl* ctl, int mode,
                                                    int pass2, int fixed,
                                                    const double* __restrict__ coef,
                                                    double* __restrict__ P, unsigned* rb_cnt,
                                                    double* npart, unsigned* gcnt, int nw) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl && pass_skip(ctl, pass2)) return;
  const int ncols = pass_ncols(ctl, mode, fixed);
  const int nchunks = (ncols + nw - 1) / nw;
  const int rb = blockIdx.x, cc = blockIdx.y;
  if (ncols <= 0 || cc >= nchunks) return;
  __shared__ double s_c[kNW];
  __shared__ bool s_last;
  const int j0 = cc * nw, jn = min(nw, ncols - j0);
  for (int q = threadIdx.x; q < jn; q += kThreads) s_c[q] = coef[j0 + q];
  __syncthreads();
  const int r = rb * kThreads + threadIdx.x;
  const bool live = r < n;
  if (live) {
    const double* __restrict__ qr = Q + (size_t)j0 * n + r;
    double p = 0.0;
    int j = 0;
    for (; j + 16 <= jn; j += 16) {
      double w[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) w[u] = __ldcs(qr + (size_t)(j + u) * n);
#pragma unroll
      for (int u = 0; u < 16; ++u) p = add(p, mul(s_c[j + u], w[u]));
    }
    for (; j < jn; ++j) p = add(p, mul(s_c[j], __ldcs(qr + (size_t)j * n)));
    P[(size_t)cc * n + r] = p;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&rb_cnt[rb], 1u) == (unsigned)(nchunks - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double tr = 0.0;
  if (live) {
    tr = t[r];
    for (int q = 0; q < nchunks; ++q) tr = sub(tr, __ldcg(P + (size_t)q * n + r));
    t[r] = tr;
  }
  if (threadIdx.x == 0) rb_cnt[rb] = 0u;
  if (mode != 0) return;
  // this row block's ||t||^2, then the last row block reduces all of them in order
  __shared__ bool s_glast;
  const double bs = block_sum(tr * tr);
  if (threadIdx.x == 0) npart[rb] = bs;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_glast = atomicAdd(gcnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_glast) return;
  __threadfence();
  double q = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads) q = add(q, __ldcg(npart + b));
  q = block_sum(q);
  if (threadIdx.x == 0) {
    const double after = sqrt(q);
    ctl->npass += 1;
    ctl->passes_total += 1;
    ctl->cols_total += ncols;
    if (!pass2) ctl->repass = after > kDgksEta * ctl->before ? 0 : 1;
    ctl->before = after;
    ctl->after = after;
    *gcnt = 0u;
  }
}

// beta = ||t|| (the last `after`); breakdown (beta <= 1e-14, orth.hpp:14) halts the recurrence;
// otherwise W[:, i+1] = t * (1/beta) (eigensolvers.hpp:431), beta_arr[i] = beta, i += 1.
__global__ void __launch_bounds__(kThreads) k_normalize(int n, const double* __restrict__ t,
                                                        double* __restrict__ W, Ctl* ctl,
                                                        double* beta_arr, unsigned* cnt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  const double beta = ctl->after;
  const int i = ctl->i;
  const bool brk = beta <= 1e-14;
  if (!brk) {
    const double inv = 1.0 / beta;
    double* __restrict__ wn = W + (size_t)(i + 1) * n;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
      wn[r] = mul(t[r], inv);
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    beta_arr[i] = beta;
    if (brk) {
      ctl->halted = 1;
    } else {
      ctl->i = i + 1;
    }
    *cnt = 0u;
  }
}

// Candidate statistics, one CTA per column (eigensolvers.hpp:289-316):
//   uu = u.u, lambda = u.Au / uu, r = Au - lambda u, res = (1/sqrt(uu)) ||r||, u *= 1/sqrt(uu).
__global__ void __launch_bounds__(kThreads) k_candidate_stats(int n, double* __restrict__ U,
                                                              const double* __restrict__ AU,
                                                              const double* __restrict__ w,
                                                              double* out3) {
  const size_t off = (size_t)blockIdx.x * n;
  double* __restrict__ u = U + off;
  const double* __restrict__ au = AU + off;
  double suu = 0.0, sua = 0.0;
  for (int r = threadIdx.x; r < n; r += kThreads) {
    suu = add(suu, mul(u[r], u[r]));
    sua = add(sua, mul(u[r], au[r]));
  }
  __shared__ double s_uu, s_lam;
  double tuu = block_sum(suu);
  if (threadIdx.x == 0) s_uu = tuu;
  __syncthreads();
  double tua = block_sum(sua);
  if (threadIdx.x == 0) s_lam = s_uu > 0.0 ? tua / s_uu : 0.0;
  __syncthreads();
  const double uu = s_uu, lam = s_lam;
  double srr = 0.0;
  if (uu > 0.0)
    for (int r = threadIdx.x; r < n; r += kThreads) {
      double rr = add(au[r], mul(-lam, u[r]));
      if (w) rr = mul(w[r], rr);
      srr = add(srr, mul(rr, rr));
    }
  const double trr = block_sum(srr);
  if (threadIdx.x == 0) {
    const double s = uu > 0.0 ? 1.0 / sqrt(uu) : 0.0;
    out3[3 * blockIdx.x + 0] = lam;
    out3[3 * blockIdx.x + 1] = mul(s, sqrt(trr));
    out3[3 * blockIdx.x + 2] = uu;
  }
}

// One Chebyshev degree of the filter on a precomputed operator product sx = S x (pencils, where
// S = P A P is a composition and cannot be fused into the SpMV): the same update as the fused
// kernel (filter_poly.hpp:261-276): t = (sx - c x) / d; first: y = t, out = mu0 x + mu1 t;
// next: y = 2 t - prev, out += mu_j y.
__global__ void k_cheb_combine(int n, int first, const double* __restrict__ sx,
                               const double* __restrict__ x, const double* __restrict__ prev,
                               double* __restrict__ y, double* __restrict__ out, double c,
                               double invd, double mu0, double muj, const Ctl* halt) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (halt && halt->halted) return;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const double xr = x[r];
    const double t = mul(sub(sx[r], mul(c, xr)), invd);
    if (first) {
      y[r] = t;
      out[r] = add(add(0.0, mul(mu0, xr)), mul(muj, t));
    } else {
      const double tj = sub(mul(2.0, t), prev[r]);
      y[r] = tj;
      out[r] = add(out[r], mul(muj, tj));
    }
  }
}

// Pencil candidate statistics, one CTA per column (eigensolvers.hpp:289-316 with b != nullptr):
// x = P u, ax = A x, bx = B x:  lambda = x.ax / x.bx, res = ||ax - lambda bx|| / sqrt(x.bx),
// out3 = (lambda, res, u.u).
__global__ void __launch_bounds__(kThreads) k_pencil_stats(int n, const double* __restrict__ U,
                                                           const double* __restrict__ X,
                                                           const double* __restrict__ AX,
                                                           const double* __restrict__ BX,
                                                           double* out3) {
  const size_t off = (size_t)blockIdx.x * n;
  const double *u = U + off, *x = X + off, *ax = AX + off, *bx = BX + off;
  double suu = 0.0, sxa = 0.0, sxb = 0.0;
  for (int r = threadIdx.x; r < n; r += kThreads) {
    suu = add(suu, mul(u[r], u[r]));
    sxa = add(sxa, mul(x[r], ax[r]));
    sxb = add(sxb, mul(x[r], bx[r]));
  }
  __shared__ double s_uu, s_xb, s_lam;
  double v = block_sum(suu);
  if (threadIdx.x == 0) s_uu = v;
  __syncthreads();
  v = block_sum(sxb);
  if (threadIdx.x == 0) s_xb = v;
  __syncthreads();
  v = block_sum(sxa);
  if (threadIdx.x == 0) s_lam = s_xb > 0.0 ? v / s_xb : 0.0;
  __syncthreads();
  const double lam = s_lam;
  double srr = 0.0;
  for (int r = threadIdx.x; r < n; r += kThreads) {
    const double q = add(ax[r], mul(-lam, bx[r]));
    srr = add(srr, mul(q, q));
  }
  v = block_sum(srr);
  if (threadIdx.x == 0) {
    out3[3 * blockIdx.x + 0] = lam;
    out3[3 * blockIdx.x + 1] = s_xb > 0.0 ? sqrt(v) / sqrt(s_xb) : 0.0;
    out3[3 * blockIdx.x + 2] = s_uu;
  }
}

// x_j *= 1 / sqrt(x_j . bx_j) per column (B-normalisation of returned pencil eigenvectors)
__global__ void __launch_bounds__(kThreads) k_b_normalize(int n, double* __restrict__ X,
                                                          const double* __restrict__ BX) {
  const size_t off = (size_t)blockIdx.x * n;
  double s = 0.0;
  for (int r = threadIdx.x; r < n; r += kThreads) s = add(s, mul(X[off + r], BX[off + r]));
  __shared__ double s_scale;
  const double v = block_sum(s);
  if (threadIdx.x == 0) s_scale = v > 0.0 ? 1.0 / sqrt(v) : 0.0;
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += kThreads) X[off + r] = mul(s_scale, X[off + r]);
}

__global__ void k_dot(int n, const double* __restrict__ x, const double* __restrict__ y,
                      double* result, double* partial, unsigned* cnt) {
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    s = add(s, mul(x[r], y[r]));
  double tot;
  if (grid_sum(s, partial, cnt, &tot) && threadIdx.x == 0) *result = tot;
}

__global__ void k_scale(int n, double a, double* __restrict__ x) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    x[r] = mul(a, x[r]);
}

__global__ void k_scale_copy(int n, double a, const double* __restrict__ src, double* __restrict__ dst) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    dst[r] = mul(a, src[r]);
}

__global__ void k_stamp(Ctl* ctl, int which) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (ctl->halted) return;
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  if (which == 0) {
    ctl->ts0 = now;
  } else if (which == 1) {
    ctl->t_mv_ns += (double)(now - ctl->ts0);
    ctl->ts1 = now;
  } else {
    ctl->t_orth_ns += (double)(now - ctl->ts1);
  }
}

int rch_for(int n) { return n >= (1 << 20) ? 4096 : (n >= (1 << 16) ? 2048 : 512); }

// programmatic-dependent launch of a step kernel (the kernel starts with griddepcontrol.wait)
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

// launch attributes of the GEMV kernels: programmatic dependent launch
cudaLaunchConfig_t gemv_cfg(const Ctx& c, dim3 grid, size_t smem, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// columns per GEMV-N chunk
int nw_for() { return kNW; }

}  // namespace

// Scratch layout of a CGS pass: [GEMV-T partials nrb x cap][GEMV-N chunk partials nchunks x n]
// [row-block norms]; counters: [group counters][row-block counters].
size_t cgs_scratch_doubles(const Ctx& c, int n, int cap_cols) {
  const int rch = rch_for(n);
  const size_t nrb = (size_t)(n + rch - 1) / rch;
  const size_t gn = (size_t)(n + kThreads - 1) / kThreads;
  const size_t ncc = (size_t)(std::max(cap_cols, 1) + nw_for() - 1) / nw_for();
  return nrb * (size_t)std::max(cap_cols, 1) + ncc * (size_t)n + gn + (size_t)c.num_sms * 8 + 64;
}

int cgs_counter_slots(int n, int cap_cols) {
  return kSlotGroups + (std::max(cap_cols, 1) + kCW - 1) / kCW + (n + kThreads - 1) / kThreads + 8;
}

static void need(const Scratch& s, size_t doubles, int slots) {
  if (doubles > s.cap || slots > s.ncnt) fail(SE_EINVAL, "internal: scratch too small");
}

void norm_before(Ctx& c, const Scratch& s, int n, const double* t, Ctl* ctl) {
  const int g = grid_for(c, n);
  need(s, g, kSlotMisc + 1);
  launch_pdl(c, k_norm_before, dim3(g), dim3(kThreads), 0, n, (const double*)t, ctl, s.buf, s.cnt + kSlotNorm);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void nr_beta_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, Ctl* ctl,
                   double* alpha_arr, const double* beta_arr) {
  const int g = grid_for(c, n);
  need(s, g, kSlotMisc + 1);
  launch_pdl(c, k_nr_beta_alpha, dim3(g), dim3(kThreads), 0, n, t, W, ctl, alpha_arr, beta_arr, s.buf,
             s.cnt + kSlotNorm);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void nr_sub_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, Ctl* ctl) {
  const int g = grid_for(c, n);
  need(s, g, kSlotMisc + 1);
  launch_pdl(c, k_nr_sub_alpha, dim3(g), dim3(kThreads), 0, n, t, W, ctl, s.buf, s.cnt + kSlotNorm);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

// Scratch layout for a CGS pass: [GEMV-T partials nrb x ldp][GEMV-N norm partials].
static void cgs_impl(Ctx& c, const Scratch& s, int n, double* t, const double* Q, int mode,
                     bool pass2, Ctl* ctl, int fixed, int ldp, double* hdiag, double* coef) {
  if (n == 0) return;
  const int rch = rch_for(n);
  const int nrb = (n + rch - 1) / rch;
  const int ngrp_max = (ldp + kCW - 1) / kCW;
  const int gn = (n + kThreads - 1) / kThreads;
  need(s, cgs_scratch_doubles(c, n, ldp), cgs_counter_slots(n, ldp));
  const int ncc = (ldp + nw_for() - 1) / nw_for();
  double* part = s.buf;
  double* P = part + (size_t)nrb * ldp;
  double* npart = P + (size_t)ncc * n;
  { cudaLaunchAttribute at[1]; const cudaLaunchConfig_t cf = gemv_cfg(c, dim3(nrb * ngrp_max), rch * sizeof(double), at);
  SE_CUDA(cudaLaunchKernelEx(&cf, k_gemvt, n, rch, Q, t, ctl, mode, pass2 ? 1 : 0, fixed,
                                                     part, ldp, s.cnt + kSlotGroups, coef, hdiag)); }
  ++c.launches;
  { cudaLaunchAttribute at[1]; const cudaLaunchConfig_t cf = gemv_cfg(c, dim3(gn, ncc), 0, at);
  SE_CUDA(cudaLaunchKernelEx(&cf, k_gemvn, n, Q, t, ctl, mode, pass2 ? 1 : 0, fixed, coef, P,
                                                    s.cnt + kSlotGroups + ngrp_max, npart,
                                                    s.cnt + kSlotMisc, nw_for())); }
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void gemvt_only(Ctx& c, const Scratch& s, int n, const double* t, const double* Q, bool pass2,
                Ctl* ctl, double* hdiag, double* coef, int cap) {
  if (n == 0) return;
  const int ldp = std::max(cap, 1);
  const int rch = rch_for(n);
  const int nrb = (n + rch - 1) / rch;
  const int ngrp_max = (ldp + kCW - 1) / kCW;
  need(s, cgs_scratch_doubles(c, n, ldp), cgs_counter_slots(n, ldp));
  { cudaLaunchAttribute at[1]; const cudaLaunchConfig_t cf = gemv_cfg(c, dim3(nrb * ngrp_max), rch * sizeof(double), at);
  SE_CUDA(cudaLaunchKernelEx(&cf, k_gemvt, n, rch, Q, t, ctl, 0, pass2 ? 1 : 0, -1, s.buf,
                                                     ldp, s.cnt + kSlotGroups, coef, hdiag)); }
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void gemvn_only(Ctx& c, const Scratch& s, int n, double* t, const double* Q, bool pass2, Ctl* ctl,
                const double* coef, int cap) {
  if (n == 0) return;
  const int ldp = std::max(cap, 1);
  const int rch = rch_for(n);
  const int nrb = (n + rch - 1) / rch;
  const int ngrp_max = (ldp + kCW - 1) / kCW;
  const int gn = (n + kThreads - 1) / kThreads;
  const int ncc = (ldp + nw_for() - 1) / nw_for();
  need(s, cgs_scratch_doubles(c, n, ldp), cgs_counter_slots(n, ldp));
  double* P = s.buf + (size_t)nrb * ldp;
  double* npart = P + (size_t)ncc * n;
  { cudaLaunchAttribute at[1]; const cudaLaunchConfig_t cf = gemv_cfg(c, dim3(gn, ncc), 0, at);
  SE_CUDA(cudaLaunchKernelEx(&cf, k_gemvn, n, Q, t, ctl, 0, pass2 ? 1 : 0, -1, coef, P,
                                                    s.cnt + kSlotGroups + ngrp_max, npart,
                                                    s.cnt + kSlotMisc, nw_for())); }
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void cgs_pass(Ctx& c, const Scratch& s, int n, double* t, const double* Q, bool use_lock,
              bool pass2, Ctl* ctl, double* hdiag, double* coef, int cap) {
  cgs_impl(c, s, n, t, Q, use_lock ? 1 : 0, pass2, ctl, -1, std::max(cap, 1), hdiag, coef);
}

void project_out(Ctx& c, const Scratch& s, int n, int kq, const double* Q, double* t,
                 double* coef) {
  if (kq <= 0) return;
  cgs_impl(c, s, n, t, Q, 2, false, nullptr, kq, kq, nullptr, coef);
}

void normalize_next(Ctx& c, const Scratch& s, int n, const double* t, double* W, Ctl* ctl,
                    double* beta_arr) {
  const int g = grid_for(c, n);
  need(s, 0, kSlotMisc + 1);
  launch_pdl(c, k_normalize, dim3(g), dim3(kThreads), 0, n, t, W, ctl, beta_arr, s.cnt + kSlotNorm);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void cheb_combine(Ctx& c, int n, bool first, const double* sx, const double* x, const double* prev,
                  double* y, double* out, double cc, double invd, double mu0, double muj,
                  const Ctl* halt) {
  launch_pdl(c, k_cheb_combine, dim3(grid_for(c, n)), dim3(kThreads), 0, n, first ? 1 : 0, sx, x,
             prev, y, out, cc, invd, mu0, muj, halt);
  ++c.launches;
}

void pencil_stats(Ctx& c, int n, int nc, const double* U, const double* X, const double* AX,
                  const double* BX, double* out3) {
  if (nc <= 0) return;
  k_pencil_stats<<<nc, kThreads, 0, c.stream>>>(n, U, X, AX, BX, out3);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void b_normalize(Ctx& c, int n, int nc, double* X, const double* BX) {
  if (nc <= 0) return;
  k_b_normalize<<<nc, kThreads, 0, c.stream>>>(n, X, BX);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void candidate_stats(Ctx& c, int n, int nc, double* U, const double* AU, double* out3,
                     const double* w) {
  if (nc <= 0 || n == 0) return;
  k_candidate_stats<<<nc, kThreads, 0, c.stream>>>(n, U, AU, w, out3);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void dot_dev(Ctx& c, const Scratch& s, int n, const double* x, const double* y, double* result_dev) {
  const int g = grid_for(c, n);
  need(s, g, kSlotMisc + 1);
  k_dot<<<g, kThreads, 0, c.stream>>>(n, x, y, result_dev, s.buf, s.cnt + kSlotNorm);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void scale_copy(Ctx& c, int n, double a, const double* src, double* dst) {
  if (n == 0) return;
  k_scale_copy<<<grid_for(c, n), kThreads, 0, c.stream>>>(n, a, src, dst);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void stamp(Ctx& c, Ctl* ctl, int which) {
  launch_pdl(c, k_stamp, dim3(1), dim3(1), 0, ctl, which);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

void scale(Ctx& c, int n, double a, double* x) {
  if (n == 0) return;
  k_scale<<<grid_for(c, n), kThreads, 0, c.stream>>>(n, a, x);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
}

}  // namespace k
}  // namespace se
