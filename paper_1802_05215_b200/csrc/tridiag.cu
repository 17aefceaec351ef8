// Projected-problem eigenvalues for the stagnation checks of run_nr / run_tr
// (eigensolvers.hpp:436-444, 562-572: tnew = sum of Ritz values >= bar every ncycle steps).
// The reference runs a host QL sweep per check (O(m^2) each, O(m^3/ncycle) per cycle); here the
// symmetric tridiagonal form (NR's T, or TR's arrowhead reduced by Givens rotations, host O(l^2)
// once per cycle) is bisected on the device with Sturm counts, one thread per wanted eigenvalue.
#include <cfloat>

#include <chrono>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

__device__ __forceinline__ int sturm_count(int m, const double* __restrict__ d,
                                           const double* __restrict__ e, double x, double piv) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < piv) q = -piv;
  cnt += q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = (d[i] - x) - (e[i - 1] * e[i - 1]) / q;
    if (fabs(q) < piv) q = -piv;
    cnt += q < 0.0;
  }
  return cnt;
}

// One warp per wanted eigenvalue (ascending index idx = nbelow + warp): 32-point multisection,
// each lane evaluating one Sturm count, so the bracket shrinks 33x per round (~10 rounds to
// machine precision instead of ~55 bisection steps).
__global__ void k_tridiag_above(int m, const double* __restrict__ d, const double* __restrict__ e,
                                double bar, double* __restrict__ vals, int* __restrict__ count) {
  __shared__ double s_lo, s_hi, s_piv;
  __shared__ int s_below;
  if (threadIdx.x == 0) {
    double lo = DBL_MAX, hi = -DBL_MAX, emax = 0.0;
    for (int i = 0; i < m; ++i) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
      if (i + 1 < m) emax = fmax(emax, e[i] * e[i]);
    }
    s_piv = DBL_MIN * fmax(1.0, emax);
    const double pad = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + s_piv;
    s_lo = lo - pad;
    s_hi = hi + pad;
    s_below = sturm_count(m, d, e, bar, s_piv);
    if (blockIdx.x == 0) *count = m - s_below;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int idx = s_below + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (idx >= m) return;
  const double piv = s_piv;
  double a = fmax(bar, s_lo), b = s_hi;
  if (a > b) a = b;
  for (int round = 0; round < 40; ++round) {
    if ((b - a) <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b)) + piv) break;
    const double x = a + (b - a) * (double)(lane + 1) / 33.0;
    const int c = sturm_count(m, d, e, x, piv);
    // points with count <= idx lie left of the wanted eigenvalue
    const unsigned left = __ballot_sync(0xffffffffu, c <= idx);
    const int nl = __popc(left);  // points 0..nl-1 are left (counts are monotone in x)
    const double na = nl > 0 ? __shfl_sync(0xffffffffu, x, nl - 1) : a;
    const double nb = nl < 32 ? __shfl_sync(0xffffffffu, x, nl < 32 ? nl : 31) : b;
    if (!(na >= a && nb <= b) || na == a && nb == b) break;
    a = na;
    b = nb;
  }
  if (lane == 0) vals[idx - s_below] = 0.5 * (a + b);
}

}  // namespace

// Eigenvalues >= bar of the symmetric tridiagonal (d[m], e[m-1]) on the device.
// work: device scratch of >= 4*m + 8 doubles.  Returns them ascending in `out`.
void tridiag_eigs_above(Ctx& c, int m, const double* d_host, const double* e_host, double bar,
                        double* work, std::vector<double>& out) {
  out.clear();
  if (m <= 0) return;
  double* d = work;
  double* e = work + m;
  double* vals = work + 3 * m;
  int* cnt = reinterpret_cast<int*>(work + 4 * m);
  const auto t0 = std::chrono::steady_clock::now();
  h2d(c, d, d_host, sizeof(double) * m);
  if (m > 1)
    h2d(c, e, e_host, sizeof(double) * (m - 1));
  const auto t1 = std::chrono::steady_clock::now();
  const int tb = 128;  // 4 eigenvalues (warps) per CTA
  SE_CUDA(cudaEventRecord(c.evk0, c.stream));
  k_tridiag_above<<<(m + 3) / 4, tb, 0, c.stream>>>(m, d, e, bar, vals, cnt);
  SE_CUDA(cudaEventRecord(c.evk1, c.stream));
  ++c.launches;
  SE_CUDA(cudaGetLastError());
  int h = 0;
  d2h(c, &h, cnt, sizeof(int));
  ctx_sync(c);
  const auto t2 = std::chrono::steady_clock::now();
  float kms = 0.f;
  SE_CUDA(cudaEventElapsedTime(&kms, c.evk0, c.evk1));
  c.prof_kernel_ms += kms;
  out.resize(h);
  if (h)
    d2h(c, out.data(), vals, sizeof(double) * h);
  ctx_sync(c);
  const auto t3 = std::chrono::steady_clock::now();
  auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  c.prof_chk[0] += sec(t0, t1);
  c.prof_chk[1] += sec(t1, t2);
  c.prof_chk[2] += sec(t2, t3);
}

}  // namespace k
}  // namespace se
