// Projected-problem eigenvalues for the stagnation checks of run_nr / run_tr
// (eigensolvers.hpp:436-444, 562-572: tnew = sum of Ritz values >= bar every ncycle steps).
// The reference runs a host QL sweep per check (O(m^2) each, O(m^3/ncycle) per cycle); here the
// symmetric tridiagonal form (NR's T, or TR's arrowhead reduced by Givens rotations, host O(l^2)
// once per cycle) is bisected on the device with Sturm counts, one thread per wanted eigenvalue.
#include <cfloat>

#include <chrono>
#include <cmath>
#include <vector>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

// 1/q to full double precision without the division subroutine: the 23-bit hardware estimate
// refined by two Newton steps (the count below depends only on signs, and bisection on it is
// backward stable; results are deterministic).
__device__ __forceinline__ double recip(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

// Sturm count (number of eigenvalues < x) of the tridiagonal (d, e2 = e^2), pivot floor piv.
__device__ __forceinline__ int sturm_count(int m, const double* __restrict__ d,
                                           const double* __restrict__ e2, double x, double piv) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < piv) q = -piv;
  cnt += q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = (d[i] - x) - e2[i - 1] * recip(q);
    if (fabs(q) < piv) q = -piv;
    cnt += q < 0.0;
  }
  return cnt;
}

// One warp per wanted eigenvalue (ascending index idx = below + warp): 32-point multisection,
// each lane evaluating one Sturm count, so the bracket shrinks 33x per round (~10 rounds to
// machine precision instead of ~55 bisection steps).  The Gershgorin bracket, pivot floor and
// the count below `bar` are computed once on the host (O(m)) and passed in.
__global__ void k_tridiag_above(int m, const double* __restrict__ d, const double* __restrict__ e2,
                                double bar, double glo, double ghi, double piv, int below,
                                double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int idx = below + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (idx >= m) return;
  double a = fmax(bar, glo), b = ghi;
  if (a > b) a = b;
  for (int round = 0; round < 40; ++round) {
    if ((b - a) <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b)) + piv) break;
    const double x = a + (b - a) * (double)(lane + 1) / 33.0;
    const int c = sturm_count(m, d, e2, x, piv);
    // points with count <= idx lie left of the wanted eigenvalue
    const unsigned left = __ballot_sync(0xffffffffu, c <= idx);
    const int nl = __popc(left);  // points 0..nl-1 are left (counts are monotone in x)
    const double na = nl > 0 ? __shfl_sync(0xffffffffu, x, nl - 1) : a;
    const double nb = nl < 32 ? __shfl_sync(0xffffffffu, x, nl < 32 ? nl : 31) : b;
    if (!(na >= a && nb <= b) || (na == a && nb == b)) break;
    a = na;
    b = nb;
  }
  if (lane == 0) vals[idx - below] = 0.5 * (a + b);
}

}  // namespace

// Eigenvalues >= bar of the symmetric tridiagonal (d[m], e[m-1]) on the device.
// work: device scratch of >= 4*m + 8 doubles.  Returns them ascending in `out`.
void tridiag_eigs_above(Ctx& c, int m, const double* d_host, const double* e_host, double bar,
                        double* work, std::vector<double>& out) {
  out.clear();
  if (m <= 0) return;
  double* d = work;
  double* e2 = work + m;
  double* vals = work + 3 * m;
  const auto t0 = std::chrono::steady_clock::now();
  // host O(m): Gershgorin bracket, pivot floor, squared off-diagonal, count below bar (the same
  // recurrence the device runs, so the device's indices start exactly at the first value >= bar)
  std::vector<double> h2((size_t)std::max(m - 1, 1));
  double glo = DBL_MAX, ghi = -DBL_MAX, emax = 0.0;
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::fabs(e_host[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(e_host[i]) : 0.0);
    glo = std::fmin(glo, d_host[i] - r);
    ghi = std::fmax(ghi, d_host[i] + r);
    if (i + 1 < m) {
      h2[i] = e_host[i] * e_host[i];
      emax = std::fmax(emax, h2[i]);
    }
  }
  const double piv = DBL_MIN * std::fmax(1.0, emax);
  const double pad = 2.0 * DBL_EPSILON * std::fmax(std::fabs(glo), std::fabs(ghi)) + piv;
  glo -= pad;
  ghi += pad;
  int below = 0;
  {
    double q = d_host[0] - bar;
    if (std::fabs(q) < piv) q = -piv;
    below += q < 0.0;
    for (int i = 1; i < m; ++i) {
      q = (d_host[i] - bar) - h2[i - 1] / q;
      if (std::fabs(q) < piv) q = -piv;
      below += q < 0.0;
    }
  }
  const int h = m - below;
  out.resize(h);
  if (h == 0) return;
  h2d(c, d, d_host, sizeof(double) * m);
  if (m > 1) h2d(c, e2, h2.data(), sizeof(double) * (m - 1));
  const auto t1 = std::chrono::steady_clock::now();
  const int tb = 128;  // 4 eigenvalues (warps) per CTA
  SE_CUDA(cudaEventRecord(c.evk0, c.stream));
  k_tridiag_above<<<(h + 3) / 4, tb, 0, c.stream>>>(m, d, e2, bar, glo, ghi, piv, below, vals);
  SE_CUDA(cudaEventRecord(c.evk1, c.stream));
  ++c.launches;
  SE_CUDA(cudaGetLastError());
  d2h(c, out.data(), vals, sizeof(double) * h);
  ctx_sync(c);
  const auto t2 = std::chrono::steady_clock::now();
  float kms = 0.f;
  SE_CUDA(cudaEventElapsedTime(&kms, c.evk0, c.evk1));
  c.prof_kernel_ms += kms;
  const auto t3 = std::chrono::steady_clock::now();
  auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  c.prof_chk[0] += sec(t0, t1);
  c.prof_chk[1] += sec(t1, t2);
  c.prof_chk[2] += sec(t2, t3);
}

}  // namespace k
}  // namespace se
