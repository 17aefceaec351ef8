// Projected-problem eigenvalues for the stagnation checks of run_nr / run_tr
// (eigensolvers.hpp:436-444, 562-572: tnew = sum of Ritz values >= bar every ncycle steps).
// The reference runs a host QL sweep per check (O(m^2) each, O(m^3/ncycle) per cycle); here the
// symmetric tridiagonal form (NR's T, or TR's arrowhead reduced by Givens rotations, host O(l^2)
// once per cycle) is bisected on the device with Sturm counts, one thread per wanted eigenvalue.
#include <cfloat>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

__global__ void k_tridiag_above(int m, const double* __restrict__ d, const double* __restrict__ e,
                                double bar, double* __restrict__ vals,
                                int* __restrict__ count) {
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
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // count of eigenvalues < bar, with e^2 formed on the fly
    int cnt = 0;
    double q = d[0] - bar;
    if (fabs(q) < s_piv) q = -s_piv;
    cnt += q < 0.0;
    for (int i = 1; i < m; ++i) {
      q = (d[i] - bar) - (e[i - 1] * e[i - 1]) / q;
      if (fabs(q) < s_piv) q = -s_piv;
      cnt += q < 0.0;
    }
    s_below = cnt;
    if (blockIdx.x == 0) *count = m - cnt;
  }
  __syncthreads();
  const int idx = s_below + blockIdx.x * blockDim.x + threadIdx.x;  // ascending index
  if (idx >= m) return;
  double a = fmax(bar, s_lo), b = s_hi;
  if (a > b) a = b;
  const double piv = s_piv;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (a + b);
    if (mid <= a || mid >= b || (b - a) <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b))) break;
    int cnt = 0;
    double q = d[0] - mid;
    if (fabs(q) < piv) q = -piv;
    cnt += q < 0.0;
    for (int i = 1; i < m; ++i) {
      q = (d[i] - mid) - (e[i - 1] * e[i - 1]) / q;
      if (fabs(q) < piv) q = -piv;
      cnt += q < 0.0;
    }
    if (cnt <= idx)
      a = mid;
    else
      b = mid;
  }
  vals[idx - s_below] = 0.5 * (a + b);
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
  SE_CUDA(cudaMemcpyAsync(d, d_host, sizeof(double) * m, cudaMemcpyHostToDevice, c.stream));
  if (m > 1)
    SE_CUDA(cudaMemcpyAsync(e, e_host, sizeof(double) * (m - 1), cudaMemcpyHostToDevice, c.stream));
  const int tb = 64;
  k_tridiag_above<<<(m + tb - 1) / tb, tb, 0, c.stream>>>(m, d, e, bar, vals, cnt);
  ++c.launches;
  SE_CUDA(cudaGetLastError());
  int h = 0;
  SE_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SE_CUDA(cudaStreamSynchronize(c.stream));
  out.resize(h);
  if (h)
    SE_CUDA(cudaMemcpyAsync(out.data(), vals, sizeof(double) * h, cudaMemcpyDeviceToHost, c.stream));
  SE_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace k
}  // namespace se
