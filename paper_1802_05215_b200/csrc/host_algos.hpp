// Host-side scalar algorithms of the path (O(k^2) / O(m^2) work that stays on the CPU):
// filter construction, DOS curve + slicing, small symmetric eigensolvers, Rng streams.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"
#include "mt64.hpp"

namespace se {

using Vec = std::vector<double>;

// ---- rng.hpp:15-61: mt19937_64 + explicit transforms ---------------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : g_(seed) {}
  double uniform() { return double(g_() >> 11) * 0x1.0p-53; }
  double normal();
  double rademacher() { return (g_() & 1u) ? 1.0 : -1.0; }
  void normal_fill(double* out, long n) {
    for (long i = 0; i < n; ++i) out[i] = normal();
  }
  void rademacher_fill(double* out, long n) {
    for (long i = 0; i < n; ++i) out[i] = rademacher();
  }
  // the signs of the next n Rademacher draws as bits (bit i of word i / 64: 1 -> +1, 0 -> -1)
  void rademacher_bits(std::uint64_t* out, long n) {
    for (long w = 0; w * 64 < n; ++w) {
      const int lim = (int)std::min<long>(64, n - w * 64);
      std::uint64_t word = 0;
      for (int q = 0; q < lim; ++q) word |= (g_() & 1u) << q;
      out[w] = word;
    }
  }
  // advance the engine by j draws (jump-ahead for large j); the Box-Muller spare is untouched
  void discard_draws(std::uint64_t j) { g_.discard(j); }
  void jump_draws(const std::vector<std::uint64_t>& g) { g_.jump(g); }
  bool spare_pending() const { return spare_ok_; }
  long rejections() const { return rejections_; }

 private:
  Mt64 g_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
  long rejections_ = 0;  // u1 <= 0 redraws (shift the draw count; rng.hpp:36-41)
};

// Probes [0, b) of the stream (probe l = the next n draws: rademacher, or n normals), stored
// probe-major (out[l n + i]); rng ends where the serial draw would.  Host threads start their
// probes by jump-ahead when that is exact (Rademacher; Gaussian with n even and no pending
// spare -- then every probe is exactly n draws); otherwise, or on a Box-Muller redraw, serial.
void fill_probes(Rng& rng, bool gaussian, int n, int b, double* out);
// Rademacher probes [0, b) as sign bits: probe l at out + l * ((n + 63) / 64) (same stream,
// same jump-ahead threading; 1/64 of the host memory traffic of the double layout).
void fill_rademacher_bits(Rng& rng, int n, int b, std::uint64_t* out);
// Skip `count` probes of n values each (jump-ahead when exact, else serial draws).
void skip_probes(Rng& rng, bool gaussian, int n, long count);

// ---- filter_poly.hpp ----------------------------------------------------------------------
struct PolyFilter {
  int k = 0;
  double gamma = 0.0;
  Vec mu;
  double c = 0.0, d = 1.0;
  double tau = 0.8;
  double ta = -1.0, tb = 1.0;
  double bar = 0.0;
  int damping = SE_DAMP_SIGMA;
  bool cap_reached = false;
};

Vec damping_multipliers(int k, int kind);
Vec chebyshev_coeffs(double gamma, int k);
double cheb_series(const double* coef, int k, double t);
double eval_pol(const double* mu, int k, double t);  // throws SE_EINVAL outside [-1-1e-12, 1+1e-12]
double balance_center(int k, double ta, double tb, int kind);
Vec normalized_filter_coeffs(int k, double gamma, int kind);
PolyFilter find_pol(double xi, double eta, double lmin, double lmax, double tau, int max_deg,
                    int kind);

// ---- dos.hpp / slicer.hpp ------------------------------------------------------------------
struct Curve {
  Vec x, y;
  double nev_est = 0.0;
  int n = 0;
};
Vec dos_grid(double lmin, double lmax, int npts);
Curve kpm_curve(const Vec& zeta_normalised, int n, double lmin, double lmax, int npts);
void dos_finalize(Curve& c);
void add_ritz_gaussians(const Vec& theta, const Vec& tau2, const Vec& x, double sigma, Vec& y);
double dos_cumulative(const Curve& c, double t);
double dos_count(const Curve& c, double xi, double eta);
void slice_spectrum(const Curve& c, double xi, double eta, int ns, Vec& bp, Vec& est);

// ---- cheb_approx.hpp:40-88 -----------------------------------------------------------------
// Chebyshev least-squares fit of 1/t (inverse_sqrt = false) or 1/sqrt(t) on [lmin, lmax] (> 0):
// discrete cosine sums on 4 max_deg Chebyshev nodes, truncated at the smallest degree whose
// relative error on a 2,001-point grid is <= tol.  Throws SE_EINVAL for a non-positive or
// empty interval and SE_ENUMERIC when max_deg does not reach tol.
struct ChebFit {
  Vec coeff;  // degree = size - 1
  double achieved = 0.0;
};
ChebFit ls_pol_approx(bool inverse_sqrt, double lmin, double lmax, double tol, int max_deg);

// ---- tridiag_eig.hpp / dense_eig.hpp --------------------------------------------------------
// Symmetric tridiagonal eigenproblem (implicit QL, Wilkinson shift); Z (m x m col-major) optional.
void tridiag_ql(Vec& d, Vec& e, double* z, int ldz, int zrows);
void sort_eigs(Vec& d, double* z, int m);
void sym_tridiag_eig(const Vec& alpha, const Vec& beta, bool want, Vec& values, Vec& vectors);
void dense_sym_eig(int m, const double* a, bool want, Vec& values, Vec& vectors);

// Reduce a thick-restart arrowhead block (diag theta[0..l-1] coupled to index l through s[j],
// with H(l,l) = alpha_l) to tridiagonal form by Givens rotations acting on indices 0..l-1
// (index l stays last, so the following Lanczos tail continues the chain).  O(l^2).
// Output: diag[0..l], off[0..l-1] (off[j] couples j and j+1).
void arrow_to_tridiag(const Vec& theta, const Vec& s, double alpha_l, Vec& diag, Vec& off);

}  // namespace se
