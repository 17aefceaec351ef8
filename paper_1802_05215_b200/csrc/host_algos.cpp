// Host-side scalar algorithms (see host_algos.hpp).  Each routine restates the reference
// algorithm cited beside it; operation order is kept where the reference's rounding decides a
// discrete outcome (filter degree, slice breakpoints), so those match the reference bitwise.
#include "host_algos.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <thread>

namespace se {

namespace {
constexpr double kPi = 3.14159265358979323846;
inline double clamp1(double t) { return t < -1.0 ? -1.0 : (t > 1.0 ? 1.0 : t); }
}  // namespace

// rng.hpp:25-38 -- Box-Muller, first uniform strictly positive, spare kept across calls.
double Rng::normal() {
  if (spare_ok_) {
    spare_ok_ = false;
    return spare_;
  }
  double u1 = uniform();
  while (u1 <= 0.0) {
    ++rejections_;
    u1 = uniform();
  }
  const double u2 = uniform();
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * kPi * u2;
  spare_ = rad * std::sin(ang);
  spare_ok_ = true;
  return rad * std::cos(ang);
}

void fill_probes(Rng& rng, bool gaussian, int n, int b, double* out) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const bool exact = !gaussian || (n % 2 == 0 && !rng.spare_pending());
  const bool par = exact && b > 1 && hw > 1 && (long)n * b >= (1L << 21);
  auto draw = [&](Rng& r, double* dst) {
    if (gaussian)
      r.normal_fill(dst, n);
    else
      r.rademacher_fill(dst, n);
  };
  if (par) {
    // probe l starts l n draws after the block start (both kinds: exact by the test above)
    std::vector<Rng> loc((size_t)b, rng);
    std::vector<std::thread> th;
    th.reserve((size_t)b);
    for (int l = 0; l < b; ++l)
      th.emplace_back([&, l] {
        if (l) loc[(size_t)l].jump_draws(jump_poly((std::uint64_t)l * (std::uint64_t)n));
        draw(loc[(size_t)l], out + (size_t)l * n);
      });
    for (auto& t : th) t.join();
    long rej = 0;
    for (const Rng& r : loc) rej += r.rejections() - rng.rejections();
    if (rej == 0) {
      rng = loc[(size_t)b - 1];
      return;
    }
  }
  for (int l = 0; l < b; ++l) draw(rng, out + (size_t)l * n);
}

void fill_rademacher_bits(Rng& rng, int n, int b, std::uint64_t* out) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t words = ((size_t)n + 63) / 64;
  if (b > 1 && hw > 1 && (long)n * b >= (1L << 21)) {
    std::vector<Rng> loc((size_t)b, rng);
    std::vector<std::thread> th;
    th.reserve((size_t)b);
    for (int l = 0; l < b; ++l)
      th.emplace_back([&, l] {
        if (l) loc[(size_t)l].jump_draws(jump_poly((std::uint64_t)l * (std::uint64_t)n));
        loc[(size_t)l].rademacher_bits(out + (size_t)l * words, n);
      });
    for (auto& t : th) t.join();
    rng = loc[(size_t)b - 1];
    return;
  }
  for (int l = 0; l < b; ++l) rng.rademacher_bits(out + (size_t)l * words, n);
}

void skip_probes(Rng& rng, bool gaussian, int n, long count) {
  if (count <= 0) return;
  if (!gaussian || (n % 2 == 0 && !rng.spare_pending())) {
    rng.discard_draws((std::uint64_t)count * (std::uint64_t)n);
    return;
  }
  std::vector<double> skip((size_t)n);
  for (long l = 0; l < count; ++l) rng.normal_fill(skip.data(), n);
}

// ---- filters ------------------------------------------------------------------------------
// filter_poly.hpp:41-60
Vec damping_multipliers(int k, int kind) {
  Vec s(k + 1, 1.0);
  if (kind == SE_DAMP_SIGMA) {
    const double th = kPi / (k + 1);
    for (int j = 1; j <= k; ++j) s[j] = std::sin(j * th) / (j * th);
  } else if (kind == SE_DAMP_JACKSON) {
    const double q = kPi / (k + 2);
    const double cot = std::cos(q) / std::sin(q);
    for (int j = 1; j <= k; ++j) s[j] = ((k + 2 - j) * std::cos(j * q) + std::sin(j * q) * cot) / (k + 2);
  }
  return s;
}

// filter_poly.hpp:30-39
Vec chebyshev_coeffs(double gamma, int k) {
  if (!(std::abs(gamma) < 1.0))
    fail(SE_EINVAL, "chebyshev_coeffs: center must lie strictly inside (-1,1)");
  if (k < 0) fail(SE_EINVAL, "chebyshev_coeffs: negative degree");
  const double ac = std::acos(gamma);
  Vec mu(k + 1);
  mu[0] = 0.5;
  for (int j = 1; j <= k; ++j) mu[j] = std::cos(j * ac);
  return mu;
}

// filter_poly.hpp:65-77
double cheb_series(const double* coef, int k, double t) {
  double acc = coef[0];
  if (k == 0) return acc;
  double t0 = 1.0, t1 = t;
  acc += coef[1] * t1;
  for (int j = 2; j <= k; ++j) {
    const double t2 = 2.0 * t * t1 - t0;
    t0 = t1;
    t1 = t2;
    acc += coef[j] * t1;
  }
  return acc;
}

// filter_poly.hpp:93-97
double eval_pol(const double* mu, int k, double t) {
  if (std::abs(t) > 1.0 + 1e-12)
    fail(SE_EINVAL, "eval_pol: point outside the mapped interval [-1,1]");
  return cheb_series(mu, k, clamp1(t));
}

namespace {
// filter_poly.hpp:104-125 -- g(gamma) = N(ta) - N(tb) and its gamma-derivative.
void balance_eval(const Vec& s, double gamma, double ta, double tb, double& g, double& dg) {
  const int k = (int)s.size() - 1;
  const double ac = std::acos(gamma);
  const double rs = 1.0 / std::sqrt(std::max(1e-30, 1.0 - gamma * gamma));
  double pa = 1.0, ca = ta, pb = 1.0, cb = tb;
  g = 0.0;
  dg = 0.0;
  for (int j = 1; j <= k; ++j) {
    if (j > 1) {
      const double na = 2.0 * ta * ca - pa;
      pa = ca;
      ca = na;
      const double nb = 2.0 * tb * cb - pb;
      pb = cb;
      cb = nb;
    }
    const double diff = ca - cb;
    g += s[j] * std::cos(j * ac) * diff;
    dg += s[j] * j * std::sin(j * ac) * rs * diff;
  }
}
}  // namespace

// filter_poly.hpp:135-171 -- Newton from the midpoint, bisection fallback.
double balance_center(int k, double ta, double tb, int kind) {
  if (!(ta < tb) || ta < -1.0 - 1e-12 || tb > 1.0 + 1e-12)
    fail(SE_EINVAL, "balance_center: bad mapped interval");
  const Vec s = damping_multipliers(k, kind);
  const double lo = -1.0 + 1e-12, hi = 1.0 - 1e-12;
  auto settled = [](double g, double dg) { return std::abs(g) <= 1e-12 * (std::abs(dg) + 1.0); };
  double gamma = 0.5 * (ta + tb), g = 0.0, dg = 0.0;
  for (int it = 0; it < 50; ++it) {
    balance_eval(s, gamma, ta, tb, g, dg);
    if (settled(g, dg)) return gamma;
    if (dg == 0.0) break;
    gamma = std::clamp(gamma - g / dg, lo, hi);
  }
  balance_eval(s, gamma, ta, tb, g, dg);
  if (settled(g, dg)) return gamma;
  double a = ta, b = tb, ga, gb, unused;
  balance_eval(s, a, ta, tb, ga, unused);
  balance_eval(s, b, ta, tb, gb, unused);
  if (ga * gb > 0.0) {
    a = lo;
    b = hi;
    balance_eval(s, a, ta, tb, ga, unused);
    balance_eval(s, b, ta, tb, gb, unused);
    if (ga * gb > 0.0) fail(SE_ENUMERIC, "balance_center: no balanced center found");
  }
  for (int it = 0; it < 200; ++it) {
    gamma = 0.5 * (a + b);
    balance_eval(s, gamma, ta, tb, g, unused);
    if (std::abs(g) <= 1e-14 || b - a <= 1e-15) return gamma;
    if (ga * g > 0.0) {
      a = gamma;
      ga = g;
    } else {
      b = gamma;
      gb = g;
    }
  }
  return gamma;
}

// filter_poly.hpp:182-190
Vec normalized_filter_coeffs(int k, double gamma, int kind) {
  Vec mu = chebyshev_coeffs(gamma, k);
  const Vec s = damping_multipliers(k, kind);
  for (int j = 0; j <= k; ++j) mu[j] *= s[j];
  const double den = cheb_series(mu.data(), k, gamma);
  if (den == 0.0) fail(SE_ENUMERIC, "find_pol: degenerate normalization");
  for (double& m : mu) m /= den;
  return mu;
}

// filter_poly.hpp:198-253 -- lowest degree k >= 2 whose balanced filter puts both mapped slice
// endpoints under tau; one-sided filters for slices touching the spectrum ends.
PolyFilter find_pol(double xi, double eta, double lmin, double lmax, double tau, int max_deg,
                    int kind) {
  if (!(eta > xi)) fail(SE_EINVAL, "find_pol: degenerate interval");
  if (eta < lmin || xi > lmax) fail(SE_EINVAL, "find_pol: interval does not overlap the spectrum");
  PolyFilter f;
  f.c = 0.5 * (lmax + lmin);
  f.d = 0.5 * (lmax - lmin);
  if (!(f.d > 0.0)) fail(SE_EINVAL, "SpectralMap: empty spectral interval");
  f.tau = tau;
  f.damping = kind;
  const double ta_raw = (xi - f.c) / f.d, tb_raw = (eta - f.c) / f.d;
  f.ta = clamp1(ta_raw);
  f.tb = clamp1(tb_raw);
  const bool at_lo = ta_raw <= -1.0 + 1e-12, at_hi = tb_raw >= 1.0 - 1e-12;
  const double width = f.tb - f.ta;
  if (!(width > 0.0)) fail(SE_EINVAL, "find_pol: empty mapped interval");
  const double pin = std::min(0.01, 0.1 * width);
  for (int k = 2;; ++k) {
    if (at_lo && at_hi)
      f.gamma = 0.5 * (f.ta + f.tb);
    else if (at_lo)
      f.gamma = -1.0 + pin;
    else if (at_hi)
      f.gamma = 1.0 - pin;
    else
      f.gamma = balance_center(k, f.ta, f.tb, kind);
    f.k = k;
    f.mu = normalized_filter_coeffs(k, f.gamma, kind);
    const double ra = eval_pol(f.mu.data(), k, f.ta), rb = eval_pol(f.mu.data(), k, f.tb);
    bool ok;
    if (at_lo && at_hi)
      ok = true;
    else if (at_lo)
      ok = rb <= tau;
    else if (at_hi)
      ok = ra <= tau;
    else
      ok = ra <= tau && rb <= tau && f.gamma > f.ta && f.gamma < f.tb;
    if (ok || k >= max_deg) {
      f.cap_reached = !ok;
      double bar = std::min(ra, rb);
      if (at_lo || at_hi)
        for (int i = 1; i < 200; ++i)
          bar = std::min(bar, eval_pol(f.mu.data(), k, f.ta + width * i / 200.0));
      f.bar = bar;
      return f;
    }
  }
}

// ---- density of states ----------------------------------------------------------------------
Vec dos_grid(double lmin, double lmax, int npts) {  // dos.hpp:41-45
  Vec x(npts);
  for (int i = 0; i < npts; ++i) x[i] = lmin + (lmax - lmin) * i / (npts - 1);
  return x;
}

static double trapezoid(const Vec& x, const Vec& y) {  // dos.hpp:47-51
  double s = 0.0;
  for (size_t i = 1; i < x.size(); ++i) s += 0.5 * (y[i] + y[i - 1]) * (x[i] - x[i - 1]);
  return s;
}

void dos_finalize(Curve& c) {  // dos.hpp:54-60
  for (double& v : c.y) v = std::max(v, 0.0);
  const double mass = trapezoid(c.x, c.y);
  if (!(mass > 0.0)) fail(SE_ENUMERIC, "dos: vanishing density estimate");
  for (double& v : c.y) v /= mass;
  c.nev_est = c.n * trapezoid(c.x, c.y);
}

// dos.hpp:112-131 -- Jackson-damped Chebyshev density from normalised moments.
Curve kpm_curve(const Vec& zeta, int n, double lmin, double lmax, int npts) {
  const int m = (int)zeta.size() - 1;
  const double c = 0.5 * (lmax + lmin), d = 0.5 * (lmax - lmin);
  const Vec g = damping_multipliers(m, SE_DAMP_JACKSON);
  Curve cv;
  cv.n = n;
  cv.x = dos_grid(lmin, lmax, npts);
  cv.y.resize(npts);
  for (int i = 0; i < npts; ++i) {
    const double th = (cv.x[i] - c) / d;
    double s = 0.5 * g[0] * zeta[0];
    const double ang = std::acos(std::min(1.0, std::max(-1.0, th)));
    for (int k = 1; k <= m; ++k) s += g[k] * zeta[k] * std::cos(k * ang);
    const double under = std::max(1.0 - th * th, 1e-10);
    cv.y[i] = 2.0 / (kPi * std::sqrt(under)) * s / d;
  }
  cv.y[0] = cv.y[1];
  cv.y[npts - 1] = cv.y[npts - 2];
  dos_finalize(cv);
  return cv;
}

// dos.hpp:63-75 -- Ritz-value Gaussians weighted by squared first eigenvector components.
void add_ritz_gaussians(const Vec& theta, const Vec& tau2, const Vec& x, double sigma, Vec& y) {
  const double norm = 1.0 / (sigma * std::sqrt(2.0 * kPi));
  for (size_t i = 0; i < theta.size(); ++i)
    for (size_t j = 0; j < x.size(); ++j) {
      const double u = (x[j] - theta[i]) / sigma;
      y[j] += tau2[i] * norm * std::exp(-0.5 * u * u);
    }
}

// dos.hpp:190-207
double dos_cumulative(const Curve& c, double t) {
  double s = 0.0;
  for (size_t i = 1; i < c.x.size(); ++i) {
    if (t >= c.x[i]) {
      s += 0.5 * (c.y[i] + c.y[i - 1]) * (c.x[i] - c.x[i - 1]);
      continue;
    }
    const double f = (t - c.x[i - 1]) / (c.x[i] - c.x[i - 1]);
    if (f > 0.0) {
      const double yt = c.y[i - 1] + f * (c.y[i] - c.y[i - 1]);
      s += 0.5 * (yt + c.y[i - 1]) * (t - c.x[i - 1]);
    }
    break;
  }
  return s;
}

// dos.hpp:212-218
double dos_count(const Curve& c, double xi, double eta) {
  if (c.x.size() < 2) fail(SE_EINVAL, "dos_count: curve has no grid");
  const double slack = 1e-12 * (c.x.back() - c.x.front());
  if (xi > eta || xi < c.x.front() - slack || eta > c.x.back() + slack)
    fail(SE_EINVAL, "dos_count: interval outside the curve range");
  return c.n * (dos_cumulative(c, eta) - dos_cumulative(c, xi));
}

// slicer.hpp:18-64 -- breakpoints = first free grid point whose cumulative share reaches i/ns.
void slice_spectrum(const Curve& c, double xi, double eta, int ns, Vec& bp, Vec& est) {
  if (ns < 1) fail(SE_EINVAL, "slice_spectrum: need at least one slice");
  if (!(xi < eta)) fail(SE_EINVAL, "slice_spectrum: empty target interval");
  const Vec& x = c.x;
  if (x.size() < 2) fail(SE_EINVAL, "slice_spectrum: curve has no grid");
  const double slack = 1e-12 * (x.back() - x.front());
  if (xi < x.front() - slack || eta > x.back() + slack)
    fail(SE_EINVAL, "slice_spectrum: interval outside the curve range");
  const int npts = (int)x.size();
  int interior = 0;
  for (double t : x) interior += (t > xi && t < eta);
  if (ns > interior + 1) fail(SE_EINVAL, "slice_spectrum: more slices than interior grid points");
  Vec cum(npts, 0.0);
  for (int j = 1; j < npts; ++j) cum[j] = cum[j - 1] + 0.5 * (c.y[j] + c.y[j - 1]) * (x[j] - x[j - 1]);
  const double base = dos_cumulative(c, xi);
  const double total = dos_cumulative(c, eta) - base;
  bp.assign(1, xi);
  int j = 0;
  for (int i = 1; i < ns; ++i) {
    const double target = total * i / ns;
    while (j < npts && (x[j] <= bp.back() || x[j] <= xi)) ++j;
    int cand = j;
    while (cand < npts && x[cand] < eta && cum[cand] - base < target) ++cand;
    if (cand >= npts || x[cand] >= eta) cand = j;
    if (cand >= npts || x[cand] >= eta) fail(SE_ENUMERIC, "slice_spectrum: curve grid too coarse");
    bp.push_back(x[cand]);
    j = cand + 1;
  }
  bp.push_back(eta);
  est.resize(ns);
  for (int i = 0; i < ns; ++i) est[i] = dos_count(c, bp[i], bp[i + 1]);
}

// ---- symmetric eigensolvers -------------------------------------------------------------------
// Implicit QL with Wilkinson shifts on (d, e), e[i] couples d[i], d[i+1] (tridiag_eig.hpp:34-90).
// z: optional column-major rotation accumulator with `zrows` rows.
void tridiag_ql(Vec& d, Vec& e, double* z, int ldz, int zrows) {
  const int m = (int)d.size();
  if (m == 0) return;
  e.resize(m);
  e[m - 1] = 0.0;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    for (;;) {
      int sp = l;
      for (; sp < m - 1; ++sp) {
        const double dd = std::abs(d[sp]) + std::abs(d[sp + 1]);
        if (std::abs(e[sp]) <= 1e-16 * dd) break;
      }
      if (sp == l) break;
      if (iter++ == 60) fail(SE_ENUMERIC, "ql_implicit: too many iterations (should not happen)");
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[sp] - d[l] + e[l] / (g + std::copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0;
      bool underflow = false;
      for (int i = sp - 1; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[sp] = 0.0;
          underflow = true;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        if (z) {
          double* zi = z + (size_t)i * ldz;
          double* zj = z + (size_t)(i + 1) * ldz;
          for (int q = 0; q < zrows; ++q) {
            const double t = zj[q];
            zj[q] = s * zi[q] + c * t;
            zi[q] = c * zi[q] - s * t;
          }
        }
      }
      if (underflow) continue;
      d[l] -= p;
      e[l] = g;
      e[sp] = 0.0;
    }
  }
}

void sort_eigs(Vec& d, double* z, int m) {  // stable ascending (tridiag_eig.hpp:93-107)
  std::vector<int> perm(m);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return d[a] < d[b]; });
  Vec ds(m);
  for (int j = 0; j < m; ++j) ds[j] = d[perm[j]];
  d.swap(ds);
  if (z) {
    Vec zs((size_t)m * m);
    for (int j = 0; j < m; ++j)
      std::copy(z + (size_t)perm[j] * m, z + (size_t)perm[j] * m + m, zs.data() + (size_t)j * m);
    std::copy(zs.begin(), zs.end(), z);
  }
}

void sym_tridiag_eig(const Vec& alpha, const Vec& beta, bool want, Vec& values, Vec& vectors) {
  const int m = (int)alpha.size();
  if (m > 0 && (int)beta.size() != m - 1)
    fail(SE_EINVAL, "sym_tridiag_eig: beta must have length m-1");
  values = alpha;
  Vec e = beta;
  e.resize(std::max(m, 1));
  if (want) {
    vectors.assign((size_t)m * m, 0.0);
    for (int j = 0; j < m; ++j) vectors[(size_t)j * m + j] = 1.0;
    tridiag_ql(values, e, vectors.data(), m, m);
    sort_eigs(values, vectors.data(), m);
  } else {
    vectors.clear();
    tridiag_ql(values, e, nullptr, 0, 0);
    sort_eigs(values, nullptr, m);
  }
}

// Dense symmetric eigensolver for small host problems: Householder tridiagonalisation with the
// accumulated orthogonal factor, then implicit QL (the method of dense_eig.hpp:114-139).
void dense_sym_eig(int m, const double* a, bool want, Vec& values, Vec& vectors) {
  Vec A(a, a + (size_t)m * m);  // column-major, symmetric
  auto at = [&](int i, int j) -> double& { return A[(size_t)j * m + i]; };
  Vec Q;
  if (want) {
    Q.assign((size_t)m * m, 0.0);
    for (int j = 0; j < m; ++j) Q[(size_t)j * m + j] = 1.0;
  }
  Vec v(m), p(m), w(m);
  for (int k = 0; k + 2 < m; ++k) {
    // Householder vector for A[k+1:, k]
    double alpha = 0.0;
    for (int i = k + 1; i < m; ++i) alpha += at(i, k) * at(i, k);
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    const double x0 = at(k + 1, k);
    if (x0 > 0) alpha = -alpha;
    std::fill(v.begin(), v.end(), 0.0);
    v[k + 1] = x0 - alpha;
    for (int i = k + 2; i < m; ++i) v[i] = at(i, k);
    double vv = 0.0;
    for (int i = k + 1; i < m; ++i) vv += v[i] * v[i];
    if (vv == 0.0) continue;
    const double tau = 2.0 / vv;
    // p = tau A v ; w = p - (tau/2)(v'p) v ; A -= v w' + w v'
    for (int i = k; i < m; ++i) {
      double s = 0.0;
      for (int j = k + 1; j < m; ++j) s += at(i, j) * v[j];
      p[i] = tau * s;
    }
    double vp = 0.0;
    for (int i = k + 1; i < m; ++i) vp += v[i] * p[i];
    const double kk = 0.5 * tau * vp;
    for (int i = k; i < m; ++i) w[i] = p[i] - kk * v[i];
    for (int j = k; j < m; ++j)
      for (int i = k; i < m; ++i) at(i, j) -= v[i] * w[j] + w[i] * v[j];
    if (want)  // Q <- Q H
      for (int i = 0; i < m; ++i) {
        double s = 0.0;
        for (int j = k + 1; j < m; ++j) s += Q[(size_t)j * m + i] * v[j];
        s *= tau;
        for (int j = k + 1; j < m; ++j) Q[(size_t)j * m + i] -= s * v[j];
      }
  }
  values.resize(m);
  Vec e(std::max(m, 1), 0.0);
  for (int i = 0; i < m; ++i) values[i] = at(i, i);
  for (int i = 0; i + 1 < m; ++i) e[i] = at(i + 1, i);
  if (want) {
    tridiag_ql(values, e, Q.data(), m, m);
    sort_eigs(values, Q.data(), m);
    vectors.swap(Q);
  } else {
    tridiag_ql(values, e, nullptr, 0, 0);
    sort_eigs(values, nullptr, m);
    vectors.clear();
  }
}

// Givens reduction of the thick-restart arrowhead (see header).  Invariant after bringing in
// index j: the block 0..j is tridiagonal (a, b) and only row j couples to the tip (sigma).
void arrow_to_tridiag(const Vec& theta, const Vec& s, double alpha_l, Vec& diag, Vec& off) {
  const int l = (int)theta.size();
  diag.assign(l + 1, 0.0);
  off.assign(l, 0.0);
  if (l == 0) {
    diag[0] = alpha_l;
    return;
  }
  Vec a(theta), b(l, 0.0);  // b[q] couples q and q+1 (q < l-1 inside the block)
  double sigma = s[0];
  for (int j = 0; j + 1 < l; ++j) {
    // rotate plane (j, j+1) so that the tip coupling moves entirely to row j+1
    const double sn = s[j + 1];
    const double r = std::hypot(sigma, sn);
    if (r == 0.0) {
      sigma = 0.0;
      continue;
    }
    const double c = sn / r, sg = -sigma / r;  // new_p = c x_p + sg x_{p+1}, new_{p+1} = -sg x_p + c x_{p+1}
    double bulge = 0.0;
    if (j > 0) {
      const double bj = b[j - 1];
      b[j - 1] = c * bj;
      bulge = -sg * bj;  // entry (j-1, j+1)
    }
    {
      const double x = a[j], z = a[j + 1], y = 0.0;
      a[j] = c * c * x + 2.0 * c * sg * y + sg * sg * z;
      a[j + 1] = sg * sg * x - 2.0 * c * sg * y + c * c * z;
      b[j] = c * sg * (z - x) + (c * c - sg * sg) * y;
    }
    sigma = r;
    // chase the bulge at (q-1, q+1) upwards with rotations in plane (q-1, q)
    for (int q = j; q >= 1 && bulge != 0.0; --q) {
      const double bq = b[q];  // (q, q+1)
      const double rr = std::hypot(bq, bulge);
      const double cc = bq / rr, ss = -bulge / rr;
      b[q] = rr;  // new (q, q+1)
      double nb = 0.0;
      if (q >= 2) {
        const double bm = b[q - 2];  // (q-2, q-1)
        b[q - 2] = cc * bm;
        nb = -ss * bm;  // new bulge (q-2, q)
      }
      const double x = a[q - 1], z = a[q], y = b[q - 1];
      a[q - 1] = cc * cc * x + 2.0 * cc * ss * y + ss * ss * z;
      a[q] = ss * ss * x - 2.0 * cc * ss * y + cc * cc * z;
      b[q - 1] = cc * ss * (z - x) + (cc * cc - ss * ss) * y;
      bulge = nb;
    }
  }
  for (int q = 0; q < l; ++q) diag[q] = a[q];
  diag[l] = alpha_l;
  for (int q = 0; q + 1 < l; ++q) off[q] = b[q];
  off[l - 1] = sigma;
}

}  // namespace se

namespace se {

// Chebyshev least squares for B^-1 / B^-1/2 (cheb_approx.hpp:40-88): the normal equations of a
// Chebyshev-weighted fit on Chebyshev nodes are diagonal, so each coefficient is a cosine sum.
ChebFit ls_pol_approx(bool inverse_sqrt, double lmin, double lmax, double tol, int max_deg) {
  if (lmin <= 0.0) fail(SE_EINVAL, "ls_pol_approx: interval must be positive (B must be SPD)");
  if (lmax <= lmin) fail(SE_EINVAL, "ls_pol_approx: empty interval");
  if (max_deg < 1) fail(SE_EINVAL, "ls_pol_approx: max_deg must be positive");
  const double pi = 3.14159265358979323846;
  const double mid = 0.5 * (lmax + lmin), half = 0.5 * (lmax - lmin);
  auto fun = [&](double t) { return inverse_sqrt ? 1.0 / std::sqrt(t) : 1.0 / t; };
  const int nodes = 4 * max_deg;
  Vec node(nodes), fval(nodes);
  for (int i = 0; i < nodes; ++i) {
    node[i] = std::cos(pi * (i + 0.5) / nodes);
    fval[i] = fun(mid + half * node[i]);
  }
  Vec coef(max_deg + 1);
  for (int j = 0; j <= max_deg; ++j) {
    double acc = 0.0;
    for (int i = 0; i < nodes; ++i) acc += fval[i] * std::cos(j * std::acos(node[i]));
    coef[j] = (j == 0 ? 1.0 : 2.0) * acc / nodes;
  }
  // Clenshaw evaluation of a truncation on the mapped argument
  auto series = [&](int deg, double t) {
    const double x = (t - mid) / half;
    double b1 = 0.0, b2 = 0.0;
    for (int j = deg; j >= 1; --j) {
      const double b0 = 2.0 * x * b1 - b2 + coef[j];
      b2 = b1;
      b1 = b0;
    }
    return x * b1 - b2 + coef[0];
  };
  const int grid = 2000;
  double worst = 0.0;
  for (int deg = 1; deg <= max_deg; ++deg) {
    worst = 0.0;
    for (int i = 0; i <= grid; ++i) {
      const double t = lmin + (lmax - lmin) * i / grid;
      worst = std::max(worst, std::abs(series(deg, t) - fun(t)) / std::abs(fun(t)));
    }
    if (worst <= tol) return {Vec(coef.begin(), coef.begin() + deg + 1), worst};
  }
  fail(SE_ENUMERIC, "ls_pol_approx: tolerance not reached; best relative error " +
                        std::to_string(worst) + " at degree " + std::to_string(max_deg));
}

}  // namespace se
