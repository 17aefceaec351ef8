// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never on the product path).
//
// A thin C-ABI harness around the UNMODIFIED reference headers
// (/root/reference/proj/include/sliceeig/*.hpp, compiled in place; nothing is copied).
// Built by oracle/Makefile into oracle/_ref/libsliceeig_ref.so.  Used by:
//   * tests/golden/make_golden.py  -- generates the committed golden fixtures;
//   * tests/ (as the checker)        -- parity of the CUDA path against the real reference;
//   * bench.py --impl reference / cpu_baseline -- the reference CPU path timed on the host.
//
// Where the reference has no public entry point for a quantity the parity contract needs
// (the raw KPM moments; Gaussian probes from BASELINE cfg2), the harness restates the
// reference loop using the reference's own primitives, citing the lines it follows.

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "sliceeig/cheb_approx.hpp"
#include "sliceeig/cholesky.hpp"
#include "sliceeig/dos.hpp"
#include "sliceeig/eigensolvers.hpp"
#include "sliceeig/filter_poly.hpp"
#include "sliceeig/laplacian.hpp"
#include "sliceeig/lanczos.hpp"
#include "sliceeig/orth.hpp"
#include "sliceeig/slicer.hpp"

using namespace sliceeig;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

CsrMatrix make_csr(int n, const int* rp, const int* ci, const double* v) {
  // Assemble through from_triplets so the reference's own invariants hold.
  std::vector<Triplet> t;
  t.reserve(rp[n]);
  for (int i = 0; i < n; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) t.push_back({i, ci[k], v[k]});
  return CsrMatrix::from_triplets(n, std::move(t));
}

Damping damping_of(int d) {
  return d == 0 ? Damping::None : (d == 2 ? Damping::Jackson : Damping::LanczosSigma);
}

// Raw (normalised) KPM moments, restating dos.hpp:96-110 with the reference primitives.
// probe_kind 0 = Rademacher (rng.hpp:41, as dos.hpp:97), 1 = Gaussian (rng.hpp:25-38,
// BASELINE cfg2's "seeded Gaussian probes": Rng(seed).normal_vec(n) per probe, probe order).
Vec kpm_moments(const Operator& op, const SpectralBounds& bounds, int m, int n_vec,
                std::uint64_t seed, int probe_kind, int first_probe, int nprobes) {
  const SpectralMap map{bounds};
  const int n = op.n;
  auto mapped = [&](const Vec& w, Vec& t) {
    op.apply(w, t);
    for (int i = 0; i < n; ++i) t[i] = (t[i] - map.c * w[i]) / map.d;
  };
  Vec zeta(m + 1, 0.0);
  Rng rng(seed);
  Vec w0, w1(n), t(n);
  for (int l = 0; l < n_vec; ++l) {
    const Vec v = probe_kind == 1 ? rng.normal_vec(n) : rng.rademacher_vec(n);
    if (l < first_probe || l >= first_probe + nprobes) continue;
    w0 = v;
    mapped(w0, w1);
    zeta[0] += dot(v, w0);
    if (m >= 1) zeta[1] += dot(v, w1);
    for (int k = 2; k <= m; ++k) {
      mapped(w1, t);
      for (int i = 0; i < n; ++i) t[i] = 2.0 * t[i] - w0[i];
      zeta[k] += dot(v, t);
      w0.swap(w1);
      w1.swap(t);
    }
  }
  return zeta;  // unnormalised sums; caller divides by n_vec*n (dos.hpp:110)
}

// KPM curve from normalised moments, restating dos.hpp:112-131 (used for Gaussian probes;
// checked bitwise against kpm_dos for Rademacher probes in tests/test_golden_ref.py).
DosCurve curve_from_moments(const Vec& zeta, int n, const SpectralBounds& bounds, int npts) {
  const SpectralMap map{bounds};
  const int m = (int)zeta.size() - 1;
  const Vec g = damping_multipliers(m, Damping::Jackson);
  DosCurve c;
  c.n = n;
  c.xdos = detail::dos_grid(bounds, npts);
  c.ydos.resize(npts);
  for (int i = 0; i < npts; ++i) {
    const double th = map.to_ref(c.xdos[i]);
    double s = 0.5 * g[0] * zeta[0];
    const double ang = std::acos(std::min(1.0, std::max(-1.0, th)));
    for (int k = 1; k <= m; ++k) s += g[k] * zeta[k] * std::cos(k * ang);
    const double under = std::max(1.0 - th * th, 1e-10);
    c.ydos[i] = 2.0 / (kPi * std::sqrt(under)) * s / map.d;
  }
  c.ydos[0] = c.ydos[1];
  c.ydos[npts - 1] = c.ydos[npts - 2];
  detail::dos_finalize(c);
  return c;
}

struct ResultSet {
  // One or more slice results, concatenated.
  std::vector<EigenResults> slices;
  std::vector<double> breakpoints, est;
  std::vector<int> degrees;
  std::vector<std::string> errors;
  double lmin = 0, lmax = 0;
  double t_bounds = 0, t_dos = 0, t_solve = 0, t_total = 0;
};

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- matrices ----------------------------------------------------------------------------
// Sizes first (rp == nullptr), then fill.
int ref_laplacian(int ndims, const int* dims, int* n, long* nnz, int* rp, int* ci, double* v) {
  return guarded([&] {
    std::vector<int> d(dims, dims + ndims);
    CsrMatrix a = gen_laplacian(d);
    *n = a.n();
    *nnz = a.nnz();
    if (rp) {
      std::memcpy(rp, a.row_ptr().data(), sizeof(int) * (a.n() + 1));
      std::memcpy(ci, a.col_idx().data(), sizeof(int) * a.nnz());
      std::memcpy(v, a.vals().data(), sizeof(double) * a.nnz());
    }
  });
}

int ref_laplacian_eigs(int ndims, const int* dims, double* out) {
  return guarded([&] {
    Vec e = laplacian_analytic_eigs(std::vector<int>(dims, dims + ndims));
    std::memcpy(out, e.data(), sizeof(double) * e.size());
  });
}

int ref_matvec(int n, const int* rp, const int* ci, const double* v, const double* x, double* y) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    Vec xx(x, x + n), yy;
    a.matvec(xx, yy);
    std::memcpy(y, yy.data(), sizeof(double) * n);
  });
}

// ---- rng -----------------------------------------------------------------------------------
// `count` consecutive normal_vec(n) / rademacher_vec(n) draws from one Rng(seed).
int ref_rng_normal(std::uint64_t seed, int n, int count, double* out) {
  return guarded([&] {
    Rng r(seed);
    for (int c = 0; c < count; ++c) {
      Vec v = r.normal_vec(n);
      std::memcpy(out + (std::size_t)c * n, v.data(), sizeof(double) * n);
    }
  });
}
int ref_rng_rademacher(std::uint64_t seed, int n, int count, double* out) {
  return guarded([&] {
    Rng r(seed);
    for (int c = 0; c < count; ++c) {
      Vec v = r.rademacher_vec(n);
      std::memcpy(out + (std::size_t)c * n, v.data(), sizeof(double) * n);
    }
  });
}
int ref_rng_uniform(std::uint64_t seed, int n, double* out) {
  return guarded([&] {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
  });
}

// ---- filters -------------------------------------------------------------------------------
int ref_find_pol(double xi, double eta, double lmin, double lmax, double tau, int max_deg,
                 int damping, int mu_cap, int* k, double* gamma, double* mu, double* ta,
                 double* tb, double* bar, int* cap_reached, double* c, double* d) {
  return guarded([&] {
    PolyOpts o;
    o.tau = tau;
    o.max_deg = max_deg;
    o.damping = damping_of(damping);
    PolynomialFilter f = find_pol(xi, eta, SpectralBounds{lmin, lmax}, o);
    *k = f.k;
    *gamma = f.gamma;
    if (f.k + 1 > mu_cap) throw std::runtime_error("ref_find_pol: mu buffer too small");
    std::memcpy(mu, f.mu.data(), sizeof(double) * (f.k + 1));
    *ta = f.ta;
    *tb = f.tb;
    *bar = f.bar;
    *cap_reached = f.cap_reached;
    *c = f.map.c;
    *d = f.map.d;
  });
}

int ref_balance_center(int k, double ta, double tb, int damping, double* gamma) {
  return guarded([&] { *gamma = balance_center(k, ta, tb, damping_of(damping)); });
}

int ref_damping(int k, int damping, double* out) {
  return guarded([&] {
    Vec s = damping_multipliers(k, damping_of(damping));
    std::memcpy(out, s.data(), sizeof(double) * (k + 1));
  });
}

int ref_normalized_coeffs(int k, double gamma, int damping, double* out) {
  return guarded([&] {
    Vec mu = detail::normalized_filter_coeffs(k, gamma, damping_of(damping));
    std::memcpy(out, mu.data(), sizeof(double) * (k + 1));
  });
}

int ref_eval_series(int k, const double* mu, double t, double* out) {
  return guarded([&] {
    PolynomialFilter f;
    f.k = k;
    f.mu.assign(mu, mu + k + 1);
    *out = eval_pol(f, t);
  });
}

// apply_pol with a filter given by (k, mu, c, d) (filter_poly.hpp:256-277).
int ref_apply_pol(int n, const int* rp, const int* ci, const double* v, int k, const double* mu,
                  double c, double d, const double* x, double* out, long* n_matvec) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    PolynomialFilter f;
    f.k = k;
    f.mu.assign(mu, mu + k + 1);
    f.map.c = c;
    f.map.d = d;
    Operator op = make_operator(a);
    Vec xx(x, x + n), o;
    Counters cnt;
    apply_pol(f, op, xx, o, &cnt);
    std::memcpy(out, o.data(), sizeof(double) * n);
    *n_matvec = cnt.n_A_matvec;
  });
}

// ---- density of states ---------------------------------------------------------------------
int ref_kpm_moments(int n, const int* rp, const int* ci, const double* v, double lmin, double lmax,
                    int m, int n_vec, std::uint64_t seed, int probe_kind, int first_probe,
                    int nprobes, double* zeta_sums) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    Vec z = kpm_moments(make_operator(a), {lmin, lmax}, m, n_vec, seed, probe_kind, first_probe,
                        nprobes);
    std::memcpy(zeta_sums, z.data(), sizeof(double) * (m + 1));
  });
}

int ref_kpm_dos(int n, const int* rp, const int* ci, const double* v, double lmin, double lmax,
                int m, int n_vec, int npts, std::uint64_t seed, double* x, double* y,
                double* nev_est) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    DosConfig cfg;
    cfg.m = m;
    cfg.n_vec = n_vec;
    cfg.npts = npts;
    cfg.seed = seed;
    DosCurve c = kpm_dos(make_operator(a), {lmin, lmax}, cfg);
    std::memcpy(x, c.xdos.data(), sizeof(double) * npts);
    std::memcpy(y, c.ydos.data(), sizeof(double) * npts);
    *nev_est = c.nev_est;
  });
}

int ref_curve_from_moments(int m, const double* zeta, int n, double lmin, double lmax, int npts,
                           double* x, double* y, double* nev_est) {
  return guarded([&] {
    DosCurve c = curve_from_moments(Vec(zeta, zeta + m + 1), n, {lmin, lmax}, npts);
    std::memcpy(x, c.xdos.data(), sizeof(double) * npts);
    std::memcpy(y, c.ydos.data(), sizeof(double) * npts);
    *nev_est = c.nev_est;
  });
}

int ref_lan_dos(int n, const int* rp, const int* ci, const double* v, double lmin, double lmax,
                int m, int n_vec, int npts, double sigma, std::uint64_t seed, double* x, double* y,
                double* nev_est) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    DosConfig cfg;
    cfg.method = DosMethod::Lanczos;
    cfg.m = m;
    cfg.n_vec = n_vec;
    cfg.npts = npts;
    cfg.gaussian_sigma = sigma;
    cfg.seed = seed;
    DosCurve c = lan_dos(make_operator(a), {lmin, lmax}, cfg);
    std::memcpy(x, c.xdos.data(), sizeof(double) * npts);
    std::memcpy(y, c.ydos.data(), sizeof(double) * npts);
    *nev_est = c.nev_est;
  });
}

int ref_dos_count(int npts, int n, const double* x, const double* y, double xi, double eta,
                  double* out) {
  return guarded([&] {
    DosCurve c;
    c.n = n;
    c.xdos.assign(x, x + npts);
    c.ydos.assign(y, y + npts);
    *out = dos_count(c, xi, eta);
  });
}

int ref_slice_spectrum(int npts, int n, const double* x, const double* y, double xi, double eta,
                       int ns, double* bp, double* est) {
  return guarded([&] {
    DosCurve c;
    c.n = n;
    c.xdos.assign(x, x + npts);
    c.ydos.assign(y, y + npts);
    SliceSet s = slice_spectrum(c, xi, eta, ns);
    std::memcpy(bp, s.breakpoints.data(), sizeof(double) * (ns + 1));
    std::memcpy(est, s.est_counts.data(), sizeof(double) * ns);
  });
}

// ---- Krylov --------------------------------------------------------------------------------
int ref_lan_tr_bounds(int n, const int* rp, const int* ci, const double* v, double tol,
                      int restart, int max_restarts, std::uint64_t seed, double* lmin,
                      double* lmax) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    SpectralBounds b = lan_tr_bounds(make_operator(a), InnerProduct{}, tol, restart, max_restarts,
                                     (unsigned long)seed);
    *lmin = b.lmin;
    *lmax = b.lmax;
  });
}

// lanczos_run: alpha[m], beta[m-1]; returns steps/breakdown/next_beta.
int ref_lanczos_run(int n, const int* rp, const int* ci, const double* v, const double* start,
                    int m, double* alpha, double* beta, int* steps, int* breakdown,
                    double* next_beta, double* basis /* n x m col-major or null */) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    LanczosState st = lanczos_run(make_operator(a), InnerProduct{}, Vec(start, start + n), m);
    *steps = st.steps;
    *breakdown = st.breakdown;
    *next_beta = st.next_beta;
    std::memcpy(alpha, st.tri.alpha.data(), sizeof(double) * st.tri.alpha.size());
    if (!st.tri.beta.empty()) std::memcpy(beta, st.tri.beta.data(), sizeof(double) * st.tri.beta.size());
    if (basis)
      for (int j = 0; j < st.basis.cols(); ++j)
        std::memcpy(basis + (std::size_t)j * n, st.basis.col(j), sizeof(double) * n);
  });
}

int ref_paired_cgs2(int n, int k, const double* w, double* t, double* h) {
  return guarded([&] {
    DenseMat q(n, k);
    for (int j = 0; j < k; ++j) std::memcpy(q.col(j), w + (std::size_t)j * n, sizeof(double) * n);
    Vec tt(t, t + n);
    paired_cgs2(tt, q, q, k, h);
    std::memcpy(t, tt.data(), sizeof(double) * n);
  });
}

int ref_sym_tridiag_eig(int m, const double* alpha, const double* beta, int want, double* values,
                        double* vectors) {
  return guarded([&] {
    TriDiag t;
    t.alpha.assign(alpha, alpha + m);
    if (m > 1) t.beta.assign(beta, beta + m - 1);
    EigDecomp d = sym_tridiag_eig(t, want != 0);
    std::memcpy(values, d.values.data(), sizeof(double) * m);
    if (want)
      for (int j = 0; j < m; ++j)
        std::memcpy(vectors + (std::size_t)j * m, d.vectors.col(j), sizeof(double) * m);
  });
}

int ref_dense_sym_eig(int m, const double* a, int want, double* values, double* vectors) {
  return guarded([&] {
    DenseMat z(m, m);
    for (int j = 0; j < m; ++j) std::memcpy(z.col(j), a + (std::size_t)j * m, sizeof(double) * m);
    EigDecomp d = dense_sym_eig(DenseSym(z), want != 0);
    std::memcpy(values, d.values.data(), sizeof(double) * m);
    if (want)
      for (int j = 0; j < m; ++j)
        std::memcpy(vectors + (std::size_t)j * m, d.vectors.col(j), sizeof(double) * m);
  });
}

// ---- slice drivers -------------------------------------------------------------------------
// solver: 0 = cheb_lan_nr, 1 = cheb_lan_tr.  Filter built by find_pol(xi, eta, {lmin,lmax}).
// Returns an opaque ResultSet* (free with ref_results_free).
void* ref_cheb_lan(int n, const int* rp, const int* ci, const double* v, int solver, double xi,
                   double eta, double lmin, double lmax, int damping, int m, long max_its,
                   int ncycle, double tau1, double res_tol, int est_count, std::uint64_t seed) {
  auto* rs = new ResultSet();
  int rc = guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    PolyOpts po;
    po.damping = damping_of(damping);
    PolynomialFilter f = find_pol(xi, eta, SpectralBounds{lmin, lmax}, po);
    SolverConfig cfg;
    cfg.m = m;
    cfg.max_its = max_its;
    cfg.ncycle = ncycle;
    cfg.tau1 = tau1;
    cfg.res_tol = res_tol;
    cfg.est_count = est_count;
    cfg.seed = (unsigned long)seed;
    rs->degrees.push_back(f.k);
    rs->slices.push_back(solver == 2   ? cheb_si(a, nullptr, f, xi, eta, est_count, cfg)
                         : solver == 1 ? cheb_lan_tr(a, nullptr, f, xi, eta, cfg)
                                       : cheb_lan_nr(a, nullptr, f, xi, eta, cfg));
  });
  if (rc != 0) {
    delete rs;
    return nullptr;
  }
  return rs;
}

// Generalized pencil (A, B) with B = diag(bdiag): the reference's own B-weighted path
// (cheb_lan_nr/tr with b != nullptr: SpdFactor solves, eigensolvers.hpp:640-690, 703-732).
void* ref_cheb_lan_pencil(int n, const int* rp, const int* ci, const double* v, const double* bdiag,
                          int solver, double xi, double eta, double lmin, double lmax, int damping,
                          double res_tol, int est_count, std::uint64_t seed) {
  auto* rs = new ResultSet();
  int rc = guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    std::vector<Triplet> tb;
    for (int i = 0; i < n; ++i) tb.push_back({i, i, bdiag[i]});
    CsrMatrix b = CsrMatrix::from_triplets(n, std::move(tb));
    PolyOpts po;
    po.damping = damping_of(damping);
    PolynomialFilter f = find_pol(xi, eta, SpectralBounds{lmin, lmax}, po);
    SolverConfig cfg;
    cfg.res_tol = res_tol;
    cfg.est_count = est_count;
    cfg.seed = (unsigned long)seed;
    rs->degrees.push_back(f.k);
    rs->slices.push_back(solver == 2   ? cheb_si(a, &b, f, xi, eta, est_count, cfg)
                         : solver == 1 ? cheb_lan_tr(a, &b, f, xi, eta, cfg)
                                       : cheb_lan_nr(a, &b, f, xi, eta, cfg));
  });
  if (rc != 0) {
    delete rs;
    return nullptr;
  }
  return rs;
}

// ---- general SPD-B pencils (the reference's Cholesky-backed path) -----------------------------
// ls_pol_approx (cheb_approx.hpp:40-88): fun 0 = B^-1, 1 = B^-1/2; coefficients out (cap).
int ref_ls_pol_approx(int fun, double lmin, double lmax, double tol, int max_deg, int cap,
                      int* degree, double* coeff, double* achieved) {
  return guarded([&] {
    ChebApprox ap = ls_pol_approx(fun == 1 ? ScalarFun::InverseSqrt : ScalarFun::Inverse,
                                  SpectralBounds{lmin, lmax}, tol, max_deg);
    if (ap.degree() + 1 > cap) throw std::runtime_error("ref_ls_pol_approx: buffer too small");
    *degree = ap.degree();
    std::memcpy(coeff, ap.coeff.data(), sizeof(double) * ap.coeff.size());
    *achieved = ap.achieved_rel_error;
  });
}

// apply_cheb (cheb_approx.hpp:91-112) with the approximation given by its coefficients
int ref_apply_cheb(int n, const int* rp, const int* ci, const double* v, int fun, double lmin,
                   double lmax, int degree, const double* coeff, const double* x, double* y) {
  return guarded([&] {
    CsrMatrix b = make_csr(n, rp, ci, v);
    ChebApprox ap{fun == 1 ? ScalarFun::InverseSqrt : ScalarFun::Inverse, lmin, lmax,
                  Vec(coeff, coeff + degree + 1), 0.0};
    Vec out;
    apply_cheb(ap, make_operator(b), Vec(x, x + n), out);
    std::memcpy(y, out.data(), sizeof(double) * n);
  });
}

// Pencil (A, B) with a general sparse SPD B given in CSR: lan_tr_bounds in the B inner product
// (sliceeig_main.cpp:128-136), dos_generalized with Cholesky solves (:138-157), and one
// cheb_lan_nr/tr slice with b != nullptr (eigensolvers.hpp:640-732).
int ref_pencil_bounds(int n, const int* rp, const int* ci, const double* v, const int* brp,
                      const int* bci, const double* bv, std::uint64_t seed, double* lmin,
                      double* lmax) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v), b = make_csr(n, brp, bci, bv);
    Operator opa = make_operator(a), opb = make_operator(b);
    SpdFactor bf = SpdFactor::factor(b);
    Operator bsolve{n, [&](const Vec& x, Vec& y) { y = bf.solve(x); }};
    InnerProduct ip{&opb, &bsolve};
    SpectralBounds r = lan_tr_bounds(opa, ip, 1e-4, 60, 40, (unsigned long)seed);
    *lmin = r.lmin;
    *lmax = r.lmax;
  });
}

int ref_pencil_dos(int n, const int* rp, const int* ci, const double* v, const int* brp,
                   const int* bci, const double* bv, double lmin, double lmax, int m, int n_vec,
                   int npts, std::uint64_t seed, double* x, double* y, double* nev_est) {
  return guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v), b = make_csr(n, brp, bci, bv);
    Operator opa = make_operator(a), opb = make_operator(b);
    SpdFactor bf = SpdFactor::factor(b);
    Operator bsolve{n, [&](const Vec& xx, Vec& yy) { yy = bf.solve(xx); }};
    Operator bhalf{n, [&](const Vec& xx, Vec& yy) { yy = bf.solve_gt(xx); }};
    DosConfig cfg;
    cfg.method = DosMethod::Lanczos;
    cfg.m = m;
    cfg.n_vec = n_vec;
    cfg.npts = npts;
    cfg.seed = seed;
    DosCurve c = dos_generalized(opa, bsolve, bhalf, opb, {lmin, lmax}, cfg);
    std::memcpy(x, c.xdos.data(), sizeof(double) * npts);
    std::memcpy(y, c.ydos.data(), sizeof(double) * npts);
    *nev_est = c.nev_est;
  });
}

void* ref_cheb_lan_pencil_csr(int n, const int* rp, const int* ci, const double* v,
                              const int* brp, const int* bci, const double* bv, int solver,
                              double xi, double eta, double lmin, double lmax, int damping,
                              double res_tol, int est_count, std::uint64_t seed) {
  auto* rs = new ResultSet();
  int rc = guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v), b = make_csr(n, brp, bci, bv);
    PolyOpts po;
    po.damping = damping_of(damping);
    PolynomialFilter f = find_pol(xi, eta, SpectralBounds{lmin, lmax}, po);
    SolverConfig cfg;
    cfg.res_tol = res_tol;
    cfg.est_count = est_count;
    cfg.seed = (unsigned long)seed;
    rs->degrees.push_back(f.k);
    rs->slices.push_back(solver == 2   ? cheb_si(a, &b, f, xi, eta, est_count, cfg)
                         : solver == 1 ? cheb_lan_tr(a, &b, f, xi, eta, cfg)
                                       : cheb_lan_nr(a, &b, f, xi, eta, cfg));
  });
  if (rc != 0) {
    delete rs;
    return nullptr;
  }
  return rs;
}

// Full sliced solve mirroring `sliceeig solve` (tools/sliceeig_main.cpp:464-523):
// bounds (lan_tr_bounds tol 1e-4, 60, 40, seed :128-136) -> DOS (:138-157) -> slice_clipped
// (:270-278) -> per-slice find_pol + cheb_lan_nr/tr (:394-418) on a std::thread pool
// (:494-523) -> trim_to_slice with delta = 1e-10*(lmax-lmin) (:422-442, :497).
// probe_kind 1 swaps the KPM probes to Gaussian (BASELINE cfg2); 0 calls kpm_dos unchanged.
// lmin/lmax: if lmin < lmax on entry they are used as fixed bounds (bounds stage skipped).
void* ref_solve(int n, const int* rp, const int* ci, const double* v, double xi, double eta,
                int ns, int solver, int damping, int dos_m, int dos_nvec, int dos_npts,
                int probe_kind, double tol, std::uint64_t seed, int jobs, double fixed_lmin,
                double fixed_lmax) {
  auto* rs = new ResultSet();
  const auto t_start = std::chrono::steady_clock::now();
  int rc = guarded([&] {
    CsrMatrix a = make_csr(n, rp, ci, v);
    Operator opa = make_operator(a);
    auto t0 = std::chrono::steady_clock::now();
    SpectralBounds bounds{fixed_lmin, fixed_lmax};
    if (!(fixed_lmin < fixed_lmax))
      bounds = lan_tr_bounds(opa, InnerProduct{}, 1e-4, 60, 40, (unsigned long)seed);
    rs->t_bounds = secs(t0);
    rs->lmin = bounds.lmin;
    rs->lmax = bounds.lmax;

    t0 = std::chrono::steady_clock::now();
    DosCurve curve;
    if (probe_kind == 0) {
      DosConfig cfg;
      cfg.m = dos_m;
      cfg.n_vec = dos_nvec;
      cfg.npts = dos_npts;
      cfg.seed = seed;
      curve = kpm_dos(opa, bounds, cfg);
    } else {
      Vec z = kpm_moments(opa, bounds, dos_m, dos_nvec, seed, probe_kind, 0, dos_nvec);
      for (double& q : z) q /= (double)dos_nvec * n;
      curve = curve_from_moments(z, n, bounds, dos_npts);
    }
    struct Task {
      int index;
      double lo, hi, est;
    };
    std::vector<Task> tasks;
    const double clo = std::max(xi, curve.xdos.front()), chi = std::min(eta, curve.xdos.back());
    if (ns <= 1) {
      tasks.push_back({0, xi, eta, clo < chi ? dos_count(curve, clo, chi) : 0.0});
    } else {
      if (!(clo < chi))
        throw std::invalid_argument("requested interval does not meet the sampled spectrum");
      SliceSet s = slice_spectrum(curve, clo, chi, ns);
      s.breakpoints.front() = xi;
      s.breakpoints.back() = eta;
      for (int i = 0; i < s.ns(); ++i)
        tasks.push_back({i, s.breakpoints[i], s.breakpoints[i + 1], s.est_counts[i]});
    }
    rs->t_dos = secs(t0);
    for (auto& t : tasks) rs->est.push_back(t.est);
    rs->breakpoints.push_back(tasks.front().lo);
    for (auto& t : tasks) rs->breakpoints.push_back(t.hi);

    const int nt = (int)tasks.size();
    const double delta = 1e-10 * (bounds.lmax - bounds.lmin);
    rs->slices.resize(nt);
    rs->degrees.assign(nt, 0);
    rs->errors.assign(nt, "");
    std::atomic<int> cursor{0};
    auto worker = [&]() {
      for (;;) {
        const int i = cursor.fetch_add(1);
        if (i >= nt) return;
        try {
          const Task& t = tasks[i];
          SolverConfig cfg;
          cfg.res_tol = tol;
          cfg.seed = (unsigned long)seed;
          cfg.est_count = std::max(1, (int)std::lround(std::ceil(t.est)));
          PolyOpts po;
          po.damping = damping_of(damping);
          PolynomialFilter f = find_pol(t.lo, t.hi, bounds, po);
          rs->degrees[i] = f.k;
          EigenResults r = solver == 2   ? cheb_si(a, nullptr, f, t.lo, t.hi, cfg.est_count, cfg)
                           : solver == 1 ? cheb_lan_tr(a, nullptr, f, t.lo, t.hi, cfg)
                                       : cheb_lan_nr(a, nullptr, f, t.lo, t.hi, cfg);
          // trim_to_slice (sliceeig_main.cpp:422-442)
          EigenResults out;
          out.niter = r.niter;
          out.counters = r.counters;
          out.hit_max_its = r.hit_max_its;
          out.vectors = DenseMat(r.vectors.rows(), 0);
          for (int q = 0; q < (int)r.eigenvalues.size(); ++q) {
            const double lam = r.eigenvalues[q];
            if (t.index > 0 && lam <= t.lo + delta) continue;
            if (t.index + 1 < nt && lam > t.hi + delta) continue;
            out.eigenvalues.push_back(lam);
            out.residuals.push_back(r.residuals[q]);
          }
          rs->slices[i] = std::move(out);
        } catch (const std::exception& e) {
          rs->errors[i] = e.what();
        }
      }
    };
    t0 = std::chrono::steady_clock::now();
    const int nj = std::max(1, std::min(jobs, nt));
    if (nj == 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < nj; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
    }
    rs->t_solve = secs(t0);
  });
  rs->t_total = secs(t_start);
  if (rc != 0) {
    delete rs;
    return nullptr;
  }
  return rs;
}

int ref_results_nslices(void* h) { return (int)static_cast<ResultSet*>(h)->slices.size(); }

// Per-slice scalars: count, niter, n_A_matvec, hit_max_its, degree; times t_mv,t_orth,t_total.
int ref_results_slice(void* h, int s, int* count, long* niter, long* nmv, int* hit, int* degree,
                      double* times3) {
  auto* rs = static_cast<ResultSet*>(h);
  if (s < 0 || s >= (int)rs->slices.size()) return -1;
  const EigenResults& r = rs->slices[s];
  *count = (int)r.eigenvalues.size();
  *niter = r.niter;
  *nmv = r.counters.n_A_matvec;
  *hit = r.hit_max_its;
  *degree = rs->degrees[s];
  times3[0] = r.counters.t_mv;
  times3[1] = r.counters.t_orth;
  times3[2] = r.counters.t_total;
  if (!rs->errors.empty() && !rs->errors[s].empty()) {
    g_err = rs->errors[s];
    return -2;
  }
  return 0;
}

int ref_results_values(void* h, int s, double* vals, double* res, double* vecs) {
  auto* rs = static_cast<ResultSet*>(h);
  const EigenResults& r = rs->slices[s];
  std::memcpy(vals, r.eigenvalues.data(), sizeof(double) * r.eigenvalues.size());
  std::memcpy(res, r.residuals.data(), sizeof(double) * r.residuals.size());
  if (vecs)
    for (int j = 0; j < r.vectors.cols(); ++j)
      std::memcpy(vecs + (std::size_t)j * r.vectors.rows(), r.vectors.col(j),
                  sizeof(double) * r.vectors.rows());
  return 0;
}

// Pipeline-level scalars: lmin, lmax, t_bounds, t_dos, t_solve, t_total; breakpoints[ns+1], est[ns].
int ref_results_pipeline(void* h, double* scalars6, double* bp, double* est) {
  auto* rs = static_cast<ResultSet*>(h);
  scalars6[0] = rs->lmin;
  scalars6[1] = rs->lmax;
  scalars6[2] = rs->t_bounds;
  scalars6[3] = rs->t_dos;
  scalars6[4] = rs->t_solve;
  scalars6[5] = rs->t_total;
  if (bp) std::memcpy(bp, rs->breakpoints.data(), sizeof(double) * rs->breakpoints.size());
  if (est) std::memcpy(est, rs->est.data(), sizeof(double) * rs->est.size());
  return 0;
}

void ref_results_free(void* h) { delete static_cast<ResultSet*>(h); }

}  // extern "C"
