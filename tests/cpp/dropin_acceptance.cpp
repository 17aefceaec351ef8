// Drop-in check of the C++ facade: code written against the reference's sliceeig API (the calls of
// tools/sliceeig_main.cpp:128-157,394-418 and the polynomial parts of acceptance.cpp criteria 1, 3,
// 4, 9) compiles unchanged against include/sliceeig/*.hpp and runs on the GPU.
// Prints one PASS/FAIL line per check; exit status 0 iff all pass.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "sliceeig/dos.hpp"
#include "sliceeig/eigensolvers.hpp"
#include "sliceeig/filter_poly.hpp"
#include "sliceeig/laplacian.hpp"
#include "sliceeig/slicer.hpp"

using namespace sliceeig;

static int failures = 0;
static void expect(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

int main() {
  // criterion 1 (polynomial drivers) on a 2-D grid window
  {
    CsrMatrix a = gen_laplacian({60, 60});
    Vec all = laplacian_analytic_eigs({60, 60});
    Vec oracle;
    for (double v : all)
      if (v >= 0.4 && v <= 0.6) oracle.push_back(v);
    SpectralBounds bb = lan_tr_bounds(make_operator(a), InnerProduct{}, 1e-4, 60, 40, 1234);
    PolynomialFilter pf = find_pol(0.4, 0.6, bb);
    SolverConfig cfg;
    cfg.est_count = (int)oracle.size();
    for (int drv = 0; drv < 2; ++drv) {
      EigenResults r = drv ? cheb_lan_tr(a, nullptr, pf, 0.4, 0.6, cfg) : cheb_lan_nr(a, nullptr, pf, 0.4, 0.6, cfg);
      bool ok = r.eigenvalues.size() == oracle.size();
      double err = 0.0, res = 0.0;
      for (std::size_t i = 0; ok && i < oracle.size(); ++i) {
        err = std::max(err, std::abs(r.eigenvalues[i] - oracle[i]));
        res = std::max(res, rayleigh_and_residual(a, nullptr, r.vectors.col_vec((int)i)).second);
      }
      expect(ok && err <= 1e-8 && res <= 1e-8,
             std::string(drv ? "cheb_lan_tr" : "cheb_lan_nr") + " 60x60 [0.4,0.6]: " +
                 std::to_string(r.eigenvalues.size()) + "/" + std::to_string(oracle.size()));
      expect(r.counters.n_A_matvec >= (long)pf.k * r.niter, "op accounting n_A_matvec >= k*niter");
    }
  }
  // generalized pencil (A, B) with a diagonal SPD B (lumped mass): reference-style call with
  // b != nullptr; B-normalised vectors and pencil residuals ||Ax - lambda Bx||
  {
    CsrMatrix a = gen_laplacian({12, 12, 12});
    Vec bd((std::size_t)a.n());
    for (int i = 0; i < a.n(); ++i) bd[i] = 0.5 + 0.25 * (1.0 + std::sin(0.37 * i));
    CsrMatrix b = CsrMatrix::diag(bd);
    PolynomialFilter pf = find_pol(1.0, 1.3, SpectralBounds{0.0, 24.0});
    SolverConfig cfg;
    cfg.est_count = 40;
    EigenResults r = cheb_lan_tr(a, &b, pf, 1.0, 1.3, cfg);
    double res = 0.0, nrm = 0.0;
    for (int j = 0; j < (int)r.eigenvalues.size(); ++j) {
      const Vec x = r.vectors.col_vec(j);
      const auto rr = rayleigh_and_residual(a, &b, x);
      res = std::max(res, rr.second / std::max(1.0, std::abs(rr.first)));
      double xbx = 0.0;
      for (int i = 0; i < a.n(); ++i) xbx += x[i] * bd[i] * x[i];
      nrm = std::max(nrm, std::abs(xbx - 1.0));
    }
    expect(!r.eigenvalues.empty() && res <= 1e-8 && nrm <= 1e-12,
           "cheb_lan_tr pencil (A, diag B) 12^3 [1.0,1.3]: " + std::to_string(r.eigenvalues.size()) +
               " pairs, max ||Ax-lBx|| " + std::to_string(res));
  }
  // criterion 3 (slicing + seam-exact union) on 20^3 through the CLI's stage calls
  {
    CsrMatrix a = gen_laplacian({20, 20, 20});
    Operator opa = make_operator(a);
    SpectralBounds b = lan_tr_bounds(opa, InnerProduct{}, 1e-4, 60, 40, 7);
    DosConfig dc;
    dc.seed = 7;
    DosCurve curve = kpm_dos(opa, b, dc);
    SliceSet s = slice_spectrum(curve, 0.5, 2.0, 3);
    Vec all = laplacian_analytic_eigs({20, 20, 20});
    const double delta = 1e-10 * (b.lmax - b.lmin);
    long found = 0;
    for (int i = 0; i < s.ns(); ++i) {
      SolverConfig cfg;
      cfg.seed = 7;
      cfg.est_count = std::max(1, (int)std::lround(std::ceil(s.est_counts[i])));
      PolynomialFilter f = find_pol(s.breakpoints[i], s.breakpoints[i + 1], b);
      EigenResults r = cheb_lan_tr(a, nullptr, f, s.breakpoints[i], s.breakpoints[i + 1], cfg);
      for (double v : r.eigenvalues) {
        if (i > 0 && v <= s.breakpoints[i] + delta) continue;
        if (i + 1 < s.ns() && v > s.breakpoints[i + 1] + delta) continue;
        ++found;
      }
    }
    expect(found == count_in_interval(all, 0.5, 2.0),
           "20^3 [0.5,2] in 3 slices: union " + std::to_string(found) + " of " +
               std::to_string(count_in_interval(all, 0.5, 2.0)));
  }
  // criterion 4 (filter invariants)
  {
    PolynomialFilter f = find_pol(0.2, 0.4, SpectralBounds{-1.0, 1.0});
    expect(std::abs(eval_pol(f, f.gamma) - 1.0) <= 1e-14, "rho(gamma) = 1");
    expect(std::abs(eval_pol(f, f.ta) - eval_pol(f, f.tb)) <= 1e-10, "balanced endpoints");
    bool threw = false;
    try {
      find_pol(0.5, 0.5, SpectralBounds{0.0, 8.0});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    expect(threw, "find_pol degenerate interval -> std::invalid_argument");
    CsrMatrix d = CsrMatrix::diag({0.5, 1.5, 2.5, 3.5});
    Vec v(4, 1.0), out;
    Counters cnt;
    PolynomialFilter g = find_pol(1.0, 2.0, SpectralBounds{0.0, 4.0});
    apply_pol(g, make_operator(d), v, out, &cnt);
    double e = 0.0;
    for (int i = 0; i < 4; ++i) e = std::max(e, std::abs(out[i] - eval_pol(g, g.map.to_ref(0.5 + i))));
    expect(e <= 1e-12 && cnt.n_A_matvec == g.k, "apply_pol on a diagonal = pointwise rho");
  }
  // criterion 9 (DOS normalisation + bitwise rerun)
  {
    CsrMatrix a = gen_laplacian({20, 20});
    Operator op = make_operator(a);
    DosCurve c1 = kpm_dos(op, SpectralBounds{0.0, 8.0});
    DosCurve c2 = kpm_dos(op, SpectralBounds{0.0, 8.0});
    expect(c1.ydos == c2.ydos, "kpm_dos bitwise rerun");
    expect(std::abs(dos_count(c1, 0.0, 8.0) - a.n()) <= 1e-6 * a.n(), "kpm_dos unit mass");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}
