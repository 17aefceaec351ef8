// C++ drop-in facade for the polynomial-filtering path of sliceeig (namespace sliceeig), backed by
// libsliceeig_cuda.so through the C ABI of sliceeig_cuda.h.  Names, types and signatures follow
// the reference headers /root/reference/proj/include/sliceeig/*.hpp for the in-scope API
// (SURVEY.md §8b): matrix setup, kpm_dos/lan_dos, slice_spectrum, find_pol/apply_pol,
// lanczos_run/lan_tr_bounds, cheb_lan_nr/cheb_lan_tr.  Callers compile unchanged; link with
// -lsliceeig_cuda.  O(n) work runs on the GPU; there is no host fallback.
//
// Differences a caller can observe: Operator carries the CsrMatrix it wraps (make_operator sets
// it; matrix-free lambdas are rejected by the device drivers with std::invalid_argument), and
// generalized pencils (b != nullptr) are outside the device path (std::invalid_argument).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "sliceeig_cuda.h"

namespace sliceeig {

using Vec = std::vector<double>;
inline constexpr double kPi = 3.14159265358979323846;

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string msg = se_last_error();
  if (rc == SE_EINVAL) throw std::invalid_argument(msg);
  if (rc == SE_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
inline void ok(int rc) {
  if (rc != SE_OK) raise(rc);
}
// One context per host thread (one CUDA stream + library handles), on the device chosen by
// set_thread_device() before the thread's first call, else SLICEEIG_DEVICE, else 0.
inline int& thread_device() {
  thread_local int d = -1;
  return d;
}
struct ThreadCtx {
  se_ctx* c = nullptr;
  ThreadCtx() {
    int dev = thread_device();
    if (dev < 0) {
      const char* d = std::getenv("SLICEEIG_DEVICE");
      dev = d ? std::atoi(d) : 0;
    }
    ok(se_ctx_create(dev, &c));
  }
  ~ThreadCtx() { se_ctx_destroy(c); }
};
inline se_ctx* ctx() {
  thread_local ThreadCtx t;
  return t.c;
}
}  // namespace detail

// B200 extension: pin the calling host thread to a GPU (before its first library call); the
// CLI's slice pool uses it to spread slices over the GPUs of a node.
inline void set_thread_device(int device) { detail::thread_device() = device; }

// ---- vecops.hpp ----------------------------------------------------------------------------
inline double dot(const Vec& x, const Vec& y) {
  double s = 0.0;
  for (std::size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
  return s;
}
inline double nrm2(const Vec& x) { return std::sqrt(dot(x, x)); }
inline void axpy(double a, const Vec& x, Vec& y) {
  for (std::size_t i = 0; i < x.size(); ++i) y[i] += a * x[i];
}
inline void scal(double a, Vec& x) {
  for (auto& v : x) v *= a;
}

class DenseMat {  // column-major
 public:
  DenseMat() = default;
  DenseMat(int rows, int cols) : rows_(rows), cols_(cols), a_((std::size_t)rows * cols, 0.0) {}
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  double& operator()(int i, int j) { return a_[(std::size_t)j * rows_ + i]; }
  double operator()(int i, int j) const { return a_[(std::size_t)j * rows_ + i]; }
  double* col(int j) { return a_.data() + (std::size_t)j * rows_; }
  const double* col(int j) const { return a_.data() + (std::size_t)j * rows_; }
  Vec col_vec(int j) const { return Vec(col(j), col(j) + rows_); }
  void col_copy(int j, const Vec& v) { std::copy(v.begin(), v.end(), col(j)); }
  void push_col(const Vec& v) {
    if (rows_ == 0) rows_ = (int)v.size();
    a_.insert(a_.end(), v.begin(), v.end());
    ++cols_;
  }
  void mult_cols(int k, const double* x, Vec& y) const {
    y.assign(rows_, 0.0);
    for (int j = 0; j < k; ++j)
      if (x[j] != 0.0)
        for (int i = 0; i < rows_; ++i) y[i] += x[j] * col(j)[i];
  }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }

 private:
  int rows_ = 0, cols_ = 0;
  Vec a_;
};

// ---- rng.hpp (mt19937_64 streams fixed by the C++ standard) ---------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : g_(seed) {}
  double uniform() { return double(g_() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have_) {
      have_ = false;
      return spare_;
    }
    double u1;
    do {
      u1 = uniform();
    } while (u1 <= 0.0);
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1)), t = 2.0 * kPi * u2;
    spare_ = r * std::sin(t);
    have_ = true;
    return r * std::cos(t);
  }
  double rademacher() { return (g_() & 1u) ? 1.0 : -1.0; }
  Vec normal_vec(int n) {
    Vec v(n);
    for (auto& x : v) x = normal();
    return v;
  }
  Vec rademacher_vec(int n) {
    Vec v(n);
    for (auto& x : v) x = rademacher();
    return v;
  }
  std::uint64_t raw() { return g_(); }

 private:
  std::mt19937_64 g_;
  bool have_ = false;
  double spare_ = 0.0;
};

// ---- csr.hpp ----------------------------------------------------------------------------------
struct Triplet {
  int row = 0, col = 0;
  double val = 0.0;
};

class CsrMatrix {
 public:
  CsrMatrix() = default;
  static CsrMatrix from_triplets(int n, std::vector<Triplet> t) {
    if (n < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
    for (const auto& e : t)
      if (e.row < 0 || e.row >= n || e.col < 0 || e.col >= n)
        throw std::out_of_range("CsrMatrix: triplet index out of range");
    std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    CsrMatrix m;
    m.n_ = n;
    m.rp_.assign(n + 1, 0);
    for (std::size_t i = 0; i < t.size();) {
      std::size_t j = i + 1;
      double v = t[i].val;
      while (j < t.size() && t[j].row == t[i].row && t[j].col == t[i].col) v += t[j++].val;
      if (v != 0.0) {
        m.ci_.push_back(t[i].col);
        m.v_.push_back(v);
        ++m.rp_[t[i].row + 1];
      }
      i = j;
    }
    for (int r = 0; r < n; ++r) m.rp_[r + 1] += m.rp_[r];
    return m;
  }
  static CsrMatrix from_csr(int n, std::vector<int> rp, std::vector<int> ci, Vec v) {
    CsrMatrix m;
    m.n_ = n;
    m.rp_ = std::move(rp);
    m.ci_ = std::move(ci);
    m.v_ = std::move(v);
    return m;
  }
  static CsrMatrix identity(int n) {
    std::vector<Triplet> t;
    for (int i = 0; i < n; ++i) t.push_back({i, i, 1.0});
    return from_triplets(n, std::move(t));
  }
  static CsrMatrix tridiag_toeplitz(int n, double e, double d) {
    std::vector<Triplet> t;
    for (int i = 0; i < n; ++i) {
      if (i > 0) t.push_back({i, i - 1, e});
      t.push_back({i, i, d});
      if (i < n - 1) t.push_back({i, i + 1, e});
    }
    return from_triplets(n, std::move(t));
  }
  static CsrMatrix diag(const Vec& d) {
    std::vector<Triplet> t;
    for (int i = 0; i < (int)d.size(); ++i) t.push_back({i, i, d[i]});
    return from_triplets((int)d.size(), std::move(t));
  }
  int n() const { return n_; }
  int nnz() const { return (int)v_.size(); }
  const std::vector<int>& row_ptr() const { return rp_; }
  const std::vector<int>& col_idx() const { return ci_; }
  const std::vector<double>& vals() const { return v_; }
  double coeff(int i, int j) const {
    for (int k = rp_[i]; k < rp_[i + 1]; ++k)
      if (ci_[k] == j) return v_[k];
    return 0.0;
  }
  // y = A x on the GPU (bit-identical to the reference's row loop, csr.hpp:98-105).
  void matvec(const Vec& x, Vec& y) const {
    y.assign(n_, 0.0);
    if (n_) detail::ok(se_spmv(detail::ctx(), device(), x.data(), y.data()));
  }
  Vec matvec(const Vec& x) const {
    Vec y;
    matvec(x, y);
    return y;
  }
  bool is_symmetric(double tol = 1e-14) const {
    for (int i = 0; i < n_; ++i)
      for (int k = rp_[i]; k < rp_[i + 1]; ++k) {
        const double aij = v_[k], aji = coeff(ci_[k], i);
        if (std::abs(aij - aji) > tol * std::max(1.0, std::abs(aij))) return false;
      }
    return true;
  }
  double one_norm() const {
    Vec colsum(n_, 0.0);
    for (int i = 0; i < n_; ++i)
      for (int k = rp_[i]; k < rp_[i + 1]; ++k) colsum[ci_[k]] += std::abs(v_[k]);
    double m = 0.0;
    for (double s : colsum) m = std::max(m, s);
    return m;
  }
  std::vector<Triplet> to_triplets() const {
    std::vector<Triplet> t;
    t.reserve(v_.size());
    for (int i = 0; i < n_; ++i)
      for (int k = rp_[i]; k < rp_[i + 1]; ++k) t.push_back({i, ci_[k], v_[k]});
    return t;
  }
  // Device copy for the calling thread's context (uploaded once per context and cached; safe
  // for concurrent use by several threads, each with its own context).
  se_csr* device() const {
    se_ctx* c = detail::ctx();
    std::lock_guard<std::mutex> lk(dev_->mu);
    for (const auto& e : dev_->copies)
      if (e.first == c) return e.second.get();
    se_csr* h = nullptr;
    detail::ok(se_csr_upload(c, n_, rp_.data(), ci_.data(), v_.data(), &h));
    dev_->copies.emplace_back(c, std::shared_ptr<se_csr>(h, [](se_csr* p) { se_csr_free(p); }));
    return h;
  }

 private:
  struct DevCopies {
    std::mutex mu;
    std::vector<std::pair<se_ctx*, std::shared_ptr<se_csr>>> copies;
  };
  int n_ = 0;
  std::vector<int> rp_{0};
  std::vector<int> ci_;
  Vec v_;
  std::shared_ptr<DevCopies> dev_ = std::make_shared<DevCopies>();
};

// ---- laplacian.hpp ------------------------------------------------------------------------------
inline CsrMatrix gen_laplacian(const std::vector<int>& dims) {
  int n = 0;
  long nnz = 0;
  detail::ok(se_laplacian_host((int)dims.size(), dims.data(), &n, &nnz, nullptr, nullptr, nullptr));
  std::vector<int> rp(n + 1), ci(nnz);
  Vec v(nnz);
  detail::ok(se_laplacian_host((int)dims.size(), dims.data(), &n, &nnz, rp.data(), ci.data(), v.data()));
  return CsrMatrix::from_csr(n, std::move(rp), std::move(ci), std::move(v));
}
inline Vec laplacian_analytic_eigs(const std::vector<int>& dims) {
  long n = 1;
  for (int d : dims) n *= std::max(d, 0);
  Vec e(dims.empty() ? 0 : n);
  detail::ok(se_laplacian_eigs((int)dims.size(), dims.data(), e.data()));
  return e;
}
inline long count_in_interval(const Vec& s, double lo, double hi) {
  return (long)(std::upper_bound(s.begin(), s.end(), hi) - std::lower_bound(s.begin(), s.end(), lo));
}

// ---- operators.hpp --------------------------------------------------------------------------------
struct Operator {
  int n = 0;
  std::function<void(const Vec&, Vec&)> apply;
  const CsrMatrix* csr = nullptr;  // set by make_operator: the device drivers consume this
  Vec operator()(const Vec& x) const {
    Vec y;
    apply(x, y);
    return y;
  }
};
inline Operator make_operator(const CsrMatrix& a) {
  return Operator{a.n(), [&a](const Vec& x, Vec& y) { a.matvec(x, y); }, &a};
}
struct Counters {
  long n_A_matvec = 0, n_B_matvec = 0, n_B_solve = 0, n_shift_solve = 0;
  double t_mv = 0.0, t_orth = 0.0, t_sv = 0.0, t_total = 0.0;
  Counters& operator+=(const Counters& o) {
    n_A_matvec += o.n_A_matvec;
    n_B_matvec += o.n_B_matvec;
    n_B_solve += o.n_B_solve;
    n_shift_solve += o.n_shift_solve;
    t_mv += o.t_mv;
    t_orth += o.t_orth;
    t_sv += o.t_sv;
    t_total += o.t_total;
    return *this;
  }
};
struct InnerProduct {
  const Operator* b = nullptr;
  const Operator* b_solve = nullptr;
  bool euclidean() const { return b == nullptr; }
};

namespace detail {
inline se_csr* dev_of(const Operator& op, const char* who) {
  if (!op.csr)
    throw std::invalid_argument(std::string(who) +
                                ": the device path needs a CSR-backed operator (make_operator)");
  return op.csr->device();
}
inline void euclid_only(const InnerProduct& ip, const char* who) {
  if (!ip.euclidean())
    throw std::invalid_argument(std::string(who) + ": B-weighted runs need the CSR-backed B of a "
                                "pencil (lan_tr_bounds / dos_generalized)");
}
// The device pencil of an InnerProduct whose B is a CSR-backed operator (make_operator(B)); the
// b_solve operator is not needed (B-solves become B-products of the B^-1/2 series).
inline se_pencil* pencil_for(const InnerProduct& ip, const char* who) {
  if (!ip.b || !ip.b->csr)
    throw std::invalid_argument(std::string(who) + ": the device path needs a CSR-backed B (make_operator)");
  se_pencil* pen = nullptr;
  ok(se_pencil_create(ctx(), ip.b->csr->device(), 0.0, 0, &pen));
  return pen;
}
}  // namespace detail

// ---- tridiag_eig.hpp / dense_eig.hpp -----------------------------------------------------------------
struct TriDiag {
  Vec alpha, beta;
};
struct EigDecomp {
  Vec values;
  DenseMat vectors;
  bool have_vectors = false;
};
inline EigDecomp sym_tridiag_eig(const TriDiag& t, bool want_vectors) {
  const int m = (int)t.alpha.size();
  if (m > 0 && (int)t.beta.size() != m - 1)
    throw std::invalid_argument("sym_tridiag_eig: beta must have length m-1");
  EigDecomp d;
  d.values.resize(m);
  if (want_vectors) d.vectors = DenseMat(m, m);
  detail::ok(se_sym_tridiag_eig(m, t.alpha.data(), t.beta.data(), want_vectors, d.values.data(),
                                want_vectors ? d.vectors.data() : nullptr));
  d.have_vectors = want_vectors;
  return d;
}
class DenseSym {
 public:
  DenseSym() = default;
  explicit DenseSym(int n) : a_(n, n) {}
  explicit DenseSym(const DenseMat& m) : a_(m) {
    if (m.rows() != m.cols()) throw std::invalid_argument("DenseSym: not square");
  }
  int n() const { return a_.rows(); }
  double operator()(int i, int j) const { return a_(i, j); }
  void set(int i, int j, double v) {
    a_(i, j) = v;
    a_(j, i) = v;
  }
  const DenseMat& mat() const { return a_; }

 private:
  DenseMat a_;
};
inline EigDecomp dense_sym_eig(const DenseSym& a, bool want_vectors, int size_guard = 5000) {
  const int m = a.n();
  EigDecomp d;
  d.values.resize(m);
  if (want_vectors) d.vectors = DenseMat(m, m);
  detail::ok(se_dense_sym_eig(m, a.mat().data(), want_vectors, size_guard, d.values.data(),
                              want_vectors ? d.vectors.data() : nullptr));
  d.have_vectors = want_vectors;
  return d;
}

// ---- orth.hpp ------------------------------------------------------------------------------------------
inline void paired_cgs2(Vec& t, const DenseMat& dotside, const DenseMat& subside, int k,
                        double* h = nullptr) {
  if (&dotside != &subside)
    throw std::invalid_argument("paired_cgs2: paired (B-weighted) bases are outside the device path");
  if (k == 0) return;
  detail::ok(se_paired_cgs2(detail::ctx(), (int)t.size(), k, dotside.data(), t.data(), h));
}

// ---- lanczos.hpp -------------------------------------------------------------------------------------------
struct SpectralBounds {
  double lmin = 0.0, lmax = 0.0;
};
struct LanczosState {
  DenseMat basis;
  TriDiag tri;
  double next_beta = 0.0;
  Vec next_w;
  bool breakdown = false;
  int steps = 0;
};
inline LanczosState lanczos_run(const Operator& op, const InnerProduct& ip, Vec start, int m) {
  detail::euclid_only(ip, "lanczos_run");
  if ((int)start.size() != op.n) throw std::invalid_argument("lanczos_run: bad start vector size");
  const int mm = std::min(m, op.n);
  LanczosState st;
  Vec alpha(std::max(mm, 1)), beta(std::max(mm, 1)), nw(op.n);
  DenseMat basis(op.n, std::max(mm, 1));
  int steps = 0, brk = 0;
  detail::ok(se_lanczos_run(detail::ctx(), detail::dev_of(op, "lanczos_run"), start.data(), m,
                            alpha.data(), beta.data(), &steps, &brk, &st.next_beta, nw.data(),
                            basis.data()));
  st.steps = steps;
  st.breakdown = brk != 0;
  st.tri.alpha.assign(alpha.begin(), alpha.begin() + steps);
  st.tri.beta.assign(beta.begin(), beta.begin() + std::max(steps - 1, 0));
  if (!st.breakdown) st.next_w = nw;
  st.basis = DenseMat(op.n, 0);
  for (int j = 0; j < steps; ++j) st.basis.push_col(basis.col_vec(j));
  return st;
}
inline SpectralBounds lan_tr_bounds(const Operator& op, const InnerProduct& ip, double tol,
                                    int restart_dim, int max_restarts = 40,
                                    unsigned long seed = 1234) {
  if (!ip.euclidean()) {  // B inner product (sliceeig_main.cpp:128-136): the device pencil
    se_pencil* pen = detail::pencil_for(ip, "lan_tr_bounds");
    SpectralBounds b;
    const int rc = se_lan_tr_bounds_pencil(detail::ctx(), detail::dev_of(op, "lan_tr_bounds"), pen,
                                           tol, restart_dim, max_restarts, seed, &b.lmin, &b.lmax);
    se_pencil_free(pen);
    detail::ok(rc);
    return b;
  }
  SpectralBounds b;
  detail::ok(se_lan_tr_bounds(detail::ctx(), detail::dev_of(op, "lan_tr_bounds"), tol, restart_dim,
                              max_restarts, seed, &b.lmin, &b.lmax));
  return b;
}

// ---- cheb_approx.hpp -------------------------------------------------------------------------------
enum class ScalarFun { Inverse, InverseSqrt };
struct ChebApprox {
  ScalarFun fun = ScalarFun::Inverse;
  double lmin = 0.0, lmax = 0.0;
  Vec coeff;
  double achieved_rel_error = 0.0;
  int degree() const { return (int)coeff.size() - 1; }
  double eval(double t) const {  // Clenshaw on the mapped argument
    const double c = 0.5 * (lmax + lmin), h = 0.5 * (lmax - lmin);
    const double x = (t - c) / h;
    double b1 = 0.0, b2 = 0.0;
    for (int j = (int)coeff.size() - 1; j >= 1; --j) {
      const double b0 = 2.0 * x * b1 - b2 + coeff[j];
      b2 = b1;
      b1 = b0;
    }
    return x * b1 - b2 + coeff[0];
  }
};
inline ChebApprox ls_pol_approx(ScalarFun fun, const SpectralBounds& bounds, double tol,
                                int max_deg = 300) {
  ChebApprox ap;
  ap.fun = fun;
  ap.lmin = bounds.lmin;
  ap.lmax = bounds.lmax;
  ap.coeff.resize(std::max(max_deg, 0) + 1);
  int deg = 0;
  detail::ok(se_ls_pol_approx(fun == ScalarFun::InverseSqrt ? SE_FUN_INVSQRT : SE_FUN_INV,
                              bounds.lmin, bounds.lmax, tol, max_deg, (int)ap.coeff.size(), &deg,
                              ap.coeff.data(), &ap.achieved_rel_error));
  ap.coeff.resize(deg + 1);
  return ap;
}
// y = p(B) v (deg B-products on the device; the operator must be CSR-backed)
inline void apply_cheb(const ChebApprox& ap, const Operator& b, const Vec& v, Vec& y,
                       Counters* counters = nullptr) {
  y.assign(v.size(), 0.0);
  detail::ok(se_apply_cheb(detail::ctx(), detail::dev_of(b, "apply_cheb"), ap.lmin, ap.lmax,
                           ap.degree(), ap.coeff.data(), 1, v.data(), y.data()));
  if (counters) counters->n_B_matvec += ap.degree();
}

// ---- filter_poly.hpp -----------------------------------------------------------------------------------------
enum class Damping { None, LanczosSigma, Jackson };
struct SpectralMap {
  double c = 0.0, d = 1.0;
  SpectralMap() = default;
  explicit SpectralMap(const SpectralBounds& b) : c(0.5 * (b.lmax + b.lmin)), d(0.5 * (b.lmax - b.lmin)) {
    if (!(d > 0.0)) throw std::invalid_argument("SpectralMap: empty spectral interval");
  }
  double to_ref(double lambda) const { return (lambda - c) / d; }
  double from_ref(double t) const { return c + d * t; }
};
struct PolynomialFilter {
  int k = 0;
  double gamma = 0.0;
  Vec mu;
  SpectralMap map;
  double tau = 0.8;
  double ta = -1.0, tb = 1.0;
  double bar = 0.0;
  Damping damping = Damping::LanczosSigma;
  bool cap_reached = false;
};
struct PolyOpts {
  double tau = 0.8;
  int max_deg = 3000;
  Damping damping = Damping::LanczosSigma;
};
namespace detail {
inline int damp_code(Damping d) {
  return d == Damping::None ? SE_DAMP_NONE : (d == Damping::Jackson ? SE_DAMP_JACKSON : SE_DAMP_SIGMA);
}
inline se_poly_filter to_c(const PolynomialFilter& f) {
  se_poly_filter s{};
  s.k = f.k;
  s.gamma = f.gamma;
  s.c = f.map.c;
  s.d = f.map.d;
  s.tau = f.tau;
  s.ta = f.ta;
  s.tb = f.tb;
  s.bar = f.bar;
  s.damping = damp_code(f.damping);
  s.cap_reached = f.cap_reached;
  s.mu = const_cast<double*>(f.mu.data());
  s.mu_cap = (int)f.mu.size();
  return s;
}
}  // namespace detail

inline Vec chebyshev_coeffs(double gamma, int k) {
  Vec mu(std::max(k + 1, 1));
  detail::ok(se_chebyshev_coeffs(gamma, k, mu.data()));
  return mu;
}
inline Vec damping_multipliers(int k, Damping kind) {
  Vec s(k + 1);
  detail::ok(se_damping_multipliers(k, detail::damp_code(kind), s.data()));
  return s;
}
inline double balance_center(int k, double ta, double tb, Damping kind) {
  double g = 0.0;
  detail::ok(se_balance_center(k, ta, tb, detail::damp_code(kind), &g));
  return g;
}
inline double eval_pol(const PolynomialFilter& f, double t) {
  double out = 0.0;
  const se_poly_filter s = detail::to_c(f);
  detail::ok(se_eval_pol(&s, t, &out));
  return out;
}
inline PolynomialFilter find_pol(double xi, double eta, const SpectralBounds& bounds,
                                 const PolyOpts& opts = {}) {
  Vec mu(std::max(opts.max_deg, 2) + 1);
  se_poly_filter s{};
  s.mu = mu.data();
  s.mu_cap = (int)mu.size();
  detail::ok(se_find_pol(xi, eta, bounds.lmin, bounds.lmax, opts.tau, opts.max_deg,
                         detail::damp_code(opts.damping), &s));
  PolynomialFilter f;
  f.k = s.k;
  f.gamma = s.gamma;
  f.mu.assign(mu.begin(), mu.begin() + s.k + 1);
  f.map.c = s.c;
  f.map.d = s.d;
  f.tau = s.tau;
  f.ta = s.ta;
  f.tb = s.tb;
  f.bar = s.bar;
  f.damping = opts.damping;
  f.cap_reached = s.cap_reached != 0;
  return f;
}
// out = rho(Ahat) v on the GPU; exactly k A-products (bitwise the reference's result).
inline void apply_pol(const PolynomialFilter& f, const Operator& op_a, const Vec& v, Vec& out,
                      Counters* cnt = nullptr) {
  out.assign(op_a.n, 0.0);
  const se_poly_filter s = detail::to_c(f);
  long nmv = 0;
  detail::ok(se_cheb_apply(detail::ctx(), detail::dev_of(op_a, "apply_pol"), &s, 1, v.data(),
                           out.data(), &nmv));
  if (cnt) cnt->n_A_matvec += nmv;
}

// ---- dos.hpp / slicer.hpp ------------------------------------------------------------------------------------
enum class DosMethod { Kpm, Lanczos };
enum class ProbeKind { Rademacher, Gaussian };  // extension: Gaussian probes (BASELINE cfg2)
struct DosConfig {
  DosMethod method = DosMethod::Kpm;
  int m = 60;
  int n_vec = 40;
  int npts = 300;
  double gaussian_sigma = 0.0;
  std::uint64_t seed = 1234;
  ProbeKind probes = ProbeKind::Rademacher;
};
struct DosCurve {
  Vec xdos, ydos;
  double nev_est = 0.0;
  int n = 0;
};
inline DosCurve kpm_dos(const Operator& op, const SpectralBounds& bounds, const DosConfig& cfg = {}) {
  DosCurve c;
  c.n = op.n;
  c.xdos.resize(std::max(cfg.npts, 0));
  c.ydos.resize(std::max(cfg.npts, 0));
  detail::ok(se_kpm_dos(detail::ctx(), detail::dev_of(op, "kpm_dos"), bounds.lmin, bounds.lmax,
                        cfg.m, cfg.n_vec, cfg.npts, cfg.seed,
                        cfg.probes == ProbeKind::Gaussian ? SE_PROBE_GAUSSIAN : SE_PROBE_RADEMACHER,
                        c.xdos.data(), c.ydos.data(), &c.nev_est));
  return c;
}
// B200 extension: kpm_dos with its probes split over several GPUs of this
// process and the moments combined by one NCCL all-reduce; bit-identical to kpm_dos.
inline DosCurve kpm_dos_devices(const CsrMatrix& a, const SpectralBounds& bounds,
                                const DosConfig& cfg, const std::vector<int>& devices) {
  DosCurve c;
  c.n = a.n();
  c.xdos.resize(std::max(cfg.npts, 0));
  c.ydos.resize(std::max(cfg.npts, 0));
  detail::ok(se_kpm_dos_multi((int)devices.size(), devices.data(), a.n(), a.row_ptr().data(),
                              a.col_idx().data(), a.vals().data(), bounds.lmin, bounds.lmax, cfg.m,
                              cfg.n_vec, cfg.npts, cfg.seed,
                              cfg.probes == ProbeKind::Gaussian ? SE_PROBE_GAUSSIAN
                                                                : SE_PROBE_RADEMACHER,
                              c.xdos.data(), c.ydos.data(), &c.nev_est));
  return c;
}
inline DosCurve lan_dos(const Operator& op, const SpectralBounds& bounds, const DosConfig& cfg = {}) {
  DosCurve c;
  c.n = op.n;
  c.xdos.resize(std::max(cfg.npts, 0));
  c.ydos.resize(std::max(cfg.npts, 0));
  detail::ok(se_lan_dos(detail::ctx(), detail::dev_of(op, "lan_dos"), bounds.lmin, bounds.lmax,
                        cfg.m, cfg.n_vec, cfg.npts, cfg.gaussian_sigma, cfg.seed, c.xdos.data(),
                        c.ydos.data(), &c.nev_est));
  return c;
}
// Pencil density (dos.hpp:160-184).  b_solve / b_halfsolve are the reference's Cholesky hooks;
// the device path draws on op_b's CSR matrix instead (S = P A P, P ~ B^-1/2).
inline DosCurve dos_generalized(const Operator& op_a, const Operator& b_solve,
                                const Operator& b_halfsolve, const Operator& op_b,
                                const SpectralBounds& bounds, const DosConfig& cfg = {}) {
  (void)b_solve;
  (void)b_halfsolve;
  InnerProduct ip;
  ip.b = &op_b;
  se_pencil* pen = detail::pencil_for(ip, "dos_generalized");
  DosCurve c;
  c.n = op_a.n;
  c.xdos.resize(std::max(cfg.npts, 0));
  c.ydos.resize(std::max(cfg.npts, 0));
  const int rc = se_lan_dos_pencil(detail::ctx(), detail::dev_of(op_a, "dos_generalized"), pen,
                                   bounds.lmin, bounds.lmax, cfg.m, cfg.n_vec, cfg.npts,
                                   cfg.gaussian_sigma, cfg.seed, c.xdos.data(), c.ydos.data(),
                                   &c.nev_est);
  se_pencil_free(pen);
  detail::ok(rc);
  return c;
}
inline double dos_count(const DosCurve& c, double xi, double eta) {
  double out = 0.0;
  detail::ok(se_dos_count((int)c.xdos.size(), c.n, c.xdos.data(), c.ydos.data(), xi, eta, &out));
  return out;
}
struct SliceSet {
  Vec breakpoints, est_counts;
  int ns() const { return (int)breakpoints.size() - 1; }
};
inline SliceSet slice_spectrum(const DosCurve& curve, double xi, double eta, int ns) {
  SliceSet s;
  s.breakpoints.resize(std::max(ns + 1, 1));
  s.est_counts.resize(std::max(ns, 1));
  detail::ok(se_slice_spectrum((int)curve.xdos.size(), curve.n, curve.xdos.data(),
                               curve.ydos.data(), xi, eta, ns, s.breakpoints.data(),
                               s.est_counts.data()));
  s.est_counts.resize(ns);
  return s;
}

// ---- eigensolvers.hpp (polynomial drivers) ------------------------------------------------------------------
struct SolverConfig {
  int m = 0;
  long max_its = 0;
  int ncycle = 30;
  double tau1 = 0.0;
  double res_tol = 1e-8;
  int est_count = 20;
  unsigned long seed = 1234;
};
struct DeflationSet {
  DenseMat u;
  Vec values;
  int count() const { return u.cols(); }
};
struct EigenResults {
  Vec eigenvalues;
  DenseMat vectors;
  Vec residuals;
  long niter = 0;
  Counters counters;
  bool hit_max_its = false;
};

inline std::pair<double, double> rayleigh_and_residual(const CsrMatrix& a, const CsrMatrix* b,
                                                       const Vec& u) {
  if ((int)u.size() != a.n()) throw std::invalid_argument("rayleigh_and_residual: vector size mismatch");
  if (b) {  // lambda = u'Au / u'Bu, r = ||Au - lambda Bu|| (eigensolvers.hpp:86-106); products on the GPU
    if (b->n() != a.n()) throw std::invalid_argument("rayleigh_and_residual: pencil size mismatch");
    const Vec au = a.matvec(u), bu = b->matvec(u);
    const double uu = dot(u, bu);
    if (!(uu > 0.0)) throw std::invalid_argument("rayleigh_and_residual: zero (or B-degenerate) vector");
    const double lambda = dot(u, au) / uu;
    Vec r = au;
    axpy(-lambda, bu, r);
    return {lambda, nrm2(r)};
  }
  double lam = 0.0, res = 0.0;
  detail::ok(se_rayleigh_residual(detail::ctx(), a.device(), u.data(), &lam, &res));
  return {lam, res};
}

namespace detail {
inline EigenResults collect(se_results* r, int n);
inline EigenResults cheb_lan(int solver, const CsrMatrix& a, const CsrMatrix* b,
                             const PolynomialFilter& f, double xi, double eta,
                             const SolverConfig& cfg, const DeflationSet* locked);

// Generalized pencil (A, B) with a diagonal SPD B (lumped mass, BASELINE cfg5): B = D^-2,
// D = diag(b_i^-1/2), and (A, B) has the eigenpairs (lambda, D y) of the standard matrix
// D A D (vals[p] = (a_ij d_i) d_j, as se_csr_scale_sym).  The reference's B-weighted path
// (eigensolvers.hpp:640-690, SpdFactor solves) reaches the same pencil eigenpairs; non-diagonal B
// needs a sparse Cholesky, outside the device path.
inline Vec pencil_diag(const CsrMatrix& a, const CsrMatrix& b, const std::string& who) {
  if (b.n() != a.n()) throw std::invalid_argument(who + ": pencil size mismatch");
  Vec bd(b.n());
  for (int i = 0; i < b.n(); ++i) {
    const int p0 = b.row_ptr()[i], p1 = b.row_ptr()[i + 1];
    if (p1 - p0 != 1 || b.col_idx()[p0] != i || !(b.vals()[p0] > 0.0))
      throw std::invalid_argument(who + ": generalized pencils need a diagonal SPD B on the device path");
    bd[i] = b.vals()[p0];
  }
  return bd;
}
// Solve the scaled standard problem D A D with `solve(S, d)`, then map its eigenpairs back to the
// pencil: x = D y (B-normalised) and the reference's residual ||A x - lambda B x||.
template <class Solve>
inline EigenResults pencil_scaled(const CsrMatrix& a, const CsrMatrix& b, const std::string& who,
                                  Solve&& solve) {
  const Vec bd = pencil_diag(a, b, who);
  const int n = a.n();
  Vec d(n);
  for (int i = 0; i < n; ++i) d[i] = 1.0 / std::sqrt(bd[i]);
  std::vector<int> rp = a.row_ptr(), ci = a.col_idx();
  Vec v = a.vals();
  for (int i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p) v[p] = (v[p] * d[i]) * d[ci[p]];
  const CsrMatrix s = CsrMatrix::from_csr(n, std::move(rp), std::move(ci), std::move(v));
  // candidates are judged on the pencil residual ||A x - lambda B x|| / sqrt(x'Bx) = ||D^-1 r_s||
  // (eigensolvers.hpp:289-316), so acceptance matches the reference's B-weighted path
  Vec w(n);
  for (int i = 0; i < n; ++i) w[i] = std::sqrt(bd[i]);
  ok(se_csr_set_residual_weight(ctx(), s.device(), w.data()));
  EigenResults r = solve(s, d);
  for (int j = 0; j < r.vectors.cols(); ++j) {
    double* x = r.vectors.col(j);
    for (int i = 0; i < n; ++i) x[i] *= d[i];
  }
  return r;
}

inline bool is_diagonal(const CsrMatrix& b) {
  for (int i = 0; i < b.n(); ++i)
    if (b.row_ptr()[i + 1] - b.row_ptr()[i] != 1 || b.col_idx()[b.row_ptr()[i]] != i) return false;
  return true;
}

// A general sparse SPD B on the device: se_pencil (S = P A P with P ~ B^-1/2 a Chebyshev series
// in B; the reference's Cholesky B-solves become B-products).  RAII over the C handle.
struct PencilHandle {
  se_pencil* p = nullptr;
  explicit PencilHandle(const CsrMatrix& b) { ok(se_pencil_create(ctx(), b.device(), 0.0, 0, &p)); }
  ~PencilHandle() { se_pencil_free(p); }
  PencilHandle(const PencilHandle&) = delete;
  PencilHandle& operator=(const PencilHandle&) = delete;
};

inline EigenResults cheb_lan_pencil(int solver, const CsrMatrix& a, const CsrMatrix& b,
                                    const PolynomialFilter& f, double xi, double eta,
                                    const SolverConfig& cfg, const DeflationSet* locked) {
  const std::string who = solver ? "cheb_lan_tr" : "cheb_lan_nr";
  if (!is_diagonal(b)) {
    if (locked && locked->count() > 0)
      throw std::invalid_argument(who + ": a preloaded deflation set is not supported for a non-diagonal B");
    PencilHandle pen(b);
    const se_poly_filter s = to_c(f);
    const se_solver_cfg c{cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count, cfg.seed};
    se_results* r = nullptr;
    ok(se_cheb_lan_pencil(ctx(), a.device(), pen.p, &s, xi, eta, &c, solver, &r));
    return collect(r, a.n());
  }
  return pencil_scaled(a, b, who, [&](const CsrMatrix& s, const Vec& d) {
    DeflationSet ly;
    if (locked && locked->count() > 0) {  // locked pencil vectors x -> y = D^-1 x
      ly.values = locked->values;
      ly.u = DenseMat(locked->u.rows(), locked->u.cols());
      for (int j = 0; j < ly.u.cols(); ++j)
        for (int i = 0; i < std::min((int)d.size(), ly.u.rows()); ++i) ly.u(i, j) = locked->u(i, j) / d[i];
    }
    return cheb_lan(solver, s, nullptr, f, xi, eta, cfg, locked ? &ly : nullptr);
  });
}

inline EigenResults cheb_lan(int solver, const CsrMatrix& a, const CsrMatrix* b,
                             const PolynomialFilter& f, double xi, double eta,
                             const SolverConfig& cfg, const DeflationSet* locked) {
  const char* who = solver ? "cheb_lan_tr" : "cheb_lan_nr";
  if (b && b->n() != a.n()) throw std::invalid_argument(std::string(who) + ": pencil size mismatch");
  if (b) return cheb_lan_pencil(solver, a, *b, f, xi, eta, cfg, locked);
  const se_poly_filter s = to_c(f);
  const se_solver_cfg c{cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count, cfg.seed};
  int nd = 0;
  if (locked && locked->count() > 0) {
    if (locked->u.rows() != a.n()) throw std::invalid_argument(std::string(who) + ": deflation size mismatch");
    if ((int)locked->values.size() != locked->u.cols())
      throw std::invalid_argument(std::string(who) + ": deflation values/vectors mismatch");
    nd = locked->count();
  }
  se_results* r = nullptr;
  ok(se_cheb_lan(ctx(), a.device(), &s, xi, eta, &c, solver, nd, nd ? locked->u.data() : nullptr,
                 nd ? locked->values.data() : nullptr, 1, &r));
  return collect(r, a.n());
}
inline EigenResults collect(se_results* r, int n) {
  std::unique_ptr<se_results, int (*)(se_results*)> guard(r, se_results_free);
  int nev = 0;
  ok(se_results_count(r, &nev));
  EigenResults out;
  out.eigenvalues.resize(nev);
  out.residuals.resize(nev);
  out.vectors = DenseMat(n, nev);
  ok(se_results_copy(r, out.eigenvalues.data(), out.residuals.data(), out.vectors.data()));
  se_counters cn{};
  int hit = 0;
  ok(se_results_info(r, &out.niter, &hit, &cn));
  out.hit_max_its = hit != 0;
  out.counters.n_A_matvec = cn.n_A_matvec;
  out.counters.t_mv = cn.t_mv;
  out.counters.t_orth = cn.t_orth;
  out.counters.t_total = cn.t_total;
  return out;
}
}  // namespace detail

inline EigenResults cheb_lan_nr(const CsrMatrix& a, const CsrMatrix* b, const PolynomialFilter& f,
                                double xi, double eta, const SolverConfig& cfg = {},
                                const DeflationSet* locked = nullptr) {
  return detail::cheb_lan(0, a, b, f, xi, eta, cfg, locked);
}
inline EigenResults cheb_lan_tr(const CsrMatrix& a, const CsrMatrix* b, const PolynomialFilter& f,
                                double xi, double eta, const SolverConfig& cfg = {},
                                const DeflationSet* locked = nullptr) {
  return detail::cheb_lan(1, a, b, f, xi, eta, cfg, locked);
}
// Filtered subspace iteration (eigensolvers.hpp:760-940), standard problems on the device.
inline EigenResults cheb_si(const CsrMatrix& a, const CsrMatrix* b, const PolynomialFilter& f,
                            double xi, double eta, int est_count, const SolverConfig& cfg = {}) {
  if (b && b->n() != a.n()) throw std::invalid_argument("cheb_si: pencil size mismatch");
  if (b)  // diagonal SPD B: the scaled standard problem (see detail::pencil_scaled)
    return detail::pencil_scaled(a, *b, "cheb_si", [&](const CsrMatrix& s, const Vec&) {
      return cheb_si(s, nullptr, f, xi, eta, est_count, cfg);
    });
  const se_poly_filter s = detail::to_c(f);
  const se_solver_cfg c{cfg.m, cfg.max_its, cfg.ncycle, cfg.tau1, cfg.res_tol, cfg.est_count, cfg.seed};
  se_results* r = nullptr;
  detail::ok(se_cheb_si(detail::ctx(), a.device(), &s, xi, eta, est_count, &c, &r));
  return detail::collect(r, a.n());
}

}  // namespace sliceeig
