// Device Lanczos engine: the recurrences of lanczos.hpp and eigensolvers.hpp with the basis,
// locked set and per-step scalars resident in HBM; host code only makes the per-ncycle
// decisions (stagnation, candidates, locking, restarts) exactly as the reference does.
#pragma once

#include <memory>

#include "host_algos.hpp"
#include "kernels.hpp"

namespace se {

// The operator applied each step: plain A (lanczos_run, lan_tr_bounds) or the polynomial filter
// rho(Ahat) (cheb_lan_nr/tr through apply_pol).
struct StepOp {
  bool plain = true;
  int k = 0;
  Vec mu;
  double c = 0.0, invd = 1.0;
};

struct SolverCfg {  // SolverConfig after resolve_config (eigensolvers.hpp:142-151)
  int m = 80;
  long max_its = 1100;
  int ncycle = 30;
  double tau1 = 0.0;
  double res_tol = 1e-8;
  int est_count = 20;
  std::uint64_t seed = 1234;
};
SolverCfg resolve_config(const se_solver_cfg* in, const char* who);

// A generalized pencil (A, B), B sparse SPD, solved as the standard problem S = P A P with
// P ~ B^(-1/2): a Chebyshev least-squares series in B (ls_pol_approx, cheb_approx.hpp:40-88)
// applied by the same fused SpMV recurrence as the filter (apply_cheb, :91-112).  The spectrum
// of S is the pencil's; eigenvectors map back as x = P y (B-normalised), and candidate
// residuals are the reference's ||A x - lambda B x|| / sqrt(x' B x) (eigensolvers.hpp:289-316).
// Every B-solve of the reference's Cholesky path (cholesky.hpp) becomes B-products on the GPU.
struct Pencil {
  const DevCsr* B = nullptr;
  StepOp P;  // plain = false, k = series degree, mu = coefficients, c / invd = the fit interval map
};

struct SliceResult {
  Vec eigenvalues, residuals;
  DevMat vectors;  // n x nev on the device (column i pairs with eigenvalues[i])
  long niter = 0;
  bool hit_max_its = false;
  se_counters counters{};
  int n = 0;
  // reorthogonalisation accounting (device counters): Krylov-basis projection passes, the
  // basis columns they covered, and their algorithmic HBM bytes
  long long orth_passes = 0, orth_cols = 0;
  double orth_bytes = 0.0;
};

// Apply the filter (plain A or rho(Ahat)) to nvec column-major device vectors.
void apply_filter_dev(Ctx& c, const DevCsr& a, const StepOp& op, int nvec, const double* v,
                      double* out);

// The same on the multi-vector kernel (8 columns per launch; bitwise the per-column result).
void apply_filter_block(Ctx& c, const DevCsr& a, const StepOp& op, int nvec, const double* v,
                        double* out);

// Lanczos-family drivers.
struct LanczosRun {
  Vec alpha, beta;
  int steps = 0;
  bool breakdown = false;
  double next_beta = 0.0;
  Vec next_w;
  Vec basis;  // n x steps (optional)
};
LanczosRun lanczos_run(Ctx& c, const DevCsr& a, const double* start_host, int m, bool want_basis,
                       const Pencil* pen = nullptr);
void lan_tr_bounds(Ctx& c, const DevCsr& a, double tol, int restart_dim, int max_restarts,
                   std::uint64_t seed, double& lmin, double& lmax, const Pencil* pen = nullptr);

// Polynomial filtered Lanczos slice drivers (run_nr eigensolvers.hpp:385-472 and run_tr
// :481-628, wired as cheb_lan_nr/tr :703-732).  defl_u: host n x ndefl preloaded locked set.
std::unique_ptr<SliceResult> cheb_lan(Ctx& c, const DevCsr& a, const PolyFilter& f, double xi,
                                      double eta, const SolverCfg& cfg, bool thick_restart,
                                      int ndefl, const double* defl_u, const double* defl_vals,
                                      const char* who, const Pencil* pen = nullptr);
// y = P x for nvec column-major vectors (the pencil's B^(-1/2) series; apply_cheb).
void pencil_map(Ctx& c, const Pencil& pen, int nvec, const double* x, double* y);

// Filtered subspace iteration (cheb_si, eigensolvers.hpp:760-940) on a block of
// ceil(1.3 est_count) + 8 vectors; standard problems.
std::unique_ptr<SliceResult> cheb_si(Ctx& c, const DevCsr& a, const PolyFilter& f, double xi,
                                     double eta, int est_count, const SolverCfg& cfg);

}  // namespace se

namespace se {
void filter_bench(Ctx& c, const DevCsr& a, const StepOp& op, int reps, double& ms, long& launches);
}
namespace se {
void cgs_bench(Ctx& c, int n, int kcols, int reps, double& ms);
void cgs2_bench(Ctx& c, int n, int kcols, int reps, int mode, double& ms);
}
namespace se {
void multi_filter_bench(Ctx& c, const DevCsr& a, int nv, int kdeg, int reps, double& ms);
void block_filter_bench(Ctx& c, const DevCsr& a, int kdeg, int reps, double& ms);
}
