/* sliceeig_cuda.h -- the C-ABI boundary of the B200-native polynomial-filtering hot path.
 *
 * libsliceeig_cuda.so (built from paper_1802_05215_b200/csrc) exports exactly the functions
 * declared here: plain pointers and sizes, no C++ or torch types.  The C++ drop-in facade in
 * include/sliceeig/*.hpp (namespace sliceeig, same names and signatures as the reference headers
 * /root/reference/proj/include/sliceeig/*.hpp) is a thin inline layer over these calls, and the
 * Python mirror (paper_1802_05215_b200/api.py) binds them with ctypes.
 *
 * Each entry point cites the reference interface it replaces (<header>:<line> under
 * proj/include/sliceeig/, or tools/sliceeig_main.cpp:<line>).
 *
 * Error convention: every function returns SE_OK (0) or a negative code; se_last_error() gives the
 * message of the last failure on the calling thread (the reference's exception text where one
 * exists).  The facade maps SE_EINVAL -> std::invalid_argument, SE_ERANGE -> std::out_of_range,
 * everything else -> std::runtime_error, matching the reference's exception types.
 *
 * Threading: one se_ctx per host thread (it owns a CUDA stream + cuBLAS/cuSOLVER handles).
 * An se_csr is read-only after creation and may be shared by contexts on the same device.
 * Host-only functions (no se_ctx argument) need no GPU.
 */
#ifndef SLICEEIG_CUDA_H
#define SLICEEIG_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SE_API __attribute__((visibility("default")))
#else
#define SE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SE_OK 0
#define SE_EINVAL (-1)   /* std::invalid_argument in the reference                     */
#define SE_ENUMERIC (-2) /* std::runtime_error (numerical failure) in the reference     */
#define SE_ECUDA (-3)    /* CUDA / cuBLAS / cuSOLVER failure                            */
#define SE_ENOMEM (-4)   /* device allocation failure                                   */
#define SE_ERANGE (-5)   /* std::out_of_range in the reference (csr.hpp:33)             */

/* Damping kinds (filter_poly.hpp:15). */
#define SE_DAMP_NONE 0
#define SE_DAMP_SIGMA 1
#define SE_DAMP_JACKSON 2

/* KPM probe distributions.  Rademacher is the reference's (dos.hpp:97); Gaussian probes
 * (Rng(seed).normal_vec(n) per probe, probe order) serve BASELINE config 2. */
#define SE_PROBE_RADEMACHER 0
#define SE_PROBE_GAUSSIAN 1

typedef struct se_ctx se_ctx;
typedef struct se_csr se_csr;
typedef struct se_results se_results;

/* PolynomialFilter (filter_poly.hpp:81-91) + its SpectralMap (filter_poly.hpp:17-27).
 * mu is caller-owned storage of capacity mu_cap (>= k+1). */
typedef struct se_poly_filter {
  int k;
  double gamma;
  double c, d; /* map: t = (lambda - c) / d */
  double tau;
  double ta, tb;
  double bar;
  int damping;
  int cap_reached;
  double* mu;
  int mu_cap;
} se_poly_filter;

/* SolverConfig (eigensolvers.hpp:46-54); zeros select the reference defaults
 * (resolve_config eigensolvers.hpp:142-151). */
typedef struct se_solver_cfg {
  int m;
  long max_its;
  int ncycle;
  double tau1;
  double res_tol;
  int est_count;
  uint64_t seed;
} se_solver_cfg;

/* Counters (operators.hpp:44-65). */
typedef struct se_counters {
  long n_A_matvec, n_B_matvec, n_B_solve, n_shift_solve;
  double t_mv, t_orth, t_sv, t_total;
} se_counters;

/* ---- library / errors ----------------------------------------------------------------- */
SE_API const char* se_last_error(void);
SE_API const char* se_version(void);
SE_API int se_device_count(int* count);
/* Free / total bytes of a device's memory (sizes the memory plan's solve windows; no reference
   counterpart: the reference is host code). */
SE_API int se_device_memory(int device, size_t* free_bytes, size_t* total_bytes);

/* ---- contexts ----------------------------------------------------------------------------- */
SE_API int se_ctx_create(int device, se_ctx** out);
/* Device bytes the Ritz-candidate evaluation of the drivers may hold at once (default 8 GB):
 * larger candidate sets (eigensolvers.hpp:275-318 over thousands of Ritz vectors at n ~ 2M)
 * are evaluated in column chunks and the thick-restart vectors recomputed once. */
SE_API int se_ctx_set_candidate_budget(se_ctx* ctx, size_t bytes);
SE_API int se_ctx_destroy(se_ctx* ctx);
SE_API int se_ctx_synchronize(se_ctx* ctx);
/* Number of this library's kernels launched on ctx so far (bench evidence). */
SE_API int se_ctx_kernel_launches(se_ctx* ctx, long* out);
/* Device time of the filter kernels (ms, CUDA events on ctx's stream) and their count, since
 * the last reset; used by bench.py for the roofline of the dominant kernel. */
SE_API int se_ctx_filter_timing(se_ctx* ctx, int enable, double* ms, long* launches, double* bytes);

/* ---- matrices (csr.hpp:23-58, laplacian.hpp:19-48) ---------------------------------------- */
/* Host-side closed-form Laplacian (laplacian.hpp:19-48), bitwise the reference's CSR: call with
 * rp == NULL to get n/nnz first. */
SE_API int se_laplacian_host(int ndims, const int* dims, int* n, long* nnz, int* rp, int* ci, double* v);
/* Closed-form spectrum, sorted ascending (laplacian.hpp:51-86). */
SE_API int se_laplacian_eigs(int ndims, const int* dims, double* out);
/* BASELINE cfg4 generator (the reference has none; SURVEY.md §8d defines it): symmetric n x n,
 * band |i-j| <= halfband plus `extras` distinct uniformly random off-band columns per row (drawn
 * in row order from Rng(seed).uniform(), resampled on collision, mirrored), one N(0,1) value per
 * unordered off-diagonal pair (row-major order, then diagonal N(0,1) per row) and diagonal +=
 * diag_frac * sum_j |a_ij|.  Call with rp == NULL for n/nnz, then again to fill. */
SE_API int se_gen_random_sparse(int n, uint64_t seed, int halfband, int extras, double diag_frac,
                                long* nnz, int* rp, int* ci, double* v);
/* BASELINE cfg5 scaling vector: b_i = 0.5 + Rng(seed).uniform(), d_i = 1/sqrt(b_i) (host). */
SE_API int se_mass_scaling(int n, uint64_t seed, double* b, double* d);
/* Upload a host CSR (int32 row_ptr[n+1], int32 col_idx[nnz], f64 vals[nnz]). */
SE_API int se_csr_upload(se_ctx* ctx, int n, const int* row_ptr, const int* col_idx, const double* vals,
                  se_csr** out);
/* Device generator kernel for gen_laplacian (bit-identical to the host / reference CSR). */
SE_API int se_csr_gen_laplacian(se_ctx* ctx, int ndims, const int* dims, se_csr** out);
SE_API int se_csr_info(const se_csr* a, int* n, long* nnz);
SE_API int se_csr_download(se_ctx* ctx, const se_csr* a, int* row_ptr, int* col_idx, double* vals);
/* vals[p] *= d[i] * d[j] for stored (i, j = col_idx[p]): diagonal congruence D A D (BASELINE cfg5). */
SE_API int se_csr_scale_sym(se_ctx* ctx, se_csr* a, const double* d_host);
/* Residual weights w (n doubles, NULL clears): candidate residuals become
   ||w .* (A u - lambda u)|| / sqrt(u.u).  For S = D A D of a diagonal-B pencil, w = D^-1 makes
   them the reference's ||A x - lambda B x|| / sqrt(x'Bx), x = D u (eigensolvers.hpp:289-316), so
   convergence is decided on the pencil residual. */
SE_API int se_csr_set_residual_weight(se_ctx* ctx, se_csr* a, const double* w_host);
SE_API int se_csr_free(se_csr* a);

/* ---- operator applications ---------------------------------------------------------------- */
/* y = A x, host buffers (CsrMatrix::matvec csr.hpp:98-105; backs make_operator operators.hpp:34). */
SE_API int se_spmv(se_ctx* ctx, const se_csr* a, const double* x, double* y);
/* out = rho(Ahat) v for nvec column-major vectors (apply_pol filter_poly.hpp:256-277); host
 * buffers; n_matvec += k per vector (Counters::n_A_matvec). */
SE_API int se_cheb_apply(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int nvec, const double* v,
                  double* out, long* n_matvec);
/* Same with device pointers (inputs already resident in HBM). */
SE_API int se_cheb_apply_dev(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int nvec,
                      const double* d_v, double* d_out);

/* Production timing of the fused filter kernels: one application captured as a CUDA graph and
 * replayed `reps` times between CUDA events on ctx's stream.  Returns the total ms, the number
 * of filter-kernel launches timed, and their algorithmic bytes (Abytes + 32n for the first
 * degree, Abytes + 40n for each further degree). */
SE_API int se_filter_bench(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int reps,
                           double* ms, long* launches, double* bytes);

/* Production timing of one reorthogonalisation pass (orth.hpp:19-32: coef = W^T t, t -= W coef,
 * ||t||) against an n x k basis, graph-captured and replayed `reps` times between CUDA events.
 * Algorithmic bytes per pass: 16 n k + 24 n. */
SE_API int se_cgs_bench(se_ctx* ctx, int n, int k, int reps, double* ms);
/* A full CGS2 step with the re-pass forced: mode 0 = two column-major passes (4 reads of W),
 * mode 2 = the product path on the row-major basis, T1 + fused MID + N2 (3 reads); mode -1 =
 * one column-major pass. */
/* The resident filter (all degrees of apply_pol, filter_poly.hpp:256-277, in one cooperative
 * launch with the matrix held in shared memory; matrices up to ~300k rows / 2.3M entries).
 * se_resident_filter(0) switches it off process-wide (A/B measurements; results are bit-identical
 * either way); se_csr_resident_tiles: row tiles of the matrix' plan, 0 when it does not apply. */
SE_API int se_resident_filter(int enable);
SE_API int se_csr_resident_tiles(const se_csr* a, int* tiles);
/* Shared-memory bytes one tile of the plan holds (0: no plan).  Above half an SM's shared memory a
 * filter launch owns the GPU while it runs, and a caller solves its slices one at a time. */
SE_API int se_csr_resident_smem(const se_csr* a, size_t* bytes);
/* mult_cols (vecops.hpp:81-89) / the Rayleigh-Ritz contractions (eigensolvers.hpp:275-283,
 * 838-871) on the fp64 tensor cores: out (m x n, column-major, ldc) = A B, B[k + col ldb],
 * A[row lda + k] (a_kcontig) or A[row + k lda]; host buffers.  With a or b NULL the operands are
 * synthetic and nothing is copied back (timing); reps > 0: mean device ms of `reps` runs -> *ms. */
SE_API int se_mult_cols(se_ctx* ctx, int m, int n, int k, const double* a, long lda, int a_kcontig,
                        const double* b, long ldb, double* out, long ldc, int reps, double* ms);
SE_API int se_cgs2_bench(se_ctx* ctx, int n, int k, int reps, int mode, double* ms);

/* Production timing of kdeg degrees of the multi-vector filter (nv <= 8 recurrences sharing one
 * staging of A per degree), graph-captured and replayed `reps` times.  Returns total ms. */
SE_API int se_multi_filter_bench(se_ctx* ctx, const se_csr* a, int nv, int kdeg, int reps, double* ms);
/* The same for the row-major block filter (8 vectors, padded-row matrices): kdeg degrees. */
SE_API int se_block_filter_bench(se_ctx* ctx, const se_csr* a, int kdeg, int reps, double* ms);

/* ---- filters (host, filter_poly.hpp) -------------------------------------------------------- */
SE_API int se_damping_multipliers(int k, int damping, double* out);            /* :41-60   */
SE_API int se_chebyshev_coeffs(double gamma, int k, double* out);              /* :30-39   */
SE_API int se_normalized_filter_coeffs(int k, double gamma, int damping, double* out); /* :182-190 */
SE_API int se_balance_center(int k, double ta, double tb, int damping, double* gamma); /* :135-171 */
SE_API int se_find_pol(double xi, double eta, double lmin, double lmax, double tau, int max_deg,
                int damping, se_poly_filter* out);                     /* :198-253  */
SE_API int se_eval_pol(const se_poly_filter* f, double t, double* out);       /* :93-97    */

/* ---- spectral density ----------------------------------------------------------------------- */
/* Unnormalised KPM moment sums over probes [first, first+count) of the probe stream drawn from
 * Rng(seed) (dos.hpp:96-109); probes are generated on the host (mt19937_64) and processed on the
 * device in blocks of up to 16.  zeta_sums has m+1 entries. */
SE_API int se_kpm_moments(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec,
                   int probe_kind, uint64_t seed, int first, int count, double* zeta_sums);
/* Per-probe moments v_l^T T_k(Ahat) v_l for probes [first, first+count): per_probe is
 * count x (m+1) row-major (probe-major).  Summing rows in probe order reproduces the reference's
 * accumulation order (dos.hpp:100-106) independently of how probes were split across GPUs. */
SE_API int se_kpm_moments_probes(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m,
                                 int n_vec, int probe_kind, uint64_t seed, int first, int count,
                                 double* per_probe);
/* Host probe generation: probes [first, first+count) of Rng(seed)'s stream (probe l = the next n
 * values, rng.hpp:43-58 normal_vec / rademacher_vec), written row-major n x count (the layout
 * the device block kernels read).  Host threads start their probes by MT19937-64 jump-ahead
 * where that is exact; the values equal the serial draw bit for bit.  No GPU needed. */
SE_API int se_probe_block(uint64_t seed, int probe_kind, int n, long first, int count, double* out);
/* Jackson-damped curve from normalised moments (dos.hpp:112-131 + dos_finalize :54-60). */
SE_API int se_kpm_curve(int m, const double* zeta, int n, double lmin, double lmax, int npts, double* x,
                 double* y, double* nev_est);
/* kpm_dos (dos.hpp:82-132): moments on the device + curve on the host. */
SE_API int se_kpm_dos(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec, int npts,
               uint64_t seed, int probe_kind, double* x, double* y, double* nev_est);
/* kpm_dos (dos.hpp:82-132) over several GPUs of this process (the reference has
 * one thread: its kpm_dos loop over probes dos.hpp:97-109 is what is split): probes in contiguous
 * ranges (whole blocks of 16 where possible), one host thread + context + CSR copy per GPU, and
 * ONE ncclAllReduce (NCCL loaded at run time) of an n_vec x (m+1) per-probe moment array in which
 * each GPU fills only its own rows -- exact, so the result is bit-identical to se_kpm_dos on one
 * GPU for any device list.  per_probe: n_vec x (m+1) row-major, unnormalised. */
SE_API int se_kpm_moments_multi(int ngpu, const int* devices, int n, const int* row_ptr,
                                const int* col_idx, const double* vals, double lmin, double lmax,
                                int m, int n_vec, int probe_kind, uint64_t seed, double* per_probe);
SE_API int se_kpm_dos_multi(int ngpu, const int* devices, int n, const int* row_ptr,
                            const int* col_idx, const double* vals, double lmin, double lmax, int m,
                            int n_vec, int npts, uint64_t seed, int probe_kind, double* x, double* y,
                            double* nev_est);
/* NCCL version linked at run time (e.g. 22809 for 2.28.9); SE_ECUDA when NCCL is absent. */
SE_API int se_nccl_version(int* version);
/* lan_dos (dos.hpp:136-154): device Lanczos per probe + host Ritz-Gaussian quadrature. */
SE_API int se_lan_dos(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec, int npts,
               double sigma, uint64_t seed, double* x, double* y, double* nev_est);
SE_API int se_dos_count(int npts, int n, const double* x, const double* y, double xi, double eta,
                 double* out);                                          /* dos.hpp:212-218 */
SE_API int se_slice_spectrum(int npts, int n, const double* x, const double* y, double xi, double eta,
                      int ns, double* breakpoints, double* est_counts); /* slicer.hpp:18-64 */

/* ---- Krylov building blocks ----------------------------------------------------------------- */
/* lan_tr_bounds (lanczos.hpp:148-277) with a device Lanczos. */
SE_API int se_lan_tr_bounds(se_ctx* ctx, const se_csr* a, double tol, int restart_dim, int max_restarts,
                     uint64_t seed, double* lmin, double* lmax);
/* lanczos_run (lanczos.hpp:37-118), euclidean.  alpha[m], beta[m-1] host; basis optional
 * (n x steps column-major host buffer, may be NULL). */
SE_API int se_lanczos_run(se_ctx* ctx, const se_csr* a, const double* start, int m, double* alpha,
                   double* beta, int* steps, int* breakdown, double* next_beta, double* next_w,
                   double* basis);
/* paired_cgs2 (orth.hpp:70-80) on host buffers: t (n) against W (n x k column-major); h may be
 * NULL (else h[k] accumulates the coefficients). */
SE_API int se_paired_cgs2(se_ctx* ctx, int n, int k, const double* W, double* t, double* h);
/* Small dense/tridiagonal symmetric eigensolvers (host; tridiag_eig.hpp:111-131,
 * dense_eig.hpp:114-139).  vectors: m x m column-major, may be NULL when want == 0. */
SE_API int se_sym_tridiag_eig(int m, const double* alpha, const double* beta, int want, double* values,
                       double* vectors);
/* Thick-restart arrowhead (theta[l], s[l], tip alpha_l) reduced to tridiagonal form by Givens
 * rotations on indices 0..l-1 (host, O(l^2)); diag[l+1], off[l].  Used for the device stagnation
 * checks of cheb_lan_tr (eigensolvers.hpp:562-572). */
SE_API int se_arrow_tridiag(int l, const double* theta, const double* s, double alpha_l,
                            double* diag, double* off);
SE_API int se_dense_sym_eig(int m, const double* a, int want, int size_guard, double* values,
                     double* vectors);

/* ---- slice drivers (eigensolvers.hpp:703-732) ------------------------------------------------ */
/* solver: 0 = cheb_lan_nr, 1 = cheb_lan_tr.  Optional deflation set (DeflationSet
 * eigensolvers.hpp:69-73): defl_u host n x ndefl column-major + defl_vals, or ndefl = 0.
 * want_vectors: 0 keeps eigenvectors on the device only (bench path).  Returns a results handle. */
SE_API int se_cheb_lan(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, double xi, double eta,
                const se_solver_cfg* cfg, int solver, int ndefl, const double* defl_u,
                const double* defl_vals, int want_vectors, se_results** out);
/* cheb_si (eigensolvers.hpp:760-940): filtered subspace iteration on a block of
 * ceil(1.3 est_count) + 8 vectors (filter sweep on the multi-vector kernel, CGS2 re-orthonormal-
 * isation, Rayleigh-Ritz by DGEMM + syevd); SE_ENUMERIC when the block saturates above the bar. */
SE_API int se_cheb_si(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, double xi, double eta,
                      int est_count, const se_solver_cfg* cfg, se_results** out);
/* ---- general SPD-B pencils (A, B) ------------------------------------------------------------
 * The reference solves them with Cholesky-backed B-solves (cholesky.hpp, eigensolvers.hpp:
 * 640-732).  Here a pencil is the standard problem S = P A P with P ~ B^-1/2 a Chebyshev series
 * in B (ls_pol_approx InverseSqrt, cheb_approx.hpp:40-88, applied like apply_cheb :91-112): every
 * B-solve becomes B-products on the GPU, eigenvalues are the pencil's, eigenvectors come back as
 * x = P y with x'Bx = 1, residuals are ||Ax - lambda Bx|| / sqrt(x'Bx).  B must outlive the
 * pencil handle. */
typedef struct se_pencil se_pencil;
#define SE_FUN_INV 0
#define SE_FUN_INVSQRT 1
/* ls_pol_approx (cheb_approx.hpp:40-88): fun SE_FUN_INV (1/t) or SE_FUN_INVSQRT (1/sqrt t). */
SE_API int se_ls_pol_approx(int fun, double lmin, double lmax, double tol, int max_deg, int cap,
                            int* degree, double* coeff, double* achieved);
/* apply_cheb (cheb_approx.hpp:91-112): y = p(B) x for nvec host column-major vectors. */
SE_API int se_apply_cheb(se_ctx* ctx, const se_csr* b, double lmin, double lmax, int degree,
                         const double* coeff, int nvec, const double* x, double* y);
/* B's spectrum by lan_tr_bounds, widened, and the B^-1/2 fit (tol 0 -> 1e-13, max_deg 0 -> 300). */
SE_API int se_pencil_create(se_ctx* ctx, const se_csr* b, double tol, int max_deg, se_pencil** out);
SE_API int se_pencil_info(const se_pencil* p, int* degree, double* bmin, double* bmax,
                          double* achieved);
SE_API int se_pencil_free(se_pencil* p);
/* lan_tr_bounds with ip = {B, B-solve} (lanczos.hpp:148-277), sliceeig_main.cpp:128-136. */
SE_API int se_lan_tr_bounds_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p, double tol,
                                   int restart_dim, int max_restarts, uint64_t seed, double* lmin,
                                   double* lmax);
/* dos_generalized (dos.hpp:160-184): Lanczos density of the pencil. */
SE_API int se_lan_dos_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p, double lmin,
                             double lmax, int m, int n_vec, int npts, double sigma, uint64_t seed,
                             double* x, double* y, double* nev_est);
/* cheb_lan_nr / cheb_lan_tr(a, &b, ...) (eigensolvers.hpp:703-732) for a general SPD B. */
SE_API int se_cheb_lan_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p,
                              const se_poly_filter* f, double xi, double eta,
                              const se_solver_cfg* cfg, int solver, se_results** out);
SE_API int se_results_count(const se_results* r, int* nev);
/* eigenvalues/residuals (nev each, ascending by eigenvalue), vectors (n x nev, may be NULL). */
SE_API int se_results_copy(const se_results* r, double* eigenvalues, double* residuals, double* vectors);
/* One eigenvector (n doubles; EigenResults.vectors column `index`, eigensolvers.hpp:75-82):
   lets a caller walk a result too large for one host block. */
SE_API int se_results_vector(const se_results* r, int index, double* vector);
SE_API int se_results_info(const se_results* r, long* niter, int* hit_max_its, se_counters* counters);
/* Reorthogonalisation accounting of a slice solve (extension, measurement only): projection
   passes over the Krylov basis, basis columns summed over them, algorithmic HBM bytes. */
SE_API int se_results_orth(const se_results* r, long long* passes, long long* cols, double* bytes);
SE_API int se_results_free(se_results* r);

/* ---- checks ---------------------------------------------------------------------------------- */
/* rayleigh_and_residual (eigensolvers.hpp:86-106), standard problem, host vector u. */
SE_API int se_rayleigh_residual(se_ctx* ctx, const se_csr* a, const double* u, double* lambda,
                         double* residual);

#ifdef __cplusplus
}
#endif

#endif /* SLICEEIG_CUDA_H */
