// Host-side launchers of the sm_100a kernels (definitions in *.cu).
//
// Device-resident control block: every Krylov kernel reads the current column index and the
// halt flag from `Ctl` in HBM, so one Lanczos step can be captured once as a CUDA graph and
// replayed without host round trips (the reference's per-step scalar logic, eigensolvers.hpp:
// 400-471 / 518-560, runs on the device between replays).
#pragma once

#include "ctx.hpp"

namespace se {

struct Ctl {
  int i;        // current Krylov column: the step filters W[:, i]
  int halted;   // set by k_normalize on breakdown (beta <= 1e-14, orth.hpp:14); later kernels no-op
  int repass;   // DGKS re-pass decision of the current CGS2 (orth.hpp:77)
  int npass;    // passes executed in the current CGS2
  int ncols;    // columns the current projection runs over (i+1)
  int nlock;    // locked columns for deflation (eigensolvers.hpp:205-215)
  int pad[2];
  double before, after;  // norms for the DGKS test
  double alpha, beta;    // NR recurrence scalars
  double beta_prev;
  unsigned long long ts0, ts1;  // %globaltimer stamps (ns) for the Counters timers
  double t_mv_ns, t_orth_ns;    // accumulated filter / orthogonalisation device time
  long long passes_total;       // CGS passes executed (DGKS statistics)
  long long cols_total;         // basis columns summed over those passes
  long long reads_cols;         // basis columns streamed from HBM (row-major CGS2: T1 + MID + N2)
};

namespace k {

enum ChebMode { kPlain = 0, kFirst = 1, kNext = 2 };

struct ChebArgs {
  const double* x = nullptr;     // input vector (or base of W when src_ctl != nullptr)
  const double* prev = nullptr;  // T_{j-2} term (kNext)
  double* y = nullptr;           // output T_j(Ahat) v (or A x for kPlain)
  double* out = nullptr;         // running sum sum_j mu_j T_j v
  double c = 0.0, invd = 1.0;    // map (filter_poly.hpp:259)
  double mu0 = 0.0, muj = 0.0;
  const Ctl* src_ctl = nullptr;  // x = x + ctl->i * src_ld when set
  long src_ld = 0;
  const Ctl* halt = nullptr;     // skip when halt->halted
  int ncols = 1;                 // kPlain: column-major batch (blockIdx.y), ld = n
};

// Fused CSR SpMV + Chebyshev three-term recurrence + mu-accumulation (one filter degree).
void spmv_cheb(Ctx& c, const DevCsr& a, int mode, const ChebArgs& args);

// One filter degree for up to 8 independent recurrences sharing A (the slices of one GPU):
// per vector q, first[q] selects the j = 1 update, x/prev may be W[:, ctl[q]->i] (x_ind/prev_ind),
// and a halted ctl[q] skips the vector.
struct MultiArgs {
  const double* x[8];
  const double* prev[8];
  double* y[8];
  double* out[8];
  double mu0[8], muj[8];
  const Ctl* ctl[8];
  int x_ind[8], prev_ind[8], first[8];
  long ld;
  double c, invd;
  int nv;
};
void spmv_cheb_multi(Ctx& c, const DevCsr& a, const MultiArgs& args);



// Block filter degree on a row-major n x 8 vector block (padded-row matrices; K2): Y = T_j,
// O = running sum; first: j = 1 (X = v, P unused), else X = T_{j-1}, P = T_{j-2}.
bool cheb_block_available(const DevCsr& a);
void cheb_block_pack(Ctx& c, const double* colmajor, double* rowmajor, int n, int nv);
void cheb_block_unpack(Ctx& c, const double* rowmajor, double* colmajor, int n, int nv);
void cheb_block_step(Ctx& c, const DevCsr& a, bool first, const double* X, const double* P,
                     double* Y, double* O, double cc, double invd, double mu0, double muj);

// Resident filter (resident.cu): out = sum_j mu[j] T_j(Ahat) x, all kdeg degrees in one
// cooperative launch with the matrix held in shared memory; available when resident_tiles(a) > 0.
// state: resident_state_bytes(a) zero-initialised device bytes that belong to one caller (the
// tile-exchange buffers and the tag epoch, which advances across launches).
void resident_build(Ctx& c, DevCsr& a);
void resident_free(DevCsr& a);
int resident_tiles(const DevCsr& a);
size_t resident_state_bytes(const DevCsr& a);
size_t resident_tile_smem(const DevCsr& a);
void resident_enable(int mode);  // process-wide switch (A/B measurements): 0 off, 1 on (default)
bool resident_enabled();
void cheb_resident(Ctx& c, const DevCsr& a, int kdeg, const double* mu_dev, double cc, double invd,
                   const double* x, double* out, void* state, const Ctl* halt);

// Block KPM step over b <= 16 row-major probe columns (dos.hpp:98-108):
//   first: w1 = (A w0 - c w0)/d ; zeta[0], zeta[1] partials
//   next : t  = 2 (A w1 - c w1)/d - w0 ; zeta[k] partial
// partials are reduced deterministically into zeta_block[b] for moment k.
struct Scratch;
size_t kpm_scratch_doubles(const Ctx& c, int n);
// mode 1: first step (w1 = Ahat v; v.v, v.w1); 0: direct (t = 2 Ahat w1 - w0; v.t -> moment kmom);
// 2: doubling (t = w_{k+1}; w_k.w_k -> slot 2 kmom, w_k.w_{k+1} -> slot 2 kmom + 1).
// rm[i b + l] = pm[l n + i]: a probe-major host block to the row-major device layout
void transpose_probes(Ctx& c, const double* pm, double* rm, int n, int b);
// Rademacher sign bits (probe-major, (n + 63) / 64 words per probe; bit set -> +1) -> row-major
// n x bk doubles, columns b .. bk-1 zero.
void expand_rademacher(Ctx& c, const std::uint64_t* bits, double* rm, int n, int b, int bk);
void kpm_step(Ctx& c, const Scratch& s, const DevCsr& a, int b, int mode, const double* v,
              const double* w0, const double* w1, double* t, double cc, double d, double* zeta_dev,
              int kmom);

// Device Laplacian generator (laplacian.hpp:19-48 in closed form).
void gen_laplacian(Ctx& c, int ndims, const int* dims, DevCsr& a);
void csr_scale_sym(Ctx& c, DevCsr& a, const double* d_dev);
// (Re)build the padded-row copy the block KPM kernel reads (no-op when rows exceed kEllW).
void build_ell(Ctx& c, DevCsr& a);
int csr_max_row_nnz(Ctx& c, const DevCsr& a);

// ---- Krylov kernels (orth.hpp, lanczos.hpp, eigensolvers.hpp) -----------------------------
// Scratch owned by the caller (allocated once, outside any graph capture): reduction partials
// and zero-initialised last-CTA counters (each kernel resets the counters it uses).
struct Scratch {
  double* buf = nullptr;
  size_t cap = 0;  // doubles
  unsigned* cnt = nullptr;
  int ncnt = 0;
};
// Doubles of scratch a CGS pass over up to `cap_cols` columns of an n-row basis needs.
size_t cgs_scratch_doubles(const Ctx& c, int n, int cap_cols);
int cgs_counter_slots(int n, int cap_cols);

// ||t|| -> ctl->before/after; resets the DGKS flags.
void norm_before(Ctx& c, const Scratch& s, int n, const double* t, Ctl* ctl);
// NR: t -= beta_arr[i-1] W[:, i-1] (if nonzero); alpha = t . W[:, i] -> ctl->alpha, alpha_arr[i]
void nr_beta_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, Ctl* ctl,
                   double* alpha_arr, const double* beta_arr);
// NR: t -= alpha W[:, i]; before = ||t||
void nr_sub_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, Ctl* ctl);
// One classical Gram-Schmidt pass against the columns of Q (count from ctl: i+1, or nlock
// when use_lock): coef = Q^T t (deterministic), t -= Q coef, after = ||t||, repass flag :=
// !(after > eta*before).  pass2 executes only when ctl->repass is set.  hdiag (optional):
// hdiag[i] += coef[i] (TR's H(i,i) += h[i], eigensolvers.hpp:534).  cap = max column count.
void cgs_pass(Ctx& c, const Scratch& s, int n, double* t, const double* Q, bool use_lock,
              bool pass2, Ctl* ctl, double* hdiag, double* coef, int cap);
// Split CGS pass launchers (same scratch layout as cgs_pass): GEMV-T (coef = Q^T t) only, and
// GEMV-N (t -= Q coef, norm, DGKS flags) only.
void gemvt_only(Ctx& c, const Scratch& s, int n, const double* t, const double* Q, bool pass2,
                Ctl* ctl, double* hdiag, double* coef, int cap);
void gemvn_only(Ctx& c, const Scratch& s, int n, double* t, const double* Q, bool pass2, Ctl* ctl,
                const double* coef, int cap);
// ---- row-major Krylov basis (rowgs.cu) --------------------------------------------------------
// The Lanczos basis W is row-major, W[r * ldw + j] with ldw = rw_ldw(capacity) (even, so every row
// is a 16-byte aligned run of column pairs).  One CGS2 step = T1 (coef1 = W^T t), MID
// (t1 = t - W coef1, ||t1||, DGKS flag, coef2 = W^T t1 from the same staged rows) and N2 (t -= W
// coef2, only when re-passed): three reads of W instead of four.
struct RowScratch {
  double* part = nullptr;   // grid x ldw per-CTA coefficient partials
  double* npart = nullptr;  // grid per-CTA sums of squares
  int grid = 0;             // persistent streaming CTAs
  int ldw = 0;
};
int rw_ldw(int cols);
RowScratch rw_scratch(const Ctx& c, int ldw);          // grid sizing for a basis capacity
size_t rw_scratch_doubles(const RowScratch& s);
void rw_bind(RowScratch& s, double* buf);              // buf: rw_scratch_doubles(s) doubles
// CGS2 of t against W[:, 0..ctl->i] (orth.hpp:63-80): coef1/coef2 (>= ldw doubles) receive the
// two passes' coefficients, hdiag[i] += c (TR, eigensolvers.hpp:534) when non-null; want_before:
// the T1 pass also sets before = after = ||t|| and resets the DGKS flags (TR's step).
// cls: the geometry class (rw_class) of the largest column count the launches will see (-1:
// the capacity's); the kernels handle any count up to it.
void rw_cgs2(Ctx& c, const RowScratch& s, int n, double* t, const double* W, int ldw, Ctl* ctl,
             double* hdiag, double* coef1, double* coef2, bool want_before, int cls = -1);
int rw_class(int ncols);
// dst = W[:, ctl->i + off] (contiguous copy of the step's source column)
void rw_col_get(Ctx& c, int n, const double* W, int ldw, const Ctl* ctl, int off, double* dst);
// beta = after; breakdown -> halted; else W[:, i+1] = t / beta, beta_arr[i] = beta, i++.
void rw_normalize(Ctx& c, unsigned* cnt, int n, const double* t, double* W, int ldw, Ctl* ctl,
                  double* beta_arr);
void rw_nr_beta_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, int ldw,
                      Ctl* ctl, double* alpha_arr, const double* beta_arr);
void rw_nr_sub_alpha(Ctx& c, const Scratch& s, int n, double* t, const double* W, int ldw, Ctl* ctl);
// W[:, col0 + q] = U[:, idx[q]] (idx null: U[:, q]), U column-major with leading dimension ldu
void rw_put_cols(Ctx& c, int n, double* W, int ldw, int col0, int cnt, const double* U, long ldu,
                 const int* idx_dev);
// dst (column-major, ld n) = W[:, col0 .. col0 + cnt)
void rw_get_cols(Ctx& c, int n, const double* W, int ldw, int col0, int cnt, double* dst);
void rw_col_move(Ctx& c, int n, double* W, int ldw, int from, int to);

// t -= Q (Q^T t) with a host-side column count (project_x, eigensolvers.hpp:223-227).
void project_out(Ctx& c, const Scratch& s, int n, int kq, const double* Q, double* t,
                 double* coef);
// beta = after; breakdown -> halted; else W[:, i+1] = t * (1/beta), beta_arr[i] = beta, i++.
void normalize_next(Ctx& c, const Scratch& s, int n, const double* t, double* W, Ctl* ctl,
                    double* beta_arr);
// Dense fp64 contraction on the tensor cores (DMMA), C (M x N, column-major, ldc) = A B with
// B[k + col ldb] and A[row lda + k] (a_kcontig: the row-major Krylov basis, or X^T of a
// column-major X with lda = its leading dimension) or A[row + k lda] (a column-major block).
// Rayleigh-Ritz combinations U = W Y (eigensolvers.hpp:275-283), thick-restart vectors, the
// subspace-iteration Gram / rotation products and the deflation-set Gram (ritz_gemm.cu).
void ritz_gemm(Ctx& c, int M, int N, int K, const double* A, long lda, bool a_kcontig,
               const double* B, long ldb, double* C, long ldc);
// Candidate statistics (eigensolvers.hpp:289-316) per column of U (n x nc) and AU:
// out3[3j..] = (lambda, residual, uu).  U is left unscaled (raw W y, kept for thick restart).
void candidate_stats(Ctx& c, int n, int nc, double* U, const double* AU, double* out3,
                     const double* w = nullptr);
// Chebyshev filter degree on a precomputed product sx = S x (pencils; filter_poly.hpp:261-276).
void cheb_combine(Ctx& c, int n, bool first, const double* sx, const double* x, const double* prev,
                  double* y, double* out, double cc, double invd, double mu0, double muj,
                  const Ctl* halt);
// Pencil candidate statistics: out3[3j..] = (x.Ax / x.Bx, ||Ax - lambda Bx|| / sqrt(x.Bx), u.u).
void pencil_stats(Ctx& c, int n, int nc, const double* U, const double* X, const double* AX,
                  const double* BX, double* out3);
// X[:, j] /= sqrt(X[:, j] . BX[:, j]).
void b_normalize(Ctx& c, int n, int nc, double* X, const double* BX);
void dot_dev(Ctx& c, const Scratch& s, int n, const double* x, const double* y, double* result_dev);
void scale(Ctx& c, int n, double a, double* x);
// dst = a * src (n doubles).
void scale_copy(Ctx& c, int n, double a, const double* src, double* dst);
// Device-time stamps: which 0 = filter start, 1 = filter end / orth start, 2 = orth end.
void stamp(Ctx& c, Ctl* ctl, int which);

}  // namespace k
}  // namespace se

namespace se {
namespace k {
// Eigenvalues >= bar of the symmetric tridiagonal (d[m], e[m-1]) by device Sturm bisection
// (stagnation checks, eigensolvers.hpp:436-444 / 562-572).  work: >= 4m + 8 device doubles.
void tridiag_eigs_above(Ctx& c, int m, const double* d_host, const double* e_host, double bar,
                        double* work, std::vector<double>& out);
}  // namespace k
}  // namespace se
