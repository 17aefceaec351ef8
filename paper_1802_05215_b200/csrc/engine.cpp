// Device Lanczos engine (see engine.hpp).  Reference: lanczos.hpp:37-277 and
// eigensolvers.hpp:142-732 under /root/reference/proj/include/sliceeig/.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>

namespace se {

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int grow(int want) { return std::max(want, 16) + std::max(want, 16) / 2; }
// Allocations above this size grow to the exact request instead of 1.5x (n ~ 2M: 16 MB a
// column, so a 1.5x basis, locked set or candidate block would not fit next to the others).
constexpr size_t kBigAlloc = (size_t)4 << 30;
int grow_for(int n, int want) { return (size_t)n * want * 8 > kBigAlloc ? want : grow(want); }

// ---- the Krylov basis: row-major (rowgs.cu) ----------------------------------------------------
// W[r * ld + j], ld = rw_ldw(cap): each row of the active basis is one contiguous run, which is
// what lets the CGS2 step stage row blocks by TMA bulk copies and read W three times per step.
struct RowBasis {
  int n = 0;
  int cap = 0;  // columns
  int ld = 0;
  double* p = nullptr;
};

void rowbasis_reserve(Ctx& c, RowBasis& w, int n, int cols, bool keep) {
  if (w.p && w.n == n && w.cap >= cols) return;
  const int ld = k::rw_ldw(cols);
  double* p = dev_alloc<double>((size_t)n * ld);
  // zero once: the CGS2 kernels read whole column pairs, so a never-written pad column must
  // hold a finite value (it is multiplied by a zero coefficient)
  SE_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)n * ld, c.stream));
  if (keep && w.p && w.cap > 0)  // re-stride the kept rows
    SE_CUDA(cudaMemcpy2DAsync(p, sizeof(double) * ld, w.p, sizeof(double) * w.ld,
                              sizeof(double) * w.ld, n, cudaMemcpyDeviceToDevice, c.stream));
  if (w.p) {
    ctx_sync(c);
    dev_free(w.p);
  }
  w.p = p;
  w.n = n;
  w.cap = cols;
  w.ld = ld;
}

// ---- one device recurrence (basis W, locked set L, step graph) ------------------------------
struct Krylov {
  Ctx& c;
  const DevCsr& A;
  const StepOp& op;
  const Pencil* pen;
  int n;
  double* pb[3] = {nullptr, nullptr, nullptr};  // pencil: the P-series recurrence buffers
  double *s1 = nullptr, *s2 = nullptr, *sx = nullptr;  // P x, A P x, S x
  RowBasis W;
  DevMat L;
  double* t = nullptr;
  double* vsrc = nullptr;  // the step's source column W[:, i], contiguous (filter input)
  double* fb[3] = {nullptr, nullptr, nullptr};
  Ctl* ctl = nullptr;
  double *alpha = nullptr, *beta = nullptr, *hdiag = nullptr, *coef = nullptr, *coef2 = nullptr,
         *coef_l = nullptr;
  double* dscal = nullptr;  // device scalars for host-side dots
  int arr_cap = 0, coefl_cap = 0;
  k::Scratch s;
  k::RowScratch rs;
  double* rbuf = nullptr;
  int* idx = nullptr;  // column indices for thick-restart copies
  int idx_cap = 0;
  // one captured step graph per (mode, CGS2 geometry class of the step's column count)
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    int nodes = 0;
  };
  std::map<std::pair<int, int>, StepGraph> graphs;
  int host_i = 0;  // the column the next step filters (host mirror of ctl->i)
  int nlock = 0;

  double* mu_dev = nullptr;
  void* res_state = nullptr;  // resident filter: tile-exchange buffers + tag epoch

  Krylov(Ctx& cc, const DevCsr& a, const StepOp& o, const Pencil* p = nullptr)
      : c(cc), A(a), op(o), pen(p), n(a.n) {
    t = dev_alloc<double>(n);
    vsrc = dev_alloc<double>(n);
    if (pen) {
      for (double*& b : pb) b = dev_alloc<double>(n);
      s1 = dev_alloc<double>(n);
      s2 = dev_alloc<double>(n);
      sx = dev_alloc<double>(n);
    }
    if (!op.plain) {
      for (double*& b : fb) b = dev_alloc<double>(n);
      mu_dev = dev_alloc<double>(op.k + 1);
      h2d(c, mu_dev, op.mu.data(), sizeof(double) * (op.k + 1));
      if (!pen && k::resident_tiles(A) > 0) {  // the whole filter in one launch (resident.cu)
        res_state = dev_alloc<char>(k::resident_state_bytes(A));
        SE_CUDA(cudaMemsetAsync(res_state, 0, k::resident_state_bytes(A), c.stream));
      }
    }
    ctl = dev_alloc<Ctl>(1);
    dscal = dev_alloc<double>(4);
    Ctl z{};
    h2d(c, ctl, &z, sizeof(Ctl));
  }
  ~Krylov() {
    cudaStreamSynchronize(c.stream);
    for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
    dev_free(W.p);
    devmat_free(L);
    dev_free(mu_dev);
    dev_free(res_state);
    for (void* p : {(void*)pb[0], (void*)pb[1], (void*)pb[2], (void*)s1, (void*)s2, (void*)sx})
      dev_free(p);
    for (void* p : {(void*)t, (void*)vsrc, (void*)fb[0], (void*)fb[1], (void*)fb[2], (void*)ctl,
                    (void*)alpha, (void*)beta, (void*)hdiag, (void*)coef, (void*)coef2,
                    (void*)coef_l, (void*)dscal, (void*)s.buf, (void*)s.cnt, (void*)rbuf,
                    (void*)idx})
      dev_free(p);
  }

  // End of the recurrence: the step graphs and the basis are released (the locked set stays).
  void release_basis() {
    drop_graph();
    ctx_sync(c);
    dev_free(W.p);
    W = RowBasis{};
  }

  void drop_graph() {
    if (!graphs.empty()) ctx_sync(c);
    for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
    graphs.clear();
  }

  // Locked-set capacity of exactly `cols` columns (large problems size it from the DOS estimate
  // up front instead of growing by 1.5x).
  void reserve_locked(int cols) {
    if (cols <= L.cap) return;
    devmat_reserve(c, L, n, cols, true);
    drop_graph();
    ensure(W.cap, cols);
  }

  // Capacity for `wcols` basis columns and `lcols` locked columns; pointers baked into the step
  // graph change only here (then the graph is re-captured).
  void ensure(int wcols, int lcols) {
    bool dirty = false;
    if (wcols > W.cap) {
      rowbasis_reserve(c, W, n, grow_for(n, wcols), true);
      dirty = true;
    }
    if (lcols > L.cap) {
      devmat_reserve(c, L, n, grow_for(n, lcols), true);
      dirty = true;
    }
    if (W.ld > arr_cap) {
      ctx_sync(c);
      auto regrow = [&](double*& p) {
        double* q = dev_alloc<double>(W.ld);
        SE_CUDA(cudaMemsetAsync(q, 0, sizeof(double) * W.ld, c.stream));
        if (p) SE_CUDA(cudaMemcpyAsync(q, p, sizeof(double) * arr_cap, cudaMemcpyDeviceToDevice, c.stream));
        ctx_sync(c);
        dev_free(p);
        p = q;
      };
      regrow(alpha);
      regrow(beta);
      regrow(hdiag);
      regrow(coef);
      regrow(coef2);
      arr_cap = W.ld;
      // streaming grid and partials of the row-major CGS2 for this capacity
      rs = k::rw_scratch(c, W.ld);
      dev_free(rbuf);
      rbuf = dev_alloc<double>(k::rw_scratch_doubles(rs));
      k::rw_bind(rs, rbuf);
      dirty = true;
    }
    if (std::max(L.cap, 1) > coefl_cap) {
      dev_free(coef_l);
      coefl_cap = std::max(L.cap, 1);
      coef_l = dev_alloc<double>(coefl_cap);
      dirty = true;
    }
    const int wide = std::max(L.cap, 1);
    const size_t need = k::cgs_scratch_doubles(c, n, wide);
    const int slots = k::cgs_counter_slots(n, wide);
    if (need > s.cap || slots > s.ncnt) {
      ctx_sync(c);
      dev_free(s.buf);
      dev_free(s.cnt);
      s.cap = need + need / 2;
      s.ncnt = slots + slots / 2;
      s.buf = dev_alloc<double>(s.cap);
      s.cnt = dev_alloc<unsigned>(s.ncnt);
      SE_CUDA(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned) * s.ncnt, c.stream));
      dirty = true;
    }
    if (dirty) drop_graph();
  }

  Ctl get() {
    Ctl h;
    d2h(c, &h, ctl, sizeof(Ctl));
    ctx_sync(c);
    return h;
  }
  void put(const Ctl& h) {
    h2d(c, ctl, &h, sizeof(Ctl));
    ctx_sync(c);
  }
  void begin(int i0) {  // new recurrence segment starting at column i0
    host_i = i0;
    Ctl h = get();
    h.i = i0;
    h.halted = 0;
    h.nlock = nlock;
    put(h);
  }

  // Basis column access for the host-driven phases (start vectors, restarts, downloads).
  void put_col(int col, const double* dev_src) { k::rw_put_cols(c, n, W.p, W.ld, col, 1, dev_src, n, nullptr); }
  void get_col(int col, double* dev_dst) { k::rw_get_cols(c, n, W.p, W.ld, col, 1, dev_dst); }
  // W[:, q] = U[:, cols[q]] for q < cols.size() (U column-major, ld n)
  void put_cols(const std::vector<int>& cols, const double* U) {
    if (cols.empty()) return;
    if ((int)cols.size() > idx_cap) {
      ctx_sync(c);
      dev_free(idx);
      idx_cap = grow((int)cols.size());
      idx = dev_alloc<int>(idx_cap);
    }
    h2d(c, idx, cols.data(), sizeof(int) * cols.size());
    k::rw_put_cols(c, n, W.p, W.ld, 0, (int)cols.size(), U, n, idx);
  }

  // out = sum_j op.mu[j] T_j((M - c I) / d) x by the fused SpMV recurrence on matrix M, with
  // buffers buf[3] (apply_pol filter_poly.hpp:256-277; apply_cheb cheb_approx.hpp:91-112 for
  // the pencil series, whose map multiplies by 1/h instead of dividing).
  void record_series(const DevCsr& M, const StepOp& sop, const double* x, double* out,
                     double* const* buf) {
    k::ChebArgs a;
    a.halt = ctl;
    a.c = sop.c;
    a.invd = sop.invd;
    a.x = x;
    a.y = buf[0];
    a.out = out;
    a.mu0 = sop.mu[0];
    a.muj = sop.mu[1];
    k::spmv_cheb(c, M, k::kFirst, a);
    // buffers: prev (j-2), cur (j-1), next; x plays prev for j = 2
    int cur = 0, prv = -1, nxt = 1;
    for (int j = 2; j <= sop.k; ++j) {
      k::ChebArgs b = a;
      b.x = buf[cur];
      b.prev = prv < 0 ? x : buf[prv];
      b.y = buf[nxt];
      b.muj = sop.mu[j];
      k::spmv_cheb(c, M, k::kNext, b);
      const int old_prv = prv < 0 ? 2 : prv;
      prv = cur;
      cur = nxt;
      nxt = old_prv;
    }
  }

  // y = S x = P A P x (pencil)
  void record_apply_s(const double* x, double* y) {
    record_series(*pen->B, pen->P, x, s1, pb);
    k::ChebArgs a;
    a.halt = ctl;
    a.x = s1;
    a.y = s2;
    k::spmv_cheb(c, A, k::kPlain, a);
    record_series(*pen->B, pen->P, s2, y, pb);
  }

  // Filter W[:, ctl->i] into t (apply_pol filter_poly.hpp:256-277, or one op application).
  void record_filter() {
    k::rw_col_get(c, n, W.p, W.ld, ctl, 0, vsrc);
    if (pen) {  // composite operator: each degree is S x, then the recurrence update
      if (op.plain) {
        record_apply_s(vsrc, t);
        return;
      }
      record_apply_s(vsrc, sx);
      k::cheb_combine(c, n, true, sx, vsrc, nullptr, fb[0], t, op.c, op.invd, op.mu[0], op.mu[1], ctl);
      int cur = 0, prv = -1, nxt = 1;
      for (int j = 2; j <= op.k; ++j) {
        record_apply_s(fb[cur], sx);
        k::cheb_combine(c, n, false, sx, fb[cur], prv < 0 ? vsrc : fb[prv], fb[nxt], t, op.c,
                        op.invd, 0.0, op.mu[j], ctl);
        const int old_prv = prv < 0 ? 2 : prv;
        prv = cur;
        cur = nxt;
        nxt = old_prv;
      }
      return;
    }
    if (op.plain) {
      k::ChebArgs a;
      a.halt = ctl;
      a.x = vsrc;
      a.y = t;
      k::spmv_cheb(c, A, k::kPlain, a);
      return;
    }
    if (res_state)
      k::cheb_resident(c, A, op.k, mu_dev, op.c, op.invd, vsrc, t, res_state, ctl);
    else
      record_series(A, op, vsrc, t, fb);
  }

  // One Lanczos step.  mode 0: NR recurrence (eigensolvers.hpp:406-433 / lanczos.hpp:151-185);
  // mode 1: TR projection with h accumulation (eigensolvers.hpp:524-556 / lanczos.hpp:284-311).
  void record_step(int mode, int cls) {
    k::stamp(c, ctl, 0);
    record_filter();
    k::stamp(c, ctl, 1);
    if (L.cap > 0) k::cgs_pass(c, s, n, t, L.p, true, false, ctl, nullptr, coef_l, L.cap);
    if (mode == 0) {
      k::rw_nr_beta_alpha(c, s, n, t, W.p, W.ld, ctl, alpha, beta);
      k::rw_nr_sub_alpha(c, s, n, t, W.p, W.ld, ctl);
    }
    // CGS2 against W[:, 0..i] with three reads of W (TR: the T1 pass also takes ||t||)
    k::rw_cgs2(c, rs, n, t, W.p, W.ld, ctl, mode == 1 ? hdiag : nullptr, coef, coef2, mode == 1,
               cls);
    k::rw_normalize(c, s.cnt, n, t, W.p, W.ld, ctl, beta);
    k::stamp(c, ctl, 2);
  }

  StepGraph& graph(int mode, int cls) {
    StepGraph& g = graphs[{mode, cls}];
    if (g.exec) return g;
    const long before = c.launches;
    SE_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      record_step(mode, cls);
    } catch (...) {
      cudaGraph_t gr;
      cudaStreamEndCapture(c.stream, &gr);
      if (gr) cudaGraphDestroy(gr);
      graphs.erase({mode, cls});
      throw;
    }
    cudaGraph_t gr;
    SE_CUDA(cudaStreamEndCapture(c.stream, &gr));
    SE_CUDA(cudaGraphInstantiate(&g.exec, gr, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(gr);
    g.nodes = (int)(c.launches - before);
    c.launches = before;
    return g;
  }

  // `count` Lanczos steps from host_i on: each replays the graph of its column count's CGS2
  // geometry class (the step at column i orthogonalises against i + 1 columns; a halted
  // recurrence makes the remaining replays no-ops)
  void run(int mode, int count) {
    for (int q = 0; q < count;) {
      const int cls = k::rw_class(std::min(host_i + q + 1, W.cap));
      int span = 1;
      while (q + span < count && k::rw_class(std::min(host_i + q + span + 1, W.cap)) == cls) ++span;
      StepGraph& g = graph(mode, cls);
      for (int r = 0; r < span; ++r) SE_CUDA(cudaGraphLaunch(g.exec, c.stream));
      c.launches += (long)g.nodes * span;
      q += span;
    }
    host_i += count;
  }

  double dot(const double* x, const double* y) {
    k::dot_dev(c, s, n, x, y, dscal);
    double h = 0.0;
    d2h(c, &h, dscal, sizeof(double));
    ctx_sync(c);
    return h;
  }

  void download(const double* d, int count, Vec& out, int offset = 0) {
    out.resize(count);
    if (count <= 0) return;
    d2h(c, out.data(), d + offset, sizeof(double) * count);
    ctx_sync(c);
  }
};

// ---- projected eigenproblems ------------------------------------------------------------------
// Dense symmetric eigen-decomposition with vectors left on the device (column j <-> values[j],
// ascending).  Small problems run on the host (launch latency dominates); larger ones through
// cuSOLVER syevd (the reference's O(m^3) host Householder+QL, dense_eig.hpp:114-139).
struct DevEig {
  Ctx& c;
  double* dA = nullptr;
  double* dW = nullptr;
  double* work = nullptr;
  int* info = nullptr;
  int cap = 0;
  int lwork = 0;
  explicit DevEig(Ctx& cc) : c(cc) {}
  ~DevEig() {
    cudaStreamSynchronize(c.stream);
    for (void* p : {(void*)dA, (void*)dW, (void*)work, (void*)info}) dev_free(p);
  }
  // H: m x m column-major host.  Returns device pointer to eigenvectors (ld = m).
  const double* solve(int m, const Vec& H, Vec& values) {
    HiPrio hp(c);
    if (m > cap) {
      ctx_sync(c);
      dev_free(dA);
      dev_free(dW);
      dev_free(info);
      cap = grow(m);
      dA = dev_alloc<double>((size_t)cap * cap);
      dW = dev_alloc<double>(cap);
      info = dev_alloc<int>(1);
    }
    if (m <= 160) {
      Vec vecs;
      dense_sym_eig(m, H.data(), true, values, vecs);
      h2d(c, dA, vecs.data(), sizeof(double) * (size_t)m * m);
      ctx_sync(c);
      return dA;
    }
    h2d(c, dA, H.data(), sizeof(double) * (size_t)m * m);
    int lw = 0;
    if (cusolverDnDsyevd_bufferSize(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                    dA, m, dW, &lw) != CUSOLVER_STATUS_SUCCESS)
      fail(SE_ECUDA, "cusolverDnDsyevd_bufferSize failed");
    if (lw > lwork) {
      ctx_sync(c);
      dev_free(work);
      lwork = lw;
      work = dev_alloc<double>(lwork);
    }
    if (cusolverDnDsyevd(c.solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, dA, m, dW,
                         work, lwork, info) != CUSOLVER_STATUS_SUCCESS)
      fail(SE_ECUDA, "cusolverDnDsyevd failed");
    ++c.launches;
    int hinfo = 0;
    values.resize(m);
    d2h(c, values.data(), dW, sizeof(double) * m);
    d2h(c, &hinfo, info, sizeof(int));
    ctx_sync(c);
    if (hinfo != 0) fail(SE_ENUMERIC, "dense_sym_eig: syevd did not converge");
    return dA;
  }
};

// ---- candidate evaluation (eigensolvers.hpp:275-318) --------------------------------------------
// Candidate (Ritz vector) columns evaluated per chunk: U and A U for a chunk take at most the
// context's candidate budget (8 GB by default).
inline int cand_chunk(const Ctx& c, int n, int ncand) {
  const size_t cols = c.cand_budget / (16 * (size_t)std::max(n, 1));
  return std::max(1, (int)std::min<size_t>((size_t)ncand, std::max<size_t>(cols, 1)));
}

struct CandBuf {
  Ctx& c;
  const Pencil* pen = nullptr;
  DevMat U, AU, X, BX;
  double* stats = nullptr;
  int stats_cap = 0;
  explicit CandBuf(Ctx& cc, const Pencil* p = nullptr) : c(cc), pen(p) {}
  ~CandBuf() {
    cudaStreamSynchronize(c.stream);
    devmat_free(U);
    devmat_free(AU);
    devmat_free(X);
    devmat_free(BX);
    dev_free(stats);
  }
  void release() {
    cudaStreamSynchronize(c.stream);
    devmat_free(U);
    devmat_free(AU);
    devmat_free(X);
    devmat_free(BX);
  }
  // U = W[:, :steps] Y (Y steps x nc, ld ldy), AU = A U, stats per column.  W is column-major
  // (ld n) when w_row_ld == 0, else the row-major Krylov basis with row stride w_row_ld.
  void eval(const DevCsr& A, const double* W, int steps, const double* Y, int ldy, int nc,
            Vec& out3, int w_row_ld = 0) {
    HiPrio hp(c);
    const int n = A.n;
    // geometric growth: every reallocation is a cudaFree, which waits for the whole device
    // (the other slices' queued work included)
    const int want = (size_t)n * nc * 8 > kBigAlloc ? nc : grow(nc);
    if (nc > U.cap || U.n != n) devmat_reserve(c, U, n, want, false);
    if (nc > AU.cap || AU.n != n) devmat_reserve(c, AU, n, want, false);
    if (nc > stats_cap) {
      dev_free(stats);
      stats_cap = grow(nc);
      stats = dev_alloc<double>(3 * (size_t)stats_cap);
    }
    // U = W Y on the fp64 tensor cores (ritz_gemm.cu): W row-major (row stride w_row_ld) or
    // column-major (ld n)
    if (w_row_ld)
      k::ritz_gemm(c, n, nc, steps, W, w_row_ld, true, Y, ldy, U.p, n);
    else
      k::ritz_gemm(c, n, nc, steps, W, n, false, Y, ldy, U.p, n);
    auto spmv_cols = [&](const DevCsr& M, const double* x, double* y) {
      for (int q0 = 0; q0 < nc; q0 += 65535) {
        k::ChebArgs a;
        a.x = x + (size_t)q0 * n;
        a.y = y + (size_t)q0 * n;
        a.ncols = std::min(65535, nc - q0);
        k::spmv_cheb(c, M, k::kPlain, a);
      }
    };
    if (pen) {  // x = P u, A x, B x: the reference's B-weighted Rayleigh quotient and residual
      if (nc > X.cap || X.n != n) devmat_reserve(c, X, n, want, false);
      if (nc > BX.cap || BX.n != n) devmat_reserve(c, BX, n, want, false);
      apply_filter_block(c, *pen->B, pen->P, nc, U.p, X.p);
      spmv_cols(A, X.p, AU.p);
      spmv_cols(*pen->B, X.p, BX.p);
      k::pencil_stats(c, n, nc, U.p, X.p, AU.p, BX.p, stats);
    } else {
      spmv_cols(A, U.p, AU.p);
      k::candidate_stats(c, n, nc, U.p, AU.p, stats, A.resw);
    }
    out3.resize(3 * (size_t)nc);
    d2h(c, out3.data(), stats, sizeof(double) * 3 * nc);
    ctx_sync(c);
  }
};

// ---- slice state (SliceSolve eigensolvers.hpp:155-346) -----------------------------------------
struct Slice {
  Ctx& c;
  const DevCsr& A;
  SolverCfg cfg;
  double bar, xi, eta;
  Rng rng;
  se_counters cnt{};
  double prof[4] = {0, 0, 0, 0};  // host seconds: stagnation checks, projected eig, candidates
  Vec lock_val, lock_res;
  int preloaded = 0;
  StepOp op;
  Krylov kr;
  DevEig eig;
  CandBuf cand;

  const Pencil* pen;
  Slice(Ctx& cc, const DevCsr& a, const PolyFilter& f, double xi_, double eta_,
        const SolverCfg& cf, const Pencil* p = nullptr)
      : c(cc), A(a), cfg(cf), bar(f.bar), xi(xi_), eta(eta_), rng(cf.seed), op(make_op(f)),
        kr(cc, a, op, p), eig(cc), cand(cc, p), pen(p) {}

  static StepOp make_op(const PolyFilter& f) {
    StepOp o;
    o.plain = false;
    o.k = f.k;
    o.mu = f.mu;
    o.c = f.c;
    o.invd = 1.0 / f.d;
    return o;
  }

  double bar_eff() const { return bar * (1.0 - 1e-4); }

  // Ritz values >= bar of a tridiagonal projected matrix (ascending), for tnew.
  double* chk_work = nullptr;
  int chk_cap = 0;
  void check_eigs(const Vec& d, const Vec& e, Vec& vals) {
    const int m = (int)d.size();
    if (m <= 64) {  // tiny: host QL (values only)
      Vec all, unused;
      sym_tridiag_eig(d, e, false, all, unused);
      vals.clear();
      for (double v : all)
        if (v >= bar) vals.push_back(v);
      return;
    }
    if (m > chk_cap) {
      ctx_sync(c);
      dev_free(chk_work);
      chk_cap = grow(m);
      chk_work = dev_alloc<double>(4 * (size_t)chk_cap + 8);
    }
    HiPrio hp(c);
    k::tridiag_eigs_above(c, m, d.data(), e.data(), bar, chk_work, vals);
  }
  ~Slice() {
    dev_free(chk_work);
    devmat_free(trbuf);
  }
  double stagnation_tol(double tnew) const {
    return cfg.tau1 > 0.0 ? cfg.tau1 : std::max(1e-12, 1e-10 * std::abs(tnew));
  }
  bool in_slice(double lam) const {
    const double slo = 10.0 * cfg.res_tol * std::max(1.0, std::abs(xi));
    const double shi = 10.0 * cfg.res_tol * std::max(1.0, std::abs(eta));
    return lam >= xi - slo && lam <= eta + shi;
  }
  bool converged(double lam, double r) const { return r <= cfg.res_tol * std::max(1.0, std::abs(lam)); }

  // start_pair (eigensolvers.hpp:231-261), standard problem: W[:, col].
  void start_vector(int col) {
    const int n = A.n;
    Vec w(n);
    for (int attempt = 0; attempt < 16; ++attempt) {
      rng.normal_fill(w.data(), n);
      double* d = kr.t;  // staged contiguous, then stored into the row-major basis
      h2d(c, d, w.data(), sizeof(double) * n);
      if (kr.nlock > 0) k::project_out(c, kr.s, n, kr.nlock, kr.L.p, d, kr.coef_l);
      const double nb = std::sqrt(kr.dot(d, d));
      if (nb > 1e-14) {
        k::scale(c, n, 1.0 / nb, d);
        kr.put_col(col, d);
        return;
      }
    }
    fail(SE_ENUMERIC, "eigensolver: could not draw a start vector outside the locked set");
  }

  void lock(const double* u_raw, double uu, double lam, double res) {
    if (kr.nlock + 1 > kr.L.cap && (size_t)A.n * (kr.nlock + 1) * 8 > kBigAlloc)
      kr.reserve_locked(kr.nlock + 1 + std::max(64, kr.nlock / 8));  // +12.5%, not +50%
    kr.ensure(kr.W.cap, kr.nlock + 1);
    k::scale_copy(c, A.n, 1.0 / std::sqrt(uu), u_raw, kr.L.col(kr.nlock));
    ++kr.nlock;
    lock_val.push_back(lam);
    lock_res.push_back(res);
  }

  void preload(int ndefl, const double* u, const double* vals, const char* who) {
    if (ndefl <= 0) return;
    const int n = A.n;
    kr.ensure(std::max(kr.W.cap, 1), ndefl);
    HiPrio hp(c);
    h2d(c, kr.L.p, u, sizeof(double) * (size_t)n * ndefl);
    double* G = dev_alloc<double>((size_t)ndefl * ndefl);
    k::ritz_gemm(c, ndefl, ndefl, n, kr.L.p, n, true, kr.L.p, n, G, ndefl);  // L^T L
    Vec g((size_t)ndefl * ndefl);
    d2h(c, g.data(), G, sizeof(double) * g.size());
    ctx_sync(c);
    dev_free(G);
    for (int j = 0; j < ndefl; ++j)
      for (int i = 0; i <= j; ++i)
        if (std::abs(g[(size_t)j * ndefl + i] - (i == j ? 1.0 : 0.0)) > 1e-10)
          fail(SE_EINVAL, std::string(who) + ": deflation set is not (B-)orthonormal to 1e-10");
    kr.nlock = ndefl;
    preloaded = ndefl;
    lock_val.assign(vals, vals + ndefl);
    lock_res.assign(ndefl, 0.0);
  }

  void add_timers() {
    const Ctl h = kr.get();
    cnt.t_mv = h.t_mv_ns * 1e-9;
    cnt.t_orth = h.t_orth_ns * 1e-9;
  }

  // Everything locked past the preload, ascending (eigensolvers.hpp:328-345).
  std::unique_ptr<SliceResult> results(long its, bool warn, double t0) {
    auto r = std::make_unique<SliceResult>();
    const int k = kr.nlock - preloaded;
    std::vector<int> idx(k);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(),
              [&](int i, int j) { return lock_val[preloaded + i] < lock_val[preloaded + j]; });
    r->n = A.n;
    for (int q = 0; q < k; ++q) {
      r->eigenvalues.push_back(lock_val[preloaded + idx[q]]);
      r->residuals.push_back(lock_res[preloaded + idx[q]]);
    }
    // the recurrence is over: its basis, candidate and restart blocks go before the result is
    // formed (at n ~ 2M the locked set alone is 80+ GB and must not meet a second copy of itself)
    kr.release_basis();
    cand.release();
    devmat_free(trbuf);
    if (preloaded == 0 && k > 0) {
      // the locked set becomes the result: columns permuted in place into ascending order
      // (cycle by cycle through one staging column), then the buffer changes owner
      std::vector<char> done(k, 0);
      const size_t colb = sizeof(double) * (size_t)A.n;
      for (int s0 = 0; s0 < k; ++s0) {
        if (done[s0] || idx[s0] == s0) {
          done[s0] = 1;
          continue;
        }
        SE_CUDA(cudaMemcpyAsync(kr.t, kr.L.col(s0), colb, cudaMemcpyDeviceToDevice, c.stream));
        int j = s0;
        while (idx[j] != s0) {
          SE_CUDA(cudaMemcpyAsync(kr.L.col(j), kr.L.col(idx[j]), colb, cudaMemcpyDeviceToDevice,
                                  c.stream));
          done[j] = 1;
          j = idx[j];
        }
        SE_CUDA(cudaMemcpyAsync(kr.L.col(j), kr.t, colb, cudaMemcpyDeviceToDevice, c.stream));
        done[j] = 1;
      }
      ctx_sync(c);
      r->vectors = kr.L;
      kr.L = DevMat{};
    } else {
      if (k > 0) devmat_reserve(c, r->vectors, A.n, k, false);
      for (int q = 0; q < k; ++q)
        SE_CUDA(cudaMemcpyAsync(r->vectors.col(q), kr.L.col(preloaded + idx[q]),
                                sizeof(double) * A.n, cudaMemcpyDeviceToDevice, c.stream));
      ctx_sync(c);
    }
    if (pen && k > 0) {  // eigenvectors of the pencil: x = P y, B-normalised
      DevMat X, BX;
      devmat_reserve(c, X, A.n, k, false);
      devmat_reserve(c, BX, A.n, k, false);
      apply_filter_block(c, *pen->B, pen->P, k, r->vectors.p, X.p);
      for (int q0 = 0; q0 < k; q0 += 65535) {
        k::ChebArgs a;
        a.x = X.col(q0);
        a.y = BX.col(q0);
        a.ncols = std::min(65535, k - q0);
        k::spmv_cheb(c, *pen->B, k::kPlain, a);
      }
      k::b_normalize(c, A.n, k, X.p, BX.p);
      SE_CUDA(cudaMemcpyAsync(r->vectors.p, X.p, sizeof(double) * (size_t)A.n * k,
                              cudaMemcpyDeviceToDevice, c.stream));
      ctx_sync(c);
      devmat_free(X);
      devmat_free(BX);
    }
    add_timers();
    cnt.t_total += now_s() - t0;
    if (std::getenv("SE_PROFILE"))
      std::fprintf(stderr,
                   "[se] n=%d its=%ld total %.3f mv %.3f orth %.3f check %.3f eig %.3f cand %.3f "
                   "passes %lld cols %lld (%.1f GB/s over t_orth) check_kernel_ms %.1f wcap %d fused %d frees %ld chk %.2f/%.2f/%.2f\n",
                   A.n, its, cnt.t_total, cnt.t_mv, cnt.t_orth, prof[0], prof[1], prof[2],
                   kr.get().passes_total, kr.get().cols_total,
                   16.0 * A.n * (double)kr.get().cols_total / std::max(1e-9, cnt.t_orth) / 1e9, c.prof_kernel_ms, kr.W.cap, 0, dev_frees().load(),
                   c.prof_chk[0], c.prof_chk[1], c.prof_chk[2]);
    r->niter = its;
    r->hit_max_its = warn;
    r->counters = cnt;
    const Ctl hc = kr.get();
    r->orth_passes = hc.passes_total;
    r->orth_cols = hc.cols_total;
    // bytes the CGS2 steps moved: every streamed basis column (8 n each: T1 + MID + N2 reads)
    // plus the vector traffic (T1 reads t, MID and N2 read and write it: 8 + 16 + 16 n)
    r->orth_bytes = 8.0 * A.n * (double)hc.reads_cols + 40.0 * A.n * (double)hc.passes_total;
    return r;
  }

  // Kept Ritz vectors of a thick restart recomputed into trbuf: trbuf[:, q] = W Y[:, j0 + cols[q]]
  // (row-major W), for when the candidates were evaluated in chunks.
  DevMat trbuf;
  void stage_ritz(const double* W, int ldw, int steps, const double* Y, int j0,
                  const std::vector<int>& cols) {
    HiPrio hp(c);
    const int n = A.n, k = (int)cols.size();
    if (k > trbuf.cap || trbuf.n != n) devmat_reserve(c, trbuf, n, k, false);
    Vec ysel((size_t)steps * k);
    for (int q = 0; q < k; ++q) {
      d2h(c, ysel.data() + (size_t)q * steps, Y + (size_t)(j0 + cols[q]) * steps, sizeof(double) * steps);
    }
    ctx_sync(c);
    double* dy = dev_alloc<double>(ysel.size());
    h2d(c, dy, ysel.data(), sizeof(double) * ysel.size());
    k::ritz_gemm(c, n, k, steps, W, ldw, true, dy, steps, trbuf.p, n);
    ctx_sync(c);
    dev_free(dy);
  }

  // Candidate rows ylast for thick restart: Y[steps-1, j] for the candidate columns.
  Vec last_row(const double* Y, int steps, int j0, int nc) {
    HiPrio hp(c);
    Vec out(nc);
    if (nc == 0) return out;
    double* p = static_cast<double*>(staging(c, sizeof(double) * nc));
    SE_CUDA(cudaMemcpy2DAsync(p, sizeof(double), Y + (size_t)j0 * steps + (steps - 1),
                              sizeof(double) * steps, sizeof(double), nc, cudaMemcpyDeviceToHost,
                              c.stream));
    ctx_sync(c);
    std::copy(p, p + nc, out.data());
    return out;
  }
};

double sum_above(const Vec& vals, double bar) {
  double s = 0.0;
  for (double th : vals)
    if (th >= bar) s += th;
  return s;
}

// ---- run_nr (eigensolvers.hpp:385-472) -----------------------------------------------------------
std::unique_ptr<SliceResult> run_nr(Slice& s) {
  const double t0 = now_s();
  const int n = s.A.n;
  const long budget = std::min<long>(s.cfg.max_its, n);
  Krylov& kr = s.kr;
  const int nc = s.cfg.ncycle;
  kr.ensure((int)std::min<long>(budget + 1, 2 * nc + 2), std::max(kr.nlock, 0));
  s.start_vector(0);
  kr.begin(0);
  double told = std::numeric_limits<double>::quiet_NaN();
  bool stagnant = false;
  long its = 0;
  while (true) {
    // advance to the next check point (its % ncycle == 0) or the budget
    const long target = std::min(budget, (its / nc + 1) * (long)nc);
    kr.ensure((int)target + 1, kr.nlock);
    kr.run(0, (int)(target - its));
    const Ctl h = kr.get();
    bool breakdown = false;
    if (h.halted) {
      breakdown = true;
      its = h.i + 1;
    } else {
      its = target;
    }
    const bool last = breakdown || its >= budget;
    if (its % nc == 0 || last) {
      Vec al, be;
      kr.download(kr.alpha, (int)its, al);
      kr.download(kr.beta, (int)its - 1, be);
      if (!stagnant && !last) {
        Vec vals, vecs;
        const double tq = now_s();
        s.check_eigs(al, be, vals);
        s.prof[0] += now_s() - tq;
        const double tnew = sum_above(vals, s.bar);
        if (!std::isnan(told) && std::abs(tnew - told) < s.stagnation_tol(tnew)) stagnant = true;
        told = tnew;
      }
      if (stagnant || last) {
        const int m = (int)its;
        Vec H((size_t)m * m, 0.0);
        for (int i = 0; i < m; ++i) H[(size_t)i * m + i] = al[i];
        for (int i = 0; i + 1 < m; ++i) H[(size_t)i * m + i + 1] = H[(size_t)(i + 1) * m + i] = be[i];
        Vec vals;
        double tq = now_s();
        const double* Y = s.eig.solve(m, H, vals);
        s.prof[1] += now_s() - tq;
        int j0 = m;
        while (j0 > 0 && vals[j0 - 1] >= s.bar_eff()) --j0;
        const int ncand = m - j0;
        Vec st;
        tq = now_s();
        if (ncand > 0) s.cand.eval(s.A, kr.W.p, m, Y + (size_t)j0 * m, m, ncand, st, kr.W.ld);
        s.prof[2] += now_s() - tq;
        s.cnt.n_A_matvec += ncand;
        std::vector<int> accepted;
        bool pending = false;
        for (int q = ncand - 1; q >= 0; --q) {  // top-down, eigensolvers.hpp:449
          const double lam = st[3 * q], res = st[3 * q + 1], uu = st[3 * q + 2];
          if (!(uu > 0.0) || !s.in_slice(lam)) continue;
          if (s.converged(lam, res))
            accepted.push_back(q);
          else
            pending = true;
        }
        if (!pending || last) {
          for (int q : accepted) s.lock(s.cand.U.col(q), st[3 * q + 2], st[3 * q], st[3 * q + 1]);
          s.cnt.n_A_matvec += (long)s.op.k * its;
          return s.results(its, pending, t0);
        }
      }
    }
  }
}

// ---- run_tr (eigensolvers.hpp:481-628) -----------------------------------------------------------
std::unique_ptr<SliceResult> run_tr(Slice& s) {
  const double t0 = now_s();
  const int n = s.A.n;
  const int m = std::min(s.cfg.m, n);
  const long budget = s.cfg.max_its;
  const int tr_cap = std::max(1, m / 2);
  const int ncyc = s.cfg.ncycle;
  Krylov& kr = s.kr;
  kr.ensure(m + 1, std::max(kr.nlock, 1));
  Vec tr_theta, tr_s;
  long its = 0;
  int empty_cycles = 0;
  bool warn = false;
  while (true) {
    const int l = (int)tr_theta.size();
    if (l == 0) s.start_vector(0);
    SE_CUDA(cudaMemsetAsync(kr.hdiag, 0, sizeof(double) * kr.arr_cap, s.c.stream));
    kr.begin(l);
    // arrowhead part of the projected matrix reduced once per cycle (checks are O(steps^2))
    Vec adiag, aoff;
    arrow_to_tridiag(tr_theta, tr_s, 0.0, adiag, aoff);
    int steps = l;
    bool broke = false;
    double trailing = 0.0;
    double told = std::numeric_limits<double>::quiet_NaN();
    int i = l;  // next step index
    while (i < m) {
      // next event: stagnation check after step i_c where (i_c + 1 - l) % ncycle == 0, the end
      // of the cycle, or the budget
      int stop = m;  // exclusive end step
      const int next_check = l + ((i - l) / ncyc + 1) * ncyc;
      if (next_check < m) stop = next_check;
      stop = (int)std::min<long>(stop, i + (budget - its));
      kr.run(1, stop - i);
      const Ctl h = kr.get();
      if (h.halted) {
        const int ib = h.i;  // breakdown at step ib
        its += ib - i + 1;
        steps = ib + 1;
        broke = true;
        trailing = 0.0;
        break;
      }
      its += stop - i;
      steps = stop;
      i = stop;
      Vec bl;
      kr.download(kr.beta, 1, bl, steps - 1);
      trailing = bl[0];
      if (its >= budget) break;
      if ((steps - l) % ncyc == 0 && steps < m) {
        Vec hd, be;
        kr.download(kr.hdiag, steps - l, hd, l);
        kr.download(kr.beta, steps - l - 1, be, l);
        Vec d(adiag.begin(), adiag.end()), e(aoff.begin(), aoff.end());
        d[l] = hd[0];
        for (int q = 1; q < steps - l; ++q) d.push_back(hd[q]);
        for (double b : be) e.push_back(b);
        Vec vals, unused;
        const double tq = now_s();
        s.check_eigs(d, e, vals);
        s.prof[0] += now_s() - tq;
        const double tnew = sum_above(vals, s.bar);
        if (!std::isnan(told) && std::abs(tnew - told) < s.stagnation_tol(tnew)) break;
        told = tnew;
      }
    }
    // projected matrix H[0:steps, 0:steps] (arrowhead + tridiagonal)
    Vec hd, be;
    kr.download(kr.hdiag, steps - l, hd, l);
    kr.download(kr.beta, std::max(steps - l - 1, 0), be, l);
    Vec H((size_t)steps * steps, 0.0);
    auto at = [&](int r, int cc) -> double& { return H[(size_t)cc * steps + r]; };
    for (int j = 0; j < l; ++j) {
      at(j, j) = tr_theta[j];
      at(j, l) = at(l, j) = tr_s[j];
    }
    for (int q = l; q < steps; ++q) at(q, q) = hd[q - l];
    for (int q = l; q + 1 < steps; ++q) at(q + 1, q) = at(q, q + 1) = be[q - l];
    Vec vals;
    double tq = now_s();
    const double* Y = s.eig.solve(steps, H, vals);
    s.prof[1] += now_s() - tq;
    int j0 = steps;
    while (j0 > 0 && vals[j0 - 1] >= s.bar_eff()) --j0;
    const int ncand = steps - j0;
    const Vec ylast = s.last_row(Y, steps, j0, ncand);
    struct TrC {
      double theta, ylast;
      int col;
    };
    std::vector<TrC> trset;
    int found = 0;
    // candidates top-down (eigensolvers.hpp:582-591), evaluated in column chunks so that U and
    // A U never hold more than ~8 GB (n ~ 2M); converged pairs lock as they are met
    const int chunk = cand_chunk(s.c, n, ncand);
    tq = now_s();
    for (int hi = ncand; hi > 0; hi -= chunk) {
      const int lo = std::max(0, hi - chunk);
      Vec st;
      s.cand.eval(s.A, kr.W.p, steps, Y + (size_t)(j0 + lo) * steps, steps, hi - lo, st, kr.W.ld);
      for (int q = hi - 1; q >= lo; --q) {
        const int u = q - lo;
        const double lam = st[3 * u], res = st[3 * u + 1], uu = st[3 * u + 2];
        if (!(uu > 0.0) || !s.in_slice(lam)) continue;
        ++found;
        if (s.converged(lam, res))
          s.lock(s.cand.U.col(u), uu, lam, res);
        else
          trset.push_back({vals[j0 + q], ylast[q], q});
      }
      // the locking copies read U on the Lanczos stream; the next chunk's evaluation rewrites U
      // on the high-priority stream, so they must have finished first
      if (lo > 0) ctx_sync(s.c);
    }
    s.prof[2] += now_s() - tq;
    s.cnt.n_A_matvec += ncand;
    if (std::getenv("SE_PROFILE"))
      std::fprintf(stderr, "[se] tr cycle: its %ld steps %d candidates %d in-slice %d locked %d kept %zu (%.1f s)\n",
                   its, steps, ncand, found, kr.nlock, trset.size(), now_s() - t0);
    if (found == 0) {
      if (++empty_cycles >= 2) break;
    } else {
      empty_cycles = 0;
    }
    if (its >= budget) {
      warn = !trset.empty();
      break;
    }
    std::sort(trset.begin(), trset.end(), [](const TrC& x, const TrC& y) { return x.theta > y.theta; });
    if ((int)trset.size() > tr_cap) trset.resize(tr_cap);
    tr_theta.clear();
    tr_s.clear();
    if (!broke) {
      const int lnew = (int)trset.size();
      std::vector<int> cols;
      for (int q = 0; q < lnew; ++q) {
        tr_theta.push_back(trset[q].theta);
        tr_s.push_back(trailing * trset[q].ylast);
        cols.push_back(trset[q].col);
      }
      // the kept Ritz vectors: straight from U when every candidate fit in one chunk, else
      // recomputed as W Y_kept into a staging block (the basis is still being read until then)
      const double* src = s.cand.U.p;
      if (chunk < ncand && lnew > 0) {
        s.stage_ritz(kr.W.p, kr.W.ld, steps, Y, j0, cols);
        src = s.trbuf.p;
        for (int q = 0; q < lnew; ++q) cols[q] = q;
      }
      // the last Lanczos vector moves to column lnew, the kept Ritz vectors fill 0..lnew-1
      k::rw_col_move(s.c, n, kr.W.p, kr.W.ld, steps, lnew);
      kr.put_cols(cols, src);
    }
  }
  s.cnt.n_A_matvec += (long)s.op.k * its;
  return s.results(its, warn, t0);
}

}  // namespace

SolverCfg resolve_config(const se_solver_cfg* in, const char* who) {
  se_solver_cfg z{0, 0, 30, 0.0, 1e-8, 20, 1234};
  const se_solver_cfg& q = in ? *in : z;
  SolverCfg c;
  if (q.est_count < 0) fail(SE_EINVAL, std::string(who) + ": negative est_count");
  c.est_count = q.est_count;
  c.m = q.m == 0 ? std::max(4 * q.est_count, 80) : q.m;
  c.max_its = q.max_its == 0 ? 40L * q.est_count + 300 : q.max_its;
  c.ncycle = q.ncycle;
  c.tau1 = q.tau1;
  c.res_tol = q.res_tol;
  c.seed = q.seed;
  if (c.m < 4) fail(SE_EINVAL, std::string(who) + ": restart dimension m < 4");
  if (c.ncycle < 1) fail(SE_EINVAL, std::string(who) + ": ncycle < 1");
  if (!(c.res_tol > 0.0)) fail(SE_EINVAL, std::string(who) + ": res_tol <= 0");
  if (c.max_its < 1) fail(SE_EINVAL, std::string(who) + ": max_its < 1");
  return c;
}

void apply_filter_dev(Ctx& c, const DevCsr& a, const StepOp& op, int nvec, const double* v,
                      double* out) {
  const int n = a.n;
  if (op.plain) {
    k::ChebArgs q;
    q.x = v;
    q.y = out;
    q.ncols = nvec;
    k::spmv_cheb(c, a, k::kPlain, q);
    return;
  }
  if (op.k < 1) fail(SE_EINVAL, "apply_pol: filter degree must be >= 1");
  double* fb[3];
  for (double*& b : fb) b = dev_alloc<double>(n);
  const int tiles = k::resident_tiles(a);
  double* mu_dev = nullptr;
  void* flags = nullptr;  // resident filter state
  if (tiles > 0) {
    mu_dev = dev_alloc<double>(op.k + 1);
    h2d(c, mu_dev, op.mu.data(), sizeof(double) * (op.k + 1));
    flags = dev_alloc<char>(k::resident_state_bytes(a));
    SE_CUDA(cudaMemsetAsync(flags, 0, k::resident_state_bytes(a), c.stream));
  }
  try {
    for (int col = 0; col < nvec; ++col) {
      const double* x = v + (size_t)col * n;
      double* o = out + (size_t)col * n;
      if (tiles > 0) {
        k::cheb_resident(c, a, op.k, mu_dev, op.c, op.invd, x, o, flags, nullptr);
        continue;
      }
      k::ChebArgs a1;
      a1.c = op.c;
      a1.invd = op.invd;
      a1.x = x;
      a1.y = fb[0];
      a1.out = o;
      a1.mu0 = op.mu[0];
      a1.muj = op.mu[1];
      k::spmv_cheb(c, a, k::kFirst, a1);
      int cur = 0, prv = -1, nxt = 1;
      for (int j = 2; j <= op.k; ++j) {
        k::ChebArgs b = a1;
        b.x = fb[cur];
        b.prev = prv < 0 ? x : fb[prv];
        b.y = fb[nxt];
        b.muj = op.mu[j];
        k::spmv_cheb(c, a, k::kNext, b);
        const int old = prv < 0 ? 2 : prv;
        prv = cur;
        cur = nxt;
        nxt = old;
      }
    }
    ctx_sync(c);
  } catch (...) {
    for (double* b : fb) dev_free(b);
    dev_free(mu_dev);
    dev_free(flags);
    throw;
  }
  for (double* b : fb) dev_free(b);
  dev_free(mu_dev);
  dev_free(flags);
}

// lanczos_run (lanczos.hpp:37-118), euclidean inner product.
LanczosRun lanczos_run(Ctx& c, const DevCsr& a, const double* start_host, int m, bool want_basis,
                       const Pencil* pen) {
  const int n = a.n;
  m = std::min(m, n);
  StepOp op;  // plain A (or S = P A P)
  Krylov kr(c, a, op, pen);
  kr.ensure(m + 1, 0);
  h2d(c, kr.t, start_host, sizeof(double) * n);
  const double nb2 = kr.dot(kr.t, kr.t);
  if (nb2 <= 0.0) fail(SE_ENUMERIC, "lanczos_run: B-inner product is not positive");
  k::scale(c, n, 1.0 / std::sqrt(nb2), kr.t);
  kr.put_col(0, kr.t);
  kr.begin(0);
  kr.run(0, m);
  const Ctl h = kr.get();
  LanczosRun r;
  r.steps = h.halted ? h.i + 1 : m;
  r.breakdown = h.halted != 0;
  kr.download(kr.alpha, r.steps, r.alpha);
  Vec be;
  kr.download(kr.beta, r.steps, be);
  if (r.breakdown) {
    r.beta.assign(be.begin(), be.begin() + std::max(r.steps - 1, 0));
    r.next_beta = 0.0;
  } else {
    r.beta.assign(be.begin(), be.begin() + (r.steps - 1));
    r.next_beta = be[r.steps - 1];
    kr.get_col(r.steps, kr.t);
    kr.download(kr.t, n, r.next_w);
  }
  if (want_basis) {
    double* cm = dev_alloc<double>((size_t)n * std::max(r.steps, 1));
    k::rw_get_cols(c, n, kr.W.p, kr.W.ld, 0, r.steps, cm);
    kr.download(cm, (int)((size_t)n * r.steps), r.basis);
    dev_free(cm);
  }
  return r;
}

// lan_tr_bounds (lanczos.hpp:148-277): keep the two extreme Ritz pairs across restarts.
void lan_tr_bounds(Ctx& c, const DevCsr& a, double tol, int restart_dim, int max_restarts,
                   std::uint64_t seed, double& lmin, double& lmax, const Pencil* pen) {
  const int n = a.n;
  const int m = std::min(restart_dim, n);
  if (m < 1) fail(SE_EINVAL, "lan_tr_bounds: empty operator");
  Rng rng(seed);
  StepOp op;
  Krylov kr(c, a, op, pen);
  kr.ensure(m + 1, 0);
  CandBuf cand(c);  // restart combinations only (the Ritz vectors stay in the Lanczos space)
  double* dY = dev_alloc<double>((size_t)m * 2);
  Vec kept_theta, kept_s;
  double prev_lo = 0.0, prev_hi = 0.0;
  bool have_prev = false;
  try {
    for (int cycle = 0; cycle < max_restarts; ++cycle) {
      const int k0 = (int)kept_theta.size();
      if (k0 == 0) {
        Vec w(n);
        rng.normal_fill(w.data(), n);
        h2d(c, kr.t, w.data(), sizeof(double) * n);
        const double nb = std::sqrt(kr.dot(kr.t, kr.t));
        k::scale(c, n, 1.0 / nb, kr.t);
        kr.put_col(0, kr.t);
      }
      SE_CUDA(cudaMemsetAsync(kr.hdiag, 0, sizeof(double) * kr.arr_cap, c.stream));
      kr.begin(k0);
      kr.run(1, m - k0);
      const Ctl h = kr.get();
      const bool broke = h.halted != 0;
      const int steps = broke ? h.i + 1 : m;
      Vec hd, be;
      kr.download(kr.hdiag, steps, hd);
      kr.download(kr.beta, steps, be);
      const double trailing = broke ? 0.0 : be[steps - 1];
      Vec H((size_t)steps * steps, 0.0);
      auto at = [&](int r, int cc) -> double& { return H[(size_t)cc * steps + r]; };
      for (int j = 0; j < k0; ++j) {
        at(j, j) = kept_theta[j];
        at(j, k0) = at(k0, j) = kept_s[j];
      }
      for (int q = k0; q < steps; ++q) at(q, q) += hd[q];
      for (int q = k0; q + 1 < steps; ++q) at(q + 1, q) = at(q, q + 1) = be[q];
      Vec vals, vecs;
      dense_sym_eig(steps, H.data(), true, vals, vecs);
      const double lo = vals.front(), hi = vals.back();
      const double spread = std::max(hi - lo, 1e-300);
      const bool settled = have_prev && std::abs(lo - prev_lo) <= tol * spread &&
                           std::abs(hi - prev_hi) <= tol * spread;
      if (settled || broke || cycle == max_restarts - 1 || steps >= n) {
        const double pad_lo = trailing * std::abs(vecs[(size_t)0 * steps + steps - 1]);
        const double pad_hi = trailing * std::abs(vecs[(size_t)(steps - 1) * steps + steps - 1]);
        lmin = lo - pad_lo;
        lmax = hi + pad_hi;
        dev_free(dY);
        return;
      }
      prev_lo = lo;
      prev_hi = hi;
      have_prev = true;
      kept_theta = {vals[0], vals[steps - 1]};
      kept_s = {trailing * vecs[(size_t)0 * steps + steps - 1],
                trailing * vecs[(size_t)(steps - 1) * steps + steps - 1]};
      h2d(c, dY, vecs.data(), sizeof(double) * steps);
      h2d(c, dY + steps, vecs.data() + (size_t)(steps - 1) * steps, sizeof(double) * steps);
      Vec st;
      cand.eval(a, kr.W.p, steps, dY, steps, 2, st, kr.W.ld);
      // seed first (column steps -> 2), then the kept combinations into columns 0, 1
      k::rw_col_move(c, n, kr.W.p, kr.W.ld, steps, 2);
      kr.put_cols({0, 1}, cand.U.p);
    }
  } catch (...) {
    dev_free(dY);
    throw;
  }
  dev_free(dY);
  fail(SE_ENUMERIC, "lan_tr_bounds: failed to settle");
}

void pencil_map(Ctx& c, const Pencil& pen, int nvec, const double* x, double* y) {
  apply_filter_block(c, *pen.B, pen.P, nvec, x, y);
}

std::unique_ptr<SliceResult> cheb_lan(Ctx& c, const DevCsr& a, const PolyFilter& f, double xi,
                                      double eta, const SolverCfg& cfg, bool thick_restart,
                                      int ndefl, const double* defl_u, const double* defl_vals,
                                      const char* who, const Pencil* pen) {
  if (!(eta > xi)) fail(SE_EINVAL, std::string(who) + ": degenerate interval");
  if (f.k < 1 || (int)f.mu.size() != f.k + 1) fail(SE_EINVAL, std::string(who) + ": malformed filter");
  if (pen && ndefl > 0)
    fail(SE_EINVAL, std::string(who) + ": a preloaded deflation set is not supported for B-pencils");
  Slice s(c, a, f, xi, eta, cfg, pen);
  s.preload(ndefl, defl_u, defl_vals, who);
  // a large locked set is reserved once from the estimate (+15% for the DOS estimate's error):
  // regrowing an 80 GB block needs the old and the new copy at once
  const int lock_est = ndefl + cfg.est_count + cfg.est_count * 3 / 20 + 64;
  if ((size_t)a.n * lock_est * 8 > kBigAlloc) s.kr.reserve_locked(lock_est);
  return thick_restart ? run_tr(s) : run_nr(s);
}

// ---- filtered subspace iteration (cheb_si, eigensolvers.hpp:760-940; standard problem) ---------
// Filter nvec columns (ld n) through the multi-vector fused kernel, 8 columns per launch:
// out_j = sum_k mu_k T_k(Ahat) v_j (apply_pol, filter_poly.hpp:256-277, column by column).
void apply_filter_block(Ctx& c, const DevCsr& a, const StepOp& op, int nvec, const double* v, double* out) {
  const int n = a.n;
  if (op.k < 2) {
    apply_filter_dev(c, a, op, nvec, v, out);
    return;
  }
  const int ngroups = (nvec + 7) / 8;
  if (k::cheb_block_available(a) && nvec > 2) {
    // padded-row matrices (stencils): groups of <= 8 columns as row-major n x 8 blocks through
    // the block kernel (one read of a row's entries for the whole group, 64-byte gathers)
    double* blk = dev_alloc<double>((size_t)n * 8 * 5);
    double* Xin = blk;
    double* T[3] = {blk + (size_t)n * 8, blk + (size_t)n * 16, blk + (size_t)n * 24};
    double* O = blk + (size_t)n * 32;
    try {
      for (int g = 0, c0 = 0; g < ngroups; ++g) {
        const int nv = nvec / ngroups + (g < nvec % ngroups ? 1 : 0);
        k::cheb_block_pack(c, v + (size_t)c0 * n, Xin, n, nv);
        k::cheb_block_step(c, a, true, Xin, nullptr, T[0], O, op.c, op.invd, op.mu[0], op.mu[1]);
        for (int j = 2; j <= op.k; ++j)
          k::cheb_block_step(c, a, false, T[(j - 2) % 3], j == 2 ? Xin : T[j % 3], T[(j - 1) % 3], O,
                             op.c, op.invd, 0.0, op.mu[j]);
        k::cheb_block_unpack(c, O, out + (size_t)c0 * n, n, nv);
        c0 += nv;
      }
      ctx_sync(c);
    } catch (...) {
      ctx_sync(c);
      dev_free(blk);
      throw;
    }
    dev_free(blk);
    return;
  }
  // longer rows: balanced groups of <= 8 columns (9 -> 5 + 4, not 8 + 1: a nearly empty
  // multi-vector launch costs almost a full one) through the CSR multi-vector kernel; groups of
  // one or two columns take the single-vector chain
  double* buf = dev_alloc<double>((size_t)n * 24);
  try {
    for (int g = 0, c0 = 0; g < ngroups; ++g) {
      const int nv = nvec / ngroups + (g < nvec % ngroups ? 1 : 0);
      if (nv <= 2) {
        apply_filter_dev(c, a, op, nv, v + (size_t)c0 * n, out + (size_t)c0 * n);
        c0 += nv;
        continue;
      }
      for (int j = 1; j <= op.k; ++j) {
        k::MultiArgs m{};
        m.nv = nv;
        m.c = op.c;
        m.invd = op.invd;
        for (int q = 0; q < nv; ++q) {
          const double* vq = v + (size_t)(c0 + q) * n;
          double* B[3] = {buf + (size_t)(3 * q) * n, buf + (size_t)(3 * q + 1) * n, buf + (size_t)(3 * q + 2) * n};
          m.x[q] = j == 1 ? vq : B[(j - 2) % 3];
          m.prev[q] = j == 2 ? vq : B[j % 3];
          m.y[q] = B[(j - 1) % 3];
          m.out[q] = out + (size_t)(c0 + q) * n;
          m.mu0[q] = op.mu[0];
          m.muj[q] = op.mu[j];
          m.first[q] = j == 1;
        }
        k::spmv_cheb_multi(c, a, m);
      }
      c0 += nv;
    }
    ctx_sync(c);
  } catch (...) {
    ctx_sync(c);
    dev_free(buf);
    throw;
  }
  dev_free(buf);
}

namespace {
// cgs2_orthogonalize (orth.hpp:39-61) of t against the first k columns of Q, in place:
// returns the final norm (t normalised) or 0.0 on breakdown (t untouched beyond the passes).
struct Orth {
  Ctx& c;
  k::Scratch s;
  Ctl* ctl = nullptr;
  double* coef = nullptr;
  int n, cap;
  Orth(Ctx& cc, int n_, int cap_) : c(cc), n(n_), cap(cap_) {
    s.cap = k::cgs_scratch_doubles(c, n, cap);
    s.ncnt = k::cgs_counter_slots(n, cap);
    s.buf = dev_alloc<double>(s.cap);
    s.cnt = dev_alloc<unsigned>(s.ncnt);
    ctl = dev_alloc<Ctl>(1);
    coef = dev_alloc<double>(std::max(cap, 1));
    SE_CUDA(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned) * s.ncnt, c.stream));
    ctx_sync(c);
  }
  ~Orth() {
    cudaStreamSynchronize(c.stream);
    for (void* p : {(void*)s.buf, (void*)s.cnt, (void*)ctl, (void*)coef}) dev_free(p);
  }
  double run(double* t, const double* Q, int kq) {
    Ctl h{};
    h.i = kq - 1;
    h2d(c, ctl, &h, sizeof(Ctl));
    k::norm_before(c, s, n, t, ctl);
    Ctl g;
    d2h(c, &g, ctl, sizeof(Ctl));
    const double initial = g.before;
    if (initial == 0.0) return 0.0;
    double after = initial;
    if (kq > 0) {
      k::cgs_pass(c, s, n, t, Q, false, false, ctl, nullptr, coef, cap);
      k::cgs_pass(c, s, n, t, Q, false, true, ctl, nullptr, coef, cap);
      d2h(c, &g, ctl, sizeof(Ctl));
      after = g.after;
    }
    if (after <= 1e-14 * initial) return 0.0;  // kBreakdownTol (orth.hpp:14)
    k::scale(c, n, 1.0 / after, t);
    return after;
  }
};

}  // namespace

std::unique_ptr<SliceResult> cheb_si(Ctx& c, const DevCsr& a, const PolyFilter& f, double xi,
                                     double eta, int est_count, const SolverCfg& cfg) {
  if (!(eta > xi)) fail(SE_EINVAL, "cheb_si: degenerate interval");
  if (est_count < 0) fail(SE_EINVAL, "cheb_si: negative est_count");
  if (f.k < 1 || (int)f.mu.size() != f.k + 1) fail(SE_EINVAL, "cheb_si: malformed filter");
  HiPrio hp(c);
  const auto t0 = std::chrono::steady_clock::now();
  const int n = a.n;
  const int q = std::min(n, (int)std::ceil(1.3 * est_count) + 8);
  const double bar_eff = f.bar * (1.0 - 1e-4);
  StepOp op;
  op.plain = false;
  op.k = f.k;
  op.mu = f.mu;
  op.c = f.c;
  op.invd = 1.0 / f.d;
  Rng rng(cfg.seed);
  auto res = std::make_unique<SliceResult>();
  res->n = n;
  se_counters& cnt = res->counters;
  DevMat Y, T, AY;
  devmat_reserve(c, Y, n, q, false);
  devmat_reserve(c, T, n, q, false);
  devmat_reserve(c, AY, n, q, false);
  Orth orth(c, n, q);
  DevEig eig(c);
  CandBuf cand(c);
  auto cleanup = [&] {
    ctx_sync(c);
    devmat_free(Y);
    devmat_free(T);
    devmat_free(AY);
  };
  auto secs = [](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
  };
  auto fresh = [&](double* dst) {  // rng.normal_vec(n) -> device column
    std::vector<double> h((size_t)n);
    rng.normal_fill(h.data(), n);
    h2d(c, dst, h.data(), sizeof(double) * n);
  };
  try {
    // random orthonormal start block (eigensolvers.hpp:818-823)
    for (int cols = 0; cols < q;) {
      fresh(Y.col(cols));
      if (orth.run(Y.col(cols), Y.p, cols) > 0.0) ++cols;
    }
    const double slo = 10.0 * cfg.res_tol * std::max(1.0, std::abs(xi));
    const double shi = 10.0 * cfg.res_tol * std::max(1.0, std::abs(eta));
    int saturated = 0, idle = 0;
    long cycle = 0;
    Vec lam, stats;
    std::vector<double> G((size_t)q * q);
    while (true) {
      ++cycle;
      // filter sweep (k A-products per column), then CGS2 re-orthonormalisation in column order
      auto tm = std::chrono::steady_clock::now();
      apply_filter_block(c, a, op, q, Y.p, T.p);
      cnt.n_A_matvec += (long)f.k * q;
      cnt.t_mv += secs(tm);
      auto to = std::chrono::steady_clock::now();
      for (int j = 0; j < q; ++j)
        while (orth.run(T.col(j), T.p, j) == 0.0) fresh(T.col(j));  // collapsed: fresh direction
      ctx_sync(c);
      cnt.t_orth += secs(to);
      // Rayleigh-Ritz: AY = A T, gram(i, j) = <AY_j, T_i> (i <= j, mirrored), eig, Y = T V
      tm = std::chrono::steady_clock::now();
      for (int j0 = 0; j0 < q; j0 += 65535) {
        k::ChebArgs pa;
        pa.x = T.col(j0);
        pa.y = AY.col(j0);
        pa.ncols = std::min(65535, q - j0);
        k::spmv_cheb(c, a, k::kPlain, pa);
      }
      cnt.n_A_matvec += q;
      double* dG = dev_alloc<double>((size_t)q * q);
      k::ritz_gemm(c, q, q, n, T.p, n, true, AY.p, n, dG, q);  // gram = T^T (A T)
      d2h(c, G.data(), dG, sizeof(double) * (size_t)q * q);
      dev_free(dG);
      for (int j = 0; j < q; ++j)
        for (int i = j + 1; i < q; ++i) G[(size_t)j * q + i] = G[(size_t)i * q + j];  // lower := upper
      const double* V = eig.solve(q, G, lam);
      k::ritz_gemm(c, n, q, q, T.p, n, false, V, q, Y.p, n);  // Y = T V
      cnt.t_mv += secs(tm);
      // candidate pass (eigensolvers.hpp:857-896): Ritz values inside the slack-widened slice
      std::vector<int> sel;
      for (int j = 0; j < q; ++j)
        if (!(lam[j] < xi - slo || lam[j] > eta + shi)) sel.push_back(j);
      struct Pair {
        double lambda, residual, scale;
        int col;
      };
      std::vector<Pair> inside;
      bool all_good = true;
      if (!sel.empty()) {
        std::vector<double> Vs((size_t)q * sel.size());
        std::vector<double> Vh((size_t)q * q);
        d2h(c, Vh.data(), V, sizeof(double) * (size_t)q * q);
        for (size_t s2 = 0; s2 < sel.size(); ++s2)
          std::copy(Vh.begin() + (size_t)sel[s2] * q, Vh.begin() + (size_t)(sel[s2] + 1) * q,
                    Vs.begin() + s2 * q);
        double* dV = dev_alloc<double>(Vs.size());
        h2d(c, dV, Vs.data(), sizeof(double) * Vs.size());
        cand.eval(a, T.p, q, dV, q, (int)sel.size(), stats);
        dev_free(dV);
        cnt.n_A_matvec += (long)sel.size();
        for (size_t s2 = 0; s2 < sel.size(); ++s2) {
          const double l = stats[3 * s2], r = stats[3 * s2 + 1], uu = stats[3 * s2 + 2];
          if (!(uu > 0.0)) continue;
          if (r > cfg.res_tol * std::max(1.0, std::abs(l))) all_good = false;
          inside.push_back({l, r, 1.0 / std::sqrt(uu), (int)s2});
        }
      }
      // a block whose every Ritz value maps above the bar cannot bracket the slice
      int above = 0;
      for (int j = 0; j < q; ++j) {
        const double t = std::clamp((lam[j] - f.c) / f.d, -1.0, 1.0);
        if (eval_pol(f.mu.data(), f.k, t) >= bar_eff) ++above;
      }
      saturated = above == q ? saturated + 1 : 0;
      if (saturated >= 3)
        fail(SE_ENUMERIC, "cheb_si: subspace saturated above the filter bar; raise est_count");
      idle = inside.empty() ? idle + 1 : 0;
      const bool done = (!inside.empty() && all_good) || idle >= 6;
      const bool budget = cycle >= cfg.max_its;
      if (done || budget) {
        std::sort(inside.begin(), inside.end(), [](const Pair& x, const Pair& y) { return x.lambda < y.lambda; });
        const int nev = (int)inside.size();
        devmat_reserve(c, res->vectors, n, std::max(nev, 1), false);
        for (int i = 0; i < nev; ++i) {
          k::scale_copy(c, n, inside[i].scale, cand.U.col(inside[i].col), res->vectors.col(i));
          res->eigenvalues.push_back(inside[i].lambda);
          res->residuals.push_back(inside[i].residual);
        }
        ctx_sync(c);
        res->niter = cycle;
        res->hit_max_its = budget && !done;
        cnt.t_total += secs(t0);
        cleanup();
        return res;
      }
    }
  } catch (...) {
    cleanup();
    throw;
  }
}

}  // namespace se

namespace se {
// Time the filter kernels as they run in production: one application (k fused SpMV launches)
// captured in a CUDA graph, replayed `reps` times between CUDA events on the context's stream.
void filter_bench(Ctx& c, const DevCsr& a, const StepOp& op, int reps, double& ms, long& launches) {
  const int n = a.n;
  double* v = dev_alloc<double>(n);
  double* out = dev_alloc<double>(n);
  double* fb[3];
  for (double*& b : fb) b = dev_alloc<double>(n);
  cudaGraphExec_t ge = nullptr;
  try {
    std::vector<double> h(n);
    Rng rng(99);
    rng.normal_fill(h.data(), n);
    h2d(c, v, h.data(), sizeof(double) * n);
    ctx_sync(c);
    const long before = c.launches;
    double* mu_dev = dev_alloc<double>(op.k + 1);
    h2d(c, mu_dev, op.mu.data(), sizeof(double) * (op.k + 1));
    const int tiles = k::resident_tiles(a);
    void* flags = nullptr;
    if (tiles > 0) {
      flags = dev_alloc<char>(k::resident_state_bytes(a));
      SE_CUDA(cudaMemsetAsync(flags, 0, k::resident_state_bytes(a), c.stream));
      ctx_sync(c);
    }
    SE_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    if (tiles > 0) {  // as in production: the whole filter is one resident launch
      k::cheb_resident(c, a, op.k, mu_dev, op.c, op.invd, v, out, flags, nullptr);
    } else {
      k::ChebArgs a1;
      a1.c = op.c;
      a1.invd = op.invd;
      a1.x = v;
      a1.y = fb[0];
      a1.out = out;
      a1.mu0 = op.mu[0];
      a1.muj = op.mu[1];
      k::spmv_cheb(c, a, k::kFirst, a1);
      int cur = 0, prv = -1, nxt = 1;
      for (int j = 2; j <= op.k; ++j) {
        k::ChebArgs b = a1;
        b.x = fb[cur];
        b.prev = prv < 0 ? v : fb[prv];
        b.y = fb[nxt];
        b.muj = op.mu[j];
        k::spmv_cheb(c, a, k::kNext, b);
        const int old = prv < 0 ? 2 : prv;
        prv = cur;
        cur = nxt;
        nxt = old;
      }
    }
    cudaGraph_t g;
    SE_CUDA(cudaStreamEndCapture(c.stream, &g));
    SE_CUDA(cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    // reported per filter degree either way (the resident launch covers op.k degrees)
    const long per = tiles > 0 ? op.k : c.launches - before;
    SE_CUDA(cudaGraphLaunch(ge, c.stream));  // warm
    SE_CUDA(cudaEventRecord(c.ev0, c.stream));
    for (int r = 0; r < reps; ++r) SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev1, c.stream));
    SE_CUDA(cudaEventSynchronize(c.ev1));
    float fms = 0.f;
    SE_CUDA(cudaEventElapsedTime(&fms, c.ev0, c.ev1));
    ms = fms;
    launches = per * reps;
    c.launches += (c.launches - before) * (reps + 1);
    dev_free(mu_dev);
    dev_free(flags);
  } catch (...) {
    if (ge) cudaGraphExecDestroy(ge);
    for (void* p : {(void*)v, (void*)out, (void*)fb[0], (void*)fb[1], (void*)fb[2]}) dev_free(p);
    throw;
  }
  cudaGraphExecDestroy(ge);
  for (void* p : {(void*)v, (void*)out, (void*)fb[0], (void*)fb[1], (void*)fb[2]}) dev_free(p);
}
}  // namespace se

namespace se {
// Time one classical Gram-Schmidt pass (k_gemvt + k_gemvn with norm) against an n x k basis, as it
// runs inside the Lanczos step graph (production path), replayed `reps` times between events.
void cgs_bench(Ctx& c, int n, int kcols, int reps, double& ms) { cgs2_bench(c, n, kcols, reps, -1, ms); }

// mode -1: one column-major pass (k_gemvt + k_gemvn, the locked-set / cheb_si path); 0: a CGS2
// step as two column-major passes (4 reads of W); 2: the product's CGS2 step on the row-major
// basis (T1 + fused MID + N2, 3 reads).  The re-pass is forced (before = 1e300).
void cgs2_bench(Ctx& c, int n, int kcols, int reps, int mode, double& ms) {
  if (n < 1 || kcols < 1 || reps < 1) fail(SE_EINVAL, "se_cgs_bench: bad sizes");
  double* W = dev_alloc<double>((size_t)n * kcols);
  double* t = dev_alloc<double>(n);
  double* coef = dev_alloc<double>(kcols);
  double* coef2 = dev_alloc<double>(kcols);
  Ctl* ctl = dev_alloc<Ctl>(2);  // [0] live, [1] the state every replay starts from
  k::Scratch s;
  s.cap = k::cgs_scratch_doubles(c, n, kcols);
  s.ncnt = k::cgs_counter_slots(n, kcols);
  s.buf = dev_alloc<double>(s.cap);
  s.cnt = dev_alloc<unsigned>(s.ncnt);
  // mode 2: row-major basis, three-read CGS2 (rowgs.cu)
  const int ldw = k::rw_ldw(kcols);
  k::RowScratch rs;
  double* rbuf = nullptr;
  if (mode == 2) {
    rs = k::rw_scratch(c, ldw);
    rbuf = dev_alloc<double>(k::rw_scratch_doubles(rs));
    k::rw_bind(rs, rbuf);
    dev_free(W);
    W = dev_alloc<double>((size_t)n * ldw);
  }
  unsigned* mcnt = dev_alloc<unsigned>(1);
  cudaGraphExec_t ge = nullptr;
  auto cleanup = [&] {
    if (ge) cudaGraphExecDestroy(ge);
    for (void* p : {(void*)W, (void*)t, (void*)coef, (void*)coef2, (void*)ctl, (void*)s.buf, (void*)s.cnt,
                    (void*)mcnt, (void*)rbuf})
      dev_free(p);
  };
  try {
    SE_CUDA(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned) * s.ncnt, c.stream));
    SE_CUDA(cudaMemsetAsync(mcnt, 0, sizeof(unsigned), c.stream));
    // deterministic pseudo-random contents (values do not affect the traffic)
    std::vector<double> h((size_t)n);
    Rng rng(7);
    rng.normal_fill(h.data(), n);
    if (mode == 2) {
      std::vector<double> row((size_t)ldw);
      for (int j = 0; j < ldw; ++j) row[j] = h[j % n];
      for (int r = 0; r < n; r += 4096) {
        const int cnt = std::min(4096, n - r);
        std::vector<double> blk((size_t)cnt * ldw);
        for (int q = 0; q < cnt; ++q) std::copy(row.begin(), row.end(), blk.begin() + (size_t)q * ldw);
        h2d(c, W + (size_t)r * ldw, blk.data(), sizeof(double) * blk.size());
      }
    } else {
      for (int j = 0; j < kcols; ++j)
        h2d(c, W + (size_t)j * n, h.data(), sizeof(double) * n);
    }
    h2d(c, t, h.data(), sizeof(double) * n);
    Ctl z{};
    z.i = kcols - 1;
    z.before = mode < 0 ? 1.0 : 1e300;
    h2d(c, ctl, &z, sizeof(Ctl));
    h2d(c, ctl + 1, &z, sizeof(Ctl));
    ctx_sync(c);
    const long before = c.launches;
    SE_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    SE_CUDA(cudaMemcpyAsync(ctl, ctl + 1, sizeof(Ctl), cudaMemcpyDeviceToDevice, c.stream));
    if (mode < 0) {
      k::cgs_pass(c, s, n, t, W, false, false, ctl, nullptr, coef, kcols);
    } else if (mode == 0) {
      k::cgs_pass(c, s, n, t, W, false, false, ctl, nullptr, coef, kcols);
      k::cgs_pass(c, s, n, t, W, false, true, ctl, nullptr, coef, kcols);
    } else if (mode == 2) {
      k::rw_cgs2(c, rs, n, t, W, ldw, ctl, nullptr, coef, coef2, false);
    } else {
      fail(SE_EINVAL, "se_cgs2_bench: mode is -1, 0 or 2");
    }
    cudaGraph_t g;
    SE_CUDA(cudaStreamEndCapture(c.stream, &g));
    SE_CUDA(cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    const long per = c.launches - before;
    SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev0, c.stream));
    for (int r = 0; r < reps; ++r) SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev1, c.stream));
    SE_CUDA(cudaEventSynchronize(c.ev1));
    float fms = 0.f;
    SE_CUDA(cudaEventElapsedTime(&fms, c.ev0, c.ev1));
    ms = fms;
    c.launches += per * (reps + 1);
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}
}  // namespace se

namespace se {
// Time k degrees of the multi-vector filter over nv vectors (graph-captured, replayed).
// Time kdeg degrees of the row-major block filter (8 vectors; graph-captured, replayed).
void block_filter_bench(Ctx& c, const DevCsr& a, int kdeg, int reps, double& ms) {
  if (kdeg < 2 || reps < 1) fail(SE_EINVAL, "se_block_filter_bench: bad sizes");
  if (!k::cheb_block_available(a)) fail(SE_EINVAL, "se_block_filter_bench: rows longer than 8 entries");
  const int n = a.n;
  double* blk = dev_alloc<double>((size_t)n * 8 * 5);
  SE_CUDA(cudaMemsetAsync(blk, 0, sizeof(double) * (size_t)n * 40, c.stream));
  double* Xin = blk;
  double* T[3] = {blk + (size_t)n * 8, blk + (size_t)n * 16, blk + (size_t)n * 24};
  double* O = blk + (size_t)n * 32;
  cudaGraphExec_t ge = nullptr;
  try {
    ctx_sync(c);
    SE_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    k::cheb_block_step(c, a, true, Xin, nullptr, T[0], O, 6.0, 1.0 / 6.0, 0.5, 0.1);
    for (int j = 2; j <= kdeg; ++j)
      k::cheb_block_step(c, a, false, T[(j - 2) % 3], j == 2 ? Xin : T[j % 3], T[(j - 1) % 3], O, 6.0,
                         1.0 / 6.0, 0.0, 0.1);
    cudaGraph_t g;
    SE_CUDA(cudaStreamEndCapture(c.stream, &g));
    SE_CUDA(cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev0, c.stream));
    for (int r = 0; r < reps; ++r) SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev1, c.stream));
    SE_CUDA(cudaEventSynchronize(c.ev1));
    float f = 0.f;
    SE_CUDA(cudaEventElapsedTime(&f, c.ev0, c.ev1));
    ms = f;
  } catch (...) {
    if (ge) cudaGraphExecDestroy(ge);
    dev_free(blk);
    throw;
  }
  cudaGraphExecDestroy(ge);
  dev_free(blk);
}

void multi_filter_bench(Ctx& c, const DevCsr& a, int nv, int kdeg, int reps, double& ms) {
  if (nv < 1 || nv > 8 || kdeg < 2 || reps < 1) fail(SE_EINVAL, "se_multi_filter_bench: bad sizes");
  const int n = a.n;
  std::vector<double*> bufs;
  auto alloc = [&]() {
    double* p = dev_alloc<double>(n);
    SE_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * n, c.stream));
    bufs.push_back(p);
    return p;
  };
  double *V[8], *O[8], *B[8][3];
  for (int q = 0; q < nv; ++q) {
    V[q] = alloc();
    O[q] = alloc();
    for (int r = 0; r < 3; ++r) B[q][r] = alloc();
  }
  cudaGraphExec_t ge = nullptr;
  try {
    ctx_sync(c);
    SE_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    for (int j = 1; j <= kdeg; ++j) {
      k::MultiArgs m{};
      m.nv = nv;
      m.c = 6.0;
      m.invd = 1.0 / 6.0;
      for (int q = 0; q < nv; ++q) {
        m.x[q] = j == 1 ? V[q] : B[q][(j - 2) % 3];
        m.prev[q] = j == 2 ? V[q] : B[q][j % 3];
        m.y[q] = B[q][(j - 1) % 3];
        m.out[q] = O[q];
        m.mu0[q] = 0.5;
        m.muj[q] = 0.1;
        m.first[q] = j == 1;
      }
      k::spmv_cheb_multi(c, a, m);
    }
    cudaGraph_t g;
    SE_CUDA(cudaStreamEndCapture(c.stream, &g));
    SE_CUDA(cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(g);
    SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev0, c.stream));
    for (int r = 0; r < reps; ++r) SE_CUDA(cudaGraphLaunch(ge, c.stream));
    SE_CUDA(cudaEventRecord(c.ev1, c.stream));
    SE_CUDA(cudaEventSynchronize(c.ev1));
    float f = 0.f;
    SE_CUDA(cudaEventElapsedTime(&f, c.ev0, c.ev1));
    ms = f;
  } catch (...) {
    if (ge) cudaGraphExecDestroy(ge);
    for (double* p : bufs) dev_free(p);
    throw;
  }
  cudaGraphExecDestroy(ge);
  for (double* p : bufs) dev_free(p);
}
}  // namespace se
