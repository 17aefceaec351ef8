// extern "C" boundary of libsliceeig_cuda.so (declarations: include/sliceeig_cuda.h).
// Every entry point converts exceptions into SE_* status codes + a thread-local message.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "engine.hpp"
#include "host_algos.hpp"

using namespace se;

struct se_ctx {
  Ctx* c;
};
struct se_csr {
  DevCsr a;
};
struct se_pencil {
  Pencil p;
  double bmin = 0.0, bmax = 0.0, achieved = 0.0;
};
struct se_results {
  std::unique_ptr<SliceResult> r;
  int device = 0;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SE_OK;
  } catch (const se::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SE_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SE_ENUMERIC;
  }
}

Ctx& C(se_ctx* c) {
  if (!c || !c->c) fail(SE_EINVAL, "null se_ctx");
  SE_CUDA(cudaSetDevice(c->c->device));
  set_current_ctx(c->c);  // the thread's stream-ordered allocations go to this context
  return *c->c;
}
const DevCsr& M(const se_csr* a) {
  if (!a) fail(SE_EINVAL, "null se_csr");
  return a->a;
}

PolyFilter to_filter(const se_poly_filter* f) {
  if (!f || !f->mu) fail(SE_EINVAL, "null filter");
  PolyFilter p;
  p.k = f->k;
  p.gamma = f->gamma;
  p.c = f->c;
  p.d = f->d;
  p.tau = f->tau;
  p.ta = f->ta;
  p.tb = f->tb;
  p.bar = f->bar;
  p.damping = f->damping;
  p.cap_reached = f->cap_reached != 0;
  if (p.k < 1) fail(SE_EINVAL, "apply_pol: filter degree must be >= 1");
  p.mu.assign(f->mu, f->mu + f->k + 1);
  return p;
}

StepOp to_op(const PolyFilter& f) {
  StepOp o;
  o.plain = false;
  o.k = f.k;
  o.mu = f.mu;
  o.c = f.c;
  o.invd = 1.0 / f.d;
  return o;
}

void check_csr_host(int n, const int* rp, const int* ci) {
  if (n < 0) fail(SE_EINVAL, "CsrMatrix: negative dimension");
  if (!rp) fail(SE_EINVAL, "null row_ptr");
  if (rp[0] != 0) fail(SE_EINVAL, "CsrMatrix: row_ptr[0] must be 0");
  for (int i = 0; i < n; ++i)
    if (rp[i + 1] < rp[i]) fail(SE_EINVAL, "CsrMatrix: row_ptr must be non-decreasing");
  for (long p = 0; p < rp[n]; ++p)
    if (ci[p] < 0 || ci[p] >= n) fail(SE_ERANGE, "CsrMatrix: triplet index out of range");
}

}  // namespace

namespace se {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace se

extern "C" {

const char* se_last_error(void) { return g_err.c_str(); }
const char* se_version(void) { return "sliceeig-b200 0.1 (sm_100a)"; }

int se_device_memory(int device, size_t* free_bytes, size_t* total_bytes) {
  return guard([&] {
    SE_CUDA(cudaSetDevice(device));
    size_t f = 0, t = 0;
    SE_CUDA(cudaMemGetInfo(&f, &t));
    if (free_bytes) *free_bytes = f;
    if (total_bytes) *total_bytes = t;
  });
}

int se_device_count(int* count) {
  return guard([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

// ---- contexts ------------------------------------------------------------------------------
int se_ctx_set_candidate_budget(se_ctx* ctx, size_t bytes) {
  return guard([&] {
    if (bytes < 1) fail(SE_EINVAL, "se_ctx_set_candidate_budget: zero budget");
    C(ctx).cand_budget = bytes;
  });
}

int se_ctx_create(int device, se_ctx** out) {
  return guard([&] {
    *out = nullptr;
    auto* h = new se_ctx{ctx_create(device)};
    *out = h;
  });
}
int se_ctx_destroy(se_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    ctx_destroy(ctx->c);
    delete ctx;
  });
}
int se_ctx_synchronize(se_ctx* ctx) {
  return guard([&] { SE_CUDA(cudaStreamSynchronize(C(ctx).stream)); });
}
int se_ctx_kernel_launches(se_ctx* ctx, long* out) {
  return guard([&] { *out = C(ctx).launches; });
}
int se_ctx_filter_timing(se_ctx* ctx, int enable, double* ms, long* launches, double* bytes) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (ms) *ms = c.filter_ms;
    if (launches) *launches = c.filter_launches;
    if (bytes) *bytes = c.filter_bytes;
    c.time_filter = enable != 0;
    c.filter_ms = 0.0;
    c.filter_launches = 0;
    c.filter_bytes = 0.0;
  });
}

// ---- matrices -------------------------------------------------------------------------------
int se_laplacian_host(int ndims, const int* dims, int* n, long* nnz, int* rp, int* ci, double* v) {
  return guard([&] {
    if (ndims < 1 || ndims > 3) fail(SE_EINVAL, "gen_laplacian: need 1 to 3 grid dimensions");
    for (int q = 0; q < ndims; ++q)
      if (dims[q] < 1) fail(SE_EINVAL, "gen_laplacian: grid dimensions must be positive");
    const long nx = dims[0], ny = ndims > 1 ? dims[1] : 1, nz = ndims > 2 ? dims[2] : 1;
    const long nl = nx * ny * nz;
    if (nl > 40000000L) fail(SE_EINVAL, "gen_laplacian: grid too large");
    long cnt = nl + 2 * (nx - 1) * ny * nz + 2 * nx * (ny - 1) * nz + 2 * nx * ny * (nz - 1);
    *n = (int)nl;
    *nnz = cnt;
    if (!rp) return;
    const long plane = nx * ny;
    long p = 0;
    long row = 0;
    rp[0] = 0;
    for (long kz = 0; kz < nz; ++kz)
      for (long jy = 0; jy < ny; ++jy)
        for (long ix = 0; ix < nx; ++ix, ++row) {
          auto put = [&](long col, double val) {
            ci[p] = (int)col;
            v[p++] = val;
          };
          if (nz > 1 && kz > 0) put(row - plane, -1.0);
          if (ny > 1 && jy > 0) put(row - nx, -1.0);
          if (ix > 0) put(row - 1, -1.0);
          put(row, 2.0 * ndims);
          if (ix < nx - 1) put(row + 1, -1.0);
          if (ny > 1 && jy < ny - 1) put(row + nx, -1.0);
          if (nz > 1 && kz < nz - 1) put(row + plane, -1.0);
          rp[row + 1] = (int)p;
        }
  });
}

int se_laplacian_eigs(int ndims, const int* dims, double* out) {
  return guard([&] {
    if (ndims < 1 || ndims > 3) fail(SE_EINVAL, "laplacian_analytic_eigs: need 1 to 3 grid dimensions");
    long n = 1;
    for (int q = 0; q < ndims; ++q) {
      if (dims[q] < 1) fail(SE_EINVAL, "laplacian_analytic_eigs: dimensions must be positive");
      n *= dims[q];
    }
    if (n > 10000000L) fail(SE_EINVAL, "laplacian_analytic_eigs: enumeration too large");
    const double pi = 3.14159265358979323846;
    std::vector<Vec> one(ndims);
    for (int q = 0; q < ndims; ++q) {
      one[q].resize(dims[q]);
      for (int i = 1; i <= dims[q]; ++i) {
        const double s = std::sin(0.5 * pi * i / (dims[q] + 1));
        one[q][i - 1] = 4.0 * s * s;
      }
    }
    const int nx = dims[0], ny = ndims > 1 ? dims[1] : 1, nz = ndims > 2 ? dims[2] : 1;
    long p = 0;
    for (int kz = 0; kz < nz; ++kz)
      for (int jy = 0; jy < ny; ++jy)
        for (int ix = 0; ix < nx; ++ix) {
          double val = one[0][ix];
          if (ndims > 1) val += one[1][jy];
          if (ndims > 2) val += one[2][kz];
          out[p++] = val;
        }
    std::sort(out, out + n);
  });
}

int se_gen_random_sparse(int n, uint64_t seed, int halfband, int extras, double diag_frac,
                         long* nnz, int* rp, int* ci, double* v) {
  return guard([&] {
    if (n < 1 || halfband < 0 || extras < 0) fail(SE_EINVAL, "gen_random_sparse: bad parameters");
    if (extras > 0 && n - (2 * halfband + 1) < extras * 4)
      fail(SE_EINVAL, "gen_random_sparse: matrix too small for the requested extras");
    // pattern (row lists kept sorted)
    std::vector<std::vector<int>> nb(n);
    for (int i = 0; i < n; ++i) {
      nb[i].reserve(2 * halfband + 2 * extras + 8);
      for (int j = std::max(0, i - halfband); j <= std::min(n - 1, i + halfband); ++j)
        if (j != i) nb[i].push_back(j);
    }
    Rng rng(seed);
    auto has = [&](int i, int j) { return std::binary_search(nb[i].begin(), nb[i].end(), j); };
    auto insert = [&](int i, int j) { nb[i].insert(std::upper_bound(nb[i].begin(), nb[i].end(), j), j); };
    for (int i = 0; i < n; ++i) {
      int got = 0;
      while (got < extras) {
        const int j = (int)(rng.uniform() * n);
        if (std::abs(i - j) <= halfband || has(i, j)) continue;  // resample collisions
        insert(i, j);
        insert(j, i);
        ++got;
      }
    }
    long total = n;
    for (int i = 0; i < n; ++i) total += (long)nb[i].size();
    *nnz = total;
    if (!rp) return;
    // values: one N(0,1) per unordered pair (i < j) in row-major order, then the diagonal
    std::vector<long> start(n + 1, 0);
    for (int i = 0; i < n; ++i) start[i + 1] = start[i] + (long)nb[i].size() + 1;
    rp[0] = 0;
    for (int i = 0; i < n; ++i) rp[i + 1] = (int)start[i + 1];
    auto pos = [&](int i, int j) {  // index of column j in row i (diagonal included in order)
      const auto it = std::lower_bound(nb[i].begin(), nb[i].end(), j);
      const long k = it - nb[i].begin();
      return start[i] + k + (j > i ? 1 : 0);
    };
    for (int i = 0; i < n; ++i) {
      const long dpos = start[i] + (std::lower_bound(nb[i].begin(), nb[i].end(), i) - nb[i].begin());
      ci[dpos] = i;
      for (int j : nb[i]) ci[pos(i, j)] = j;
    }
    std::vector<double> rowabs(n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j : nb[i])
        if (j > i) {
          const double val = rng.normal();
          v[pos(i, j)] = val;
          v[pos(j, i)] = val;
          rowabs[i] += std::abs(val);
          rowabs[j] += std::abs(val);
        }
    for (int i = 0; i < n; ++i) {
      const long dpos = start[i] + (std::lower_bound(nb[i].begin(), nb[i].end(), i) - nb[i].begin());
      v[dpos] = rng.normal() + diag_frac * rowabs[i];
    }
  });
}

int se_mass_scaling(int n, uint64_t seed, double* b, double* d) {
  return guard([&] {
    if (n < 0) fail(SE_EINVAL, "mass_scaling: negative size");
    Rng rng(seed);
    for (int i = 0; i < n; ++i) {
      b[i] = 0.5 + rng.uniform();
      d[i] = 1.0 / std::sqrt(b[i]);
    }
  });
}

int se_csr_upload(se_ctx* ctx, int n, const int* row_ptr, const int* col_idx, const double* vals,
                  se_csr** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    check_csr_host(n, row_ptr, col_idx);
    auto h = std::make_unique<se_csr>();
    DevCsr& a = h->a;
    a.device = c.device;
    a.n = n;
    a.nnz = row_ptr[n];
    a.rp = dev_alloc_shared<int>(n + 1);
    a.alloc_entries(a.nnz);
    int mx = 0;
    for (int i = 0; i < n; ++i) mx = std::max(mx, row_ptr[i + 1] - row_ptr[i]);
    a.max_row_nnz = mx;
    SE_CUDA(cudaMemcpyAsync(a.rp, row_ptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice, c.stream));
    if (a.nnz) {
      SE_CUDA(cudaMemcpyAsync(a.ci, col_idx, sizeof(int) * a.nnz, cudaMemcpyHostToDevice, c.stream));
      SE_CUDA(cudaMemcpyAsync(a.v, vals, sizeof(double) * a.nnz, cudaMemcpyHostToDevice, c.stream));
    }
    k::build_ell(c, a);
    ctx_sync(c);
    *out = h.release();
  });
}

int se_csr_gen_laplacian(se_ctx* ctx, int ndims, const int* dims, se_csr** out) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (ndims < 1 || ndims > 3) fail(SE_EINVAL, "gen_laplacian: need 1 to 3 grid dimensions");
    long nl = 1;
    for (int q = 0; q < ndims; ++q) {
      if (dims[q] < 1) fail(SE_EINVAL, "gen_laplacian: grid dimensions must be positive");
      nl *= dims[q];
    }
    if (nl > 40000000L) fail(SE_EINVAL, "gen_laplacian: grid too large");
    auto h = std::make_unique<se_csr>();
    h->a.device = c.device;
    k::gen_laplacian(c, ndims, dims, h->a);
    ctx_sync(c);
    *out = h.release();
  });
}

int se_csr_info(const se_csr* a, int* n, long* nnz) {
  return guard([&] {
    *n = M(a).n;
    *nnz = M(a).nnz;
  });
}

int se_csr_download(se_ctx* ctx, const se_csr* a, int* row_ptr, int* col_idx, double* vals) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    SE_CUDA(cudaMemcpyAsync(row_ptr, m.rp, sizeof(int) * (m.n + 1), cudaMemcpyDeviceToHost, c.stream));
    if (m.nnz) {
      SE_CUDA(cudaMemcpyAsync(col_idx, m.ci, sizeof(int) * m.nnz, cudaMemcpyDeviceToHost, c.stream));
      SE_CUDA(cudaMemcpyAsync(vals, m.v, sizeof(double) * m.nnz, cudaMemcpyDeviceToHost, c.stream));
    }
    ctx_sync(c);
  });
}

int se_csr_scale_sym(se_ctx* ctx, se_csr* a, const double* d_host) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (!a) fail(SE_EINVAL, "null se_csr");
    double* d = dev_alloc<double>(a->a.n);
    SE_CUDA(cudaMemcpyAsync(d, d_host, sizeof(double) * a->a.n, cudaMemcpyHostToDevice, c.stream));
    k::csr_scale_sym(c, a->a, d);
    ctx_sync(c);
    dev_free(d);
  });
}

int se_csr_set_residual_weight(se_ctx* ctx, se_csr* a, const double* w_host) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (!a) fail(SE_EINVAL, "null se_csr");
    if (!w_host) {
      ctx_sync(c);
      dev_free_shared(a->a.resw);
      a->a.resw = nullptr;
      return;
    }
    if (!a->a.resw) a->a.resw = dev_alloc_shared<double>(std::max(a->a.n, 1));
    SE_CUDA(cudaMemcpyAsync(a->a.resw, w_host, sizeof(double) * a->a.n, cudaMemcpyHostToDevice,
                            c.stream));
    ctx_sync(c);
  });
}

int se_csr_free(se_csr* a) {
  return guard([&] {
    if (!a) return;
    cudaSetDevice(a->a.device);
    dev_free_shared(a->a.rp);
    dev_free_shared(a->a.resw);
    k::resident_free(a->a);
    a->a.free_entries();
    if (a->a.ell_c) {
      dev_free_shared(a->a.ell_c);
      dev_free_shared(a->a.ell_a);
    }
    delete a;
  });
}

// ---- operator applications ------------------------------------------------------------------
int se_spmv(se_ctx* ctx, const se_csr* a, const double* x, double* y) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    double* dx = dev_alloc<double>(m.n);
    double* dy = dev_alloc<double>(m.n);
    SE_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * m.n, cudaMemcpyHostToDevice, c.stream));
    StepOp op;
    apply_filter_dev(c, m, op, 1, dx, dy);
    SE_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * m.n, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    dev_free(dx);
    dev_free(dy);
  });
}

int se_cheb_apply_dev(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int nvec,
                      const double* d_v, double* d_out) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    const PolyFilter pf = to_filter(f);
    const StepOp op = to_op(pf);
    if (c.time_filter) SE_CUDA(cudaEventRecord(c.ev0, c.stream));
    apply_filter_dev(c, m, op, nvec, d_v, d_out);
    if (c.time_filter) {
      SE_CUDA(cudaEventRecord(c.ev1, c.stream));
      SE_CUDA(cudaEventSynchronize(c.ev1));
      float ms = 0.f;
      SE_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      c.filter_ms += ms;
      c.filter_launches += (long)nvec * pf.k;
      // algorithmic bytes: j = 1 step Abytes + 32 n, j >= 2 steps Abytes + 40 n
      c.filter_bytes += (double)nvec * (m.abytes() + 32.0 * m.n +
                                        (pf.k - 1) * (m.abytes() + 40.0 * m.n));
    }
  });
}

int se_filter_bench(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int reps, double* ms,
                    long* launches, double* bytes) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    const PolyFilter pf = to_filter(f);
    if (reps < 1) fail(SE_EINVAL, "se_filter_bench: reps must be positive");
    double t = 0.0;
    long nl = 0;
    filter_bench(c, m, to_op(pf), reps, t, nl);
    *ms = t;
    *launches = nl;
    *bytes = (double)reps * (m.abytes() + 32.0 * m.n + (pf.k - 1) * (m.abytes() + 40.0 * m.n));
  });
}

int se_cgs_bench(se_ctx* ctx, int n, int k, int reps, double* ms) {
  return guard([&] { cgs_bench(C(ctx), n, k, reps, *ms); });
}

int se_multi_filter_bench(se_ctx* ctx, const se_csr* a, int nv, int kdeg, int reps, double* ms) {
  return guard([&] { multi_filter_bench(C(ctx), M(a), nv, kdeg, reps, *ms); });
}

int se_block_filter_bench(se_ctx* ctx, const se_csr* a, int kdeg, int reps, double* ms) {
  return guard([&] { block_filter_bench(C(ctx), M(a), kdeg, reps, *ms); });
}

int se_cgs2_bench(se_ctx* ctx, int n, int k, int reps, int mode, double* ms) {
  return guard([&] {
    cgs2_bench(C(ctx), n, k, reps, mode, *ms);
  });
}

int se_resident_filter(int enable) {
  return guard([&] { k::resident_enable(enable); });
}

int se_csr_resident_tiles(const se_csr* a, int* tiles) {
  return guard([&] {
    if (!a || !tiles) fail(SE_EINVAL, "se_csr_resident_tiles: null argument");
    *tiles = k::resident_tiles(M(a));
  });
}

int se_csr_resident_smem(const se_csr* a, size_t* bytes) {
  return guard([&] {
    if (!a || !bytes) fail(SE_EINVAL, "se_csr_resident_smem: null argument");
    *bytes = k::resident_tile_smem(M(a));
  });
}

int se_mult_cols(se_ctx* ctx, int m, int n, int k, const double* a, long lda, int a_kcontig,
                 const double* b, long ldb, double* out, long ldc, int reps, double* ms) {
  return guard([&] {
    Ctx& c = C(ctx);
    if (m < 0 || n < 0 || k < 0 || !out) fail(SE_EINVAL, "mult_cols: bad shape");
    const size_t na = a_kcontig ? (size_t)(m - 1) * lda + k : (size_t)(k - 1) * lda + m;
    const size_t nb = (size_t)(n - 1) * ldb + k, nc = (size_t)(n - 1) * ldc + m;
    double* da = dev_alloc<double>(std::max<size_t>(na, 1));
    double* db = dev_alloc<double>(std::max<size_t>(nb, 1));
    double* dc = dev_alloc<double>(std::max<size_t>(nc, 1));
    if (a) {
      SE_CUDA(cudaMemcpyAsync(da, a, sizeof(double) * na, cudaMemcpyHostToDevice, c.stream));
    } else {  // timing only: synthetic operands
      SE_CUDA(cudaMemsetAsync(da, 0x3c, sizeof(double) * na, c.stream));
    }
    if (b)
      SE_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * nb, cudaMemcpyHostToDevice, c.stream));
    else
      SE_CUDA(cudaMemsetAsync(db, 0x3c, sizeof(double) * nb, c.stream));
    SE_CUDA(cudaMemsetAsync(dc, 0, sizeof(double) * nc, c.stream));
    k::ritz_gemm(c, m, n, k, da, lda, a_kcontig != 0, db, ldb, dc, ldc);
    if (reps > 0 && ms) {
      cudaEvent_t e0, e1;
      SE_CUDA(cudaEventCreate(&e0));
      SE_CUDA(cudaEventCreate(&e1));
      SE_CUDA(cudaEventRecord(e0, c.stream));
      for (int r = 0; r < reps; ++r) k::ritz_gemm(c, m, n, k, da, lda, a_kcontig != 0, db, ldb, dc, ldc);
      SE_CUDA(cudaEventRecord(e1, c.stream));
      SE_CUDA(cudaEventSynchronize(e1));
      float t = 0.f;
      SE_CUDA(cudaEventElapsedTime(&t, e0, e1));
      *ms = t / reps;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    if (a && b) SE_CUDA(cudaMemcpyAsync(out, dc, sizeof(double) * nc, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    dev_free(da);
    dev_free(db);
    dev_free(dc);
  });
}

int se_cheb_apply(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, int nvec, const double* v,
                  double* out, long* n_matvec) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    const PolyFilter pf = to_filter(f);
    const size_t bytes = sizeof(double) * (size_t)m.n * nvec;
    double* dv = dev_alloc<double>((size_t)m.n * nvec);
    double* dout = dev_alloc<double>((size_t)m.n * nvec);
    SE_CUDA(cudaMemcpyAsync(dv, v, bytes, cudaMemcpyHostToDevice, c.stream));
    if (nvec > 1)
      apply_filter_block(c, m, to_op(pf), nvec, dv, dout);  // 8 columns per fused launch
    else
      apply_filter_dev(c, m, to_op(pf), nvec, dv, dout);
    SE_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    dev_free(dv);
    dev_free(dout);
    if (n_matvec) *n_matvec += (long)pf.k * nvec;
  });
}

// ---- filters ---------------------------------------------------------------------------------
int se_damping_multipliers(int k, int damping, double* out) {
  return guard([&] {
    if (k < 0) fail(SE_EINVAL, "damping_multipliers: negative degree");
    const Vec s = damping_multipliers(k, damping);
    std::copy(s.begin(), s.end(), out);
  });
}
int se_chebyshev_coeffs(double gamma, int k, double* out) {
  return guard([&] {
    const Vec s = chebyshev_coeffs(gamma, k);
    std::copy(s.begin(), s.end(), out);
  });
}
int se_normalized_filter_coeffs(int k, double gamma, int damping, double* out) {
  return guard([&] {
    const Vec s = normalized_filter_coeffs(k, gamma, damping);
    std::copy(s.begin(), s.end(), out);
  });
}
int se_balance_center(int k, double ta, double tb, int damping, double* gamma) {
  return guard([&] { *gamma = balance_center(k, ta, tb, damping); });
}
int se_find_pol(double xi, double eta, double lmin, double lmax, double tau, int max_deg,
                int damping, se_poly_filter* out) {
  return guard([&] {
    if (!out) fail(SE_EINVAL, "null filter");
    const PolyFilter f = find_pol(xi, eta, lmin, lmax, tau, max_deg, damping);
    if (!out->mu || out->mu_cap < f.k + 1)
      fail(SE_EINVAL, "se_find_pol: mu buffer too small (need max_deg+1)");
    out->k = f.k;
    out->gamma = f.gamma;
    out->c = f.c;
    out->d = f.d;
    out->tau = f.tau;
    out->ta = f.ta;
    out->tb = f.tb;
    out->bar = f.bar;
    out->damping = f.damping;
    out->cap_reached = f.cap_reached;
    std::copy(f.mu.begin(), f.mu.end(), out->mu);
  });
}
int se_eval_pol(const se_poly_filter* f, double t, double* out) {
  return guard([&] {
    if (!f || !f->mu) fail(SE_EINVAL, "null filter");
    *out = eval_pol(f->mu, f->k, t);
  });
}

// ---- spectral density --------------------------------------------------------------------------
namespace {
constexpr int kBlock = 16;

// dos.hpp:96-109 on the device, probes from one host Rng(seed) stream in probe order.
void kpm_moments_impl(Ctx& c, const DevCsr& a, double lmin, double lmax, int m, int n_vec,
                      int probe_kind, std::uint64_t seed, int first, int count, Vec& zeta,
                      Vec* per_probe = nullptr) {
  constexpr bool doubling = true;  // Chebyshev doubling: floor(m/2) block SpMMs instead of m - 1
  if (!(lmin < lmax)) fail(SE_EINVAL, "dos: empty spectral interval");
  if (m < 1 || n_vec < 1) fail(SE_EINVAL, "dos: need m >= 1, n_vec >= 1, npts >= 2");
  if (a.n < 1) fail(SE_EINVAL, "dos: empty operator");
  if (first < 0 || count < 0 || first + count > n_vec) fail(SE_EINVAL, "kpm: probe range");
  const int n = a.n;
  const double cc = 0.5 * (lmax + lmin), d = 0.5 * (lmax - lmin);
  zeta.assign(m + 1, 0.0);
  if (per_probe) per_probe->assign((size_t)count * (m + 1), 0.0);
  if (count == 0) return;
  Rng rng(seed);
  const bool gaussian = probe_kind == SE_PROBE_GAUSSIAN;
  skip_probes(rng, gaussian, n, first);  // the probes owned by other ranks (jump-ahead)
  const size_t blk = (size_t)n * kBlock;
  double *V = dev_alloc<double>(blk), *X[3];
  for (double*& x : X) x = dev_alloc<double>(blk);
  double* dz = dev_alloc<double>((size_t)(m + 3) * kBlock);
  k::Scratch s;
  s.cap = k::kpm_scratch_doubles(c, n);
  s.buf = dev_alloc<double>(s.cap);
  s.cnt = dev_alloc<unsigned>(1);
  s.ncnt = 1;
  SE_CUDA(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned), c.stream));
  // Two pinned staging buffers: the host draws block q+1 (one mt19937_64 stream, probe order)
  // while the device runs the m-step recurrence of block q.
  double* hb[2] = {nullptr, nullptr};
  // staging: a block of double probes (Gaussian) or of sign bits (Rademacher, 1/64 the size;
  // pinning host memory costs ~0.2 ms per MB, so the bit path stays cheap)
  const size_t hcap = gaussian ? blk : (size_t)kBlock * (((size_t)n + 63) / 64);
  SE_CUDA(cudaMallocHost(&hb[0], sizeof(double) * hcap));
  SE_CUDA(cudaMallocHost(&hb[1], sizeof(double) * hcap));
  double* hbuf = hb[0];
  Vec hz((size_t)(m + 3) * kBlock);
  auto fill = [&](int b0, double* buf) {
    // probe j = the next n values of the one stream (probe order), probe-major; the device
    // transposes the block to the row-major layout the kernels read.  Rademacher probes travel
    // as sign bits (n / 8 bytes per probe) and are expanded on the device.
    if (gaussian)
      fill_probes(rng, gaussian, n, std::min(kBlock, count - b0), buf);
    else
      fill_rademacher_bits(rng, n, std::min(kBlock, count - b0), reinterpret_cast<std::uint64_t*>(buf));
  };
  std::future<void> next = std::async(std::launch::async, fill, 0, hb[0]);
  try {
    for (int b0 = 0, q = 0; b0 < count; b0 += kBlock, ++q) {
      const int b = std::min(kBlock, count - b0);
      // odd blocks carry one zero probe column (its moments are dropped): every row of the
      // row-major block is then 16-byte aligned for the kernels' paired loads
      const int bk = b + (b & 1);
      next.get();
      hbuf = hb[q & 1];
      if (gaussian) {
        if (bk != b) std::fill(hbuf + (size_t)n * b, hbuf + (size_t)n * bk, 0.0);
        SE_CUDA(cudaMemcpyAsync(X[2], hbuf, sizeof(double) * (size_t)n * bk, cudaMemcpyHostToDevice, c.stream));
        k::transpose_probes(c, X[2], V, n, bk);
      } else {
        const size_t words = ((size_t)n + 63) / 64;
        SE_CUDA(cudaMemcpyAsync(X[2], hbuf, sizeof(std::uint64_t) * words * b, cudaMemcpyHostToDevice, c.stream));
        k::expand_rademacher(c, reinterpret_cast<const std::uint64_t*>(X[2]), V, n, b, bk);
      }
      ctx_sync(c);  // hbuf consumed; the other buffer is free
      if (b0 + kBlock < count) next = std::async(std::launch::async, fill, b0 + kBlock, hb[(q + 1) & 1]);
      if (c.time_filter) SE_CUDA(cudaEventRecord(c.ev0, c.stream));
      k::kpm_step(c, s, a, bk, 1, V, V, nullptr, X[0], cc, d, dz, 0);
      const double* w0 = V;
      double *w1 = X[0], *tb = X[1], *spare = X[2];
      // doubling (default): step k gives w_{k+1} and the dots w_k.w_k, w_k.w_{k+1}, i.e. moments
      // 2k and 2k+1 -- floor(m/2) SpMMs instead of m-1; direct: the reference's recurrence.
      const int last = doubling ? m / 2 : m;
      int launched = 1;
      for (int kk = doubling ? 1 : 2; kk <= last; ++kk, ++launched) {
        k::kpm_step(c, s, a, bk, doubling ? 2 : 0, V, w0, w1, tb, cc, d, dz, kk);
        double* freed = (w0 == V) ? spare : const_cast<double*>(w0);  // w0 <- w1 <- t <- free
        w0 = w1;
        w1 = tb;
        tb = freed;
      }
      if (c.time_filter) {
        SE_CUDA(cudaEventRecord(c.ev1, c.stream));
        SE_CUDA(cudaEventSynchronize(c.ev1));
        float ms = 0.f;
        SE_CUDA(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
        c.filter_ms += ms;
        c.filter_launches += launched;
        // block-step bytes: direct Abytes + 32 n b; doubling drops the probe
        // stream (Abytes + 24 n b)
        c.filter_bytes += (double)launched * (a.abytes() + (doubling ? 24.0 : 32.0) * n * bk);
      }
      const int slots = doubling ? 2 * (last + 1) : m + 1;
      SE_CUDA(cudaMemcpyAsync(hz.data(), dz, sizeof(double) * (size_t)slots * bk,
                              cudaMemcpyDeviceToHost, c.stream));
      ctx_sync(c);
      if (doubling) {  // zeta_2k = 2 w_k.w_k - zeta_0, zeta_2k+1 = 2 w_k.w_k+1 - zeta_1
        for (int j = 0; j < b; ++j) {
          const double z0 = hz[j], z1 = hz[(size_t)bk + j];
          for (int kk = 2; kk <= m; ++kk) {
            const double raw = hz[(size_t)kk * bk + j];
            hz[(size_t)kk * bk + j] = 2.0 * raw - ((kk & 1) ? z1 : z0);
          }
        }
      }
      for (int j = 0; j < b; ++j)  // probe order (dos.hpp:100-106)
        for (int kk = 0; kk <= m; ++kk) {
          zeta[kk] += hz[(size_t)kk * bk + j];
          if (per_probe) (*per_probe)[(size_t)(b0 + j) * (m + 1) + kk] = hz[(size_t)kk * bk + j];
        }
    }
  } catch (...) {
    if (next.valid()) next.wait();
    cudaStreamSynchronize(c.stream);
    cudaFreeHost(hb[0]);
    cudaFreeHost(hb[1]);
    for (void* p : {(void*)V, (void*)X[0], (void*)X[1], (void*)X[2], (void*)dz, (void*)s.buf, (void*)s.cnt})
      dev_free(p);
    throw;
  }
  cudaFreeHost(hb[0]);
  cudaFreeHost(hb[1]);
  for (void* p : {(void*)V, (void*)X[0], (void*)X[1], (void*)X[2], (void*)dz, (void*)s.buf, (void*)s.cnt})
    dev_free(p);
}
}  // namespace

int se_kpm_moments(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec,
                   int probe_kind, uint64_t seed, int first, int count, double* zeta_sums) {
  return guard([&] {
    Vec z;
    kpm_moments_impl(C(ctx), M(a), lmin, lmax, m, n_vec, probe_kind, seed, first, count, z);
    std::copy(z.begin(), z.end(), zeta_sums);
  });
}

int se_kpm_moments_probes(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m,
                          int n_vec, int probe_kind, uint64_t seed, int first, int count,
                          double* per_probe) {
  return guard([&] {
    Vec z, pp;
    kpm_moments_impl(C(ctx), M(a), lmin, lmax, m, n_vec, probe_kind, seed, first, count, z, &pp);
    std::copy(pp.begin(), pp.end(), per_probe);
  });
}

int se_probe_block(uint64_t seed, int probe_kind, int n, long first, int count, double* out) {
  return guard([&] {
    if (n < 1 || first < 0 || count < 0) fail(SE_EINVAL, "se_probe_block: bad sizes");
    if (probe_kind != SE_PROBE_GAUSSIAN && probe_kind != SE_PROBE_RADEMACHER)
      fail(SE_EINVAL, "se_probe_block: unknown probe kind");
    Rng rng(seed);
    const bool gaussian = probe_kind == SE_PROBE_GAUSSIAN;
    skip_probes(rng, gaussian, n, first);
    std::vector<double> blk;
    for (int b0 = 0; b0 < count; b0 += 16) {  // the device's probe blocks
      const int b = std::min(16, count - b0);
      blk.resize((size_t)n * b);
      fill_probes(rng, gaussian, n, b, blk.data());
      for (int l = 0; l < b; ++l)
        for (int i = 0; i < n; ++i) out[(size_t)i * count + b0 + l] = blk[(size_t)l * n + i];
    }
  });
}

int se_kpm_curve(int m, const double* zeta, int n, double lmin, double lmax, int npts, double* x,
                 double* y, double* nev_est) {
  return guard([&] {
    if (!(lmin < lmax)) fail(SE_EINVAL, "dos: empty spectral interval");
    if (m < 1 || npts < 2) fail(SE_EINVAL, "dos: need m >= 1, n_vec >= 1, npts >= 2");
    const Curve cv = kpm_curve(Vec(zeta, zeta + m + 1), n, lmin, lmax, npts);
    std::copy(cv.x.begin(), cv.x.end(), x);
    std::copy(cv.y.begin(), cv.y.end(), y);
    *nev_est = cv.nev_est;
  });
}

int se_kpm_dos(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec, int npts,
               uint64_t seed, int probe_kind, double* x, double* y, double* nev_est) {
  return guard([&] {
    const DevCsr& mat = M(a);
    if (!(lmin < lmax)) fail(SE_EINVAL, "dos: empty spectral interval");
    if (m < 1 || n_vec < 1 || npts < 2) fail(SE_EINVAL, "dos: need m >= 1, n_vec >= 1, npts >= 2");
    Vec z;
    kpm_moments_impl(C(ctx), mat, lmin, lmax, m, n_vec, probe_kind, seed, 0, n_vec, z);
    for (double& q : z) q /= (double)n_vec * mat.n;  // dos.hpp:110
    const Curve cv = kpm_curve(z, mat.n, lmin, lmax, npts);
    std::copy(cv.x.begin(), cv.x.end(), x);
    std::copy(cv.y.begin(), cv.y.end(), y);
    *nev_est = cv.nev_est;
  });
}

int se_lan_dos(se_ctx* ctx, const se_csr* a, double lmin, double lmax, int m, int n_vec, int npts,
               double sigma, uint64_t seed, double* x, double* y, double* nev_est) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& mat = M(a);
    if (!(lmin < lmax)) fail(SE_EINVAL, "dos: empty spectral interval");
    if (m < 1 || n_vec < 1 || npts < 2) fail(SE_EINVAL, "dos: need m >= 1, n_vec >= 1, npts >= 2");
    if (mat.n < 1) fail(SE_EINVAL, "dos: empty operator");
    const double sg = sigma > 0.0 ? sigma : 0.4 * (lmax - lmin) / std::sqrt((double)m);
    Curve cv;
    cv.n = mat.n;
    cv.x = dos_grid(lmin, lmax, npts);
    cv.y.assign(npts, 0.0);
    Rng rng(seed);
    Vec start(mat.n);
    for (int l = 0; l < n_vec; ++l) {
      rng.normal_fill(start.data(), mat.n);
      const LanczosRun r = lanczos_run(c, mat, start.data(), m, false);
      Vec vals, vecs;
      sym_tridiag_eig(r.alpha, r.beta, true, vals, vecs);
      const int steps = (int)vals.size();
      Vec tau2(steps);
      for (int i = 0; i < steps; ++i) tau2[i] = vecs[(size_t)i * steps] * vecs[(size_t)i * steps];
      add_ritz_gaussians(vals, tau2, cv.x, sg, cv.y);
    }
    dos_finalize(cv);
    std::copy(cv.x.begin(), cv.x.end(), x);
    std::copy(cv.y.begin(), cv.y.end(), y);
    *nev_est = cv.nev_est;
  });
}

int se_dos_count(int npts, int n, const double* x, const double* y, double xi, double eta,
                 double* out) {
  return guard([&] {
    Curve cv;
    cv.n = n;
    cv.x.assign(x, x + npts);
    cv.y.assign(y, y + npts);
    *out = dos_count(cv, xi, eta);
  });
}

int se_slice_spectrum(int npts, int n, const double* x, const double* y, double xi, double eta,
                      int ns, double* breakpoints, double* est_counts) {
  return guard([&] {
    Curve cv;
    cv.n = n;
    cv.x.assign(x, x + std::max(npts, 0));
    cv.y.assign(y, y + std::max(npts, 0));
    Vec bp, est;
    slice_spectrum(cv, xi, eta, ns, bp, est);
    std::copy(bp.begin(), bp.end(), breakpoints);
    std::copy(est.begin(), est.end(), est_counts);
  });
}

// ---- Krylov ------------------------------------------------------------------------------------
int se_lan_tr_bounds(se_ctx* ctx, const se_csr* a, double tol, int restart_dim, int max_restarts,
                     uint64_t seed, double* lmin, double* lmax) {
  return guard([&] { lan_tr_bounds(C(ctx), M(a), tol, restart_dim, max_restarts, seed, *lmin, *lmax); });
}

int se_lanczos_run(se_ctx* ctx, const se_csr* a, const double* start, int m, double* alpha,
                   double* beta, int* steps, int* breakdown, double* next_beta, double* next_w,
                   double* basis) {
  return guard([&] {
    const DevCsr& mat = M(a);
    if (m < 1) fail(SE_EINVAL, "lanczos_run: m must be positive");
    const LanczosRun r = lanczos_run(C(ctx), mat, start, m, basis != nullptr);
    std::copy(r.alpha.begin(), r.alpha.end(), alpha);
    std::copy(r.beta.begin(), r.beta.end(), beta);
    *steps = r.steps;
    *breakdown = r.breakdown;
    *next_beta = r.next_beta;
    if (next_w && !r.next_w.empty()) std::copy(r.next_w.begin(), r.next_w.end(), next_w);
    if (basis) std::copy(r.basis.begin(), r.basis.end(), basis);
  });
}

int se_paired_cgs2(se_ctx* ctx, int n, int kq, const double* W, double* t, double* h) {
  // The product's CGS2 (rowgs.cu): W staged row-major, T1 + fused MID + N2.
  return guard([&] {
    Ctx& c = C(ctx);
    if (n < 1 || kq < 0) fail(SE_EINVAL, "paired_cgs2: bad sizes");
    // orth.hpp:72-73: nothing to do for a zero vector or an empty basis
    double t2 = 0.0;
    for (int r = 0; r < n; ++r) t2 += t[r] * t[r];
    if (kq == 0 || t2 == 0.0) return;
    const int ldw = k::rw_ldw(kq);
    k::RowScratch rs = k::rw_scratch(c, ldw);
    double* dW = dev_alloc<double>((size_t)n * ldw);
    double* dcm = dev_alloc<double>((size_t)n * kq);
    double* dt = dev_alloc<double>(n);
    double* cf = dev_alloc<double>(2 * (size_t)ldw);
    double* rbuf = dev_alloc<double>(k::rw_scratch_doubles(rs));
    Ctl* ctl = dev_alloc<Ctl>(1);
    k::rw_bind(rs, rbuf);
    auto cleanup = [&] {
      for (void* p : {(void*)dW, (void*)dcm, (void*)dt, (void*)cf, (void*)rbuf, (void*)ctl}) dev_free(p);
    };
    try {
      SE_CUDA(cudaMemcpyAsync(dcm, W, sizeof(double) * (size_t)n * kq, cudaMemcpyHostToDevice, c.stream));
      SE_CUDA(cudaMemcpyAsync(dt, t, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
      SE_CUDA(cudaMemsetAsync(dW, 0, sizeof(double) * (size_t)n * ldw, c.stream));
      k::rw_put_cols(c, n, dW, ldw, 0, kq, dcm, n, nullptr);
      Ctl z{};
      z.i = kq - 1;  // columns 0..i
      SE_CUDA(cudaMemcpyAsync(ctl, &z, sizeof(Ctl), cudaMemcpyHostToDevice, c.stream));
      k::rw_cgs2(c, rs, n, dt, dW, ldw, ctl, nullptr, cf, cf + ldw, true);
      Vec co(2 * (size_t)ldw);
      Ctl hh;
      SE_CUDA(cudaMemcpyAsync(&hh, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
      SE_CUDA(cudaMemcpyAsync(co.data(), cf, sizeof(double) * co.size(), cudaMemcpyDeviceToHost, c.stream));
      SE_CUDA(cudaMemcpyAsync(t, dt, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
      ctx_sync(c);
      if (h)
        for (int q = 0; q < kq; ++q) {
          h[q] += co[q];                       // pass 1 (orth.hpp:30)
          if (hh.npass == 2) h[q] += co[ldw + q];  // the DGKS re-pass (orth.hpp:77-78)
        }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int se_sym_tridiag_eig(int m, const double* alpha, const double* beta, int want, double* values,
                       double* vectors) {
  return guard([&] {
    if (m < 0) fail(SE_EINVAL, "sym_tridiag_eig: negative size");
    Vec a(alpha, alpha + m), b;
    if (m > 1) b.assign(beta, beta + m - 1);
    Vec vals, vecs;
    sym_tridiag_eig(a, b, want != 0, vals, vecs);
    std::copy(vals.begin(), vals.end(), values);
    if (want && vectors) std::copy(vecs.begin(), vecs.end(), vectors);
  });
}

int se_arrow_tridiag(int l, const double* theta, const double* s, double alpha_l, double* diag,
                     double* off) {
  return guard([&] {
    if (l < 0) fail(SE_EINVAL, "arrow_tridiag: negative size");
    Vec d, o;
    arrow_to_tridiag(Vec(theta, theta + l), Vec(s, s + l), alpha_l, d, o);
    std::copy(d.begin(), d.end(), diag);
    std::copy(o.begin(), o.end(), off);
  });
}

int se_dense_sym_eig(int m, const double* a, int want, int size_guard, double* values,
                     double* vectors) {
  return guard([&] {
    if (m > (size_guard > 0 ? size_guard : 5000))
      fail(SE_EINVAL, "dense_sym_eig: matrix exceeds the size guard");
    Vec vals, vecs;
    dense_sym_eig(m, a, want != 0, vals, vecs);
    std::copy(vals.begin(), vals.end(), values);
    if (want && vectors) std::copy(vecs.begin(), vecs.end(), vectors);
  });
}

// ---- slice drivers -------------------------------------------------------------------------------
int se_cheb_lan(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, double xi, double eta,
                const se_solver_cfg* cfg, int solver, int ndefl, const double* defl_u,
                const double* defl_vals, int want_vectors, se_results** out) {
  (void)want_vectors;
  return guard([&] {
    *out = nullptr;
    const char* who = solver == 1 ? "cheb_lan_tr" : "cheb_lan_nr";
    Ctx& c = C(ctx);
    if (!(eta > xi)) fail(SE_EINVAL, std::string(who) + ": degenerate interval");
    const SolverCfg sc = resolve_config(cfg, who);
    const PolyFilter pf = to_filter(f);
    auto res = std::make_unique<se_results>();
    res->device = c.device;
    res->r = cheb_lan(c, M(a), pf, xi, eta, sc, solver == 1, ndefl, defl_u, defl_vals, who);
    *out = res.release();
  });
}

int se_cheb_si(se_ctx* ctx, const se_csr* a, const se_poly_filter* f, double xi, double eta,
               int est_count, const se_solver_cfg* cfg, se_results** out) {
  return guard([&] {
    *out = nullptr;
    Ctx& c = C(ctx);
    if (!(eta > xi)) fail(SE_EINVAL, "cheb_si: degenerate interval");
    if (est_count < 0) fail(SE_EINVAL, "cheb_si: negative est_count");
    // NULL selects the defaults, as in se_cheb_lan (resolve_config);
    // est_count = max(cfg.est_count, est_count) (eigensolvers.hpp:770-772)
    se_solver_cfg rc = cfg ? *cfg : se_solver_cfg{0, 0, 30, 0.0, 1e-8, 20, 1234};
    rc.est_count = std::max(rc.est_count, est_count);
    const SolverCfg sc = resolve_config(&rc, "cheb_si");
    auto res = std::make_unique<se_results>();
    res->device = c.device;
    res->r = cheb_si(c, M(a), to_filter(f), xi, eta, est_count, sc);
    *out = res.release();
  });
}

// ---- general SPD-B pencils ------------------------------------------------------------------
int se_ls_pol_approx(int fun, double lmin, double lmax, double tol, int max_deg, int cap,
                     int* degree, double* coeff, double* achieved) {
  return guard([&] {
    const ChebFit f = ls_pol_approx(fun == SE_FUN_INVSQRT, lmin, lmax, tol, max_deg);
    if ((int)f.coeff.size() > cap) fail(SE_EINVAL, "ls_pol_approx: coefficient buffer too small");
    std::copy(f.coeff.begin(), f.coeff.end(), coeff);
    *degree = (int)f.coeff.size() - 1;
    if (achieved) *achieved = f.achieved;
  });
}

int se_apply_cheb(se_ctx* ctx, const se_csr* b, double lmin, double lmax, int degree,
                  const double* coeff, int nvec, const double* x, double* y) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& B = M(b);
    if (degree < 0 || !(lmax > lmin) || nvec < 0) fail(SE_EINVAL, "apply_cheb: bad arguments");
    const size_t len = (size_t)B.n * nvec;
    if (len == 0) return;
    double* dx = dev_alloc<double>(len);
    double* dy = dev_alloc<double>(len);
    try {
      h2d(c, dx, x, sizeof(double) * len);
      if (degree == 0) {  // y = c0 x
        k::scale_copy(c, (int)len, coeff[0], dx, dy);
      } else {
        StepOp op;
        op.plain = false;
        op.k = degree;
        op.mu.assign(coeff, coeff + degree + 1);
        op.c = 0.5 * (lmax + lmin);
        op.invd = 1.0 / (0.5 * (lmax - lmin));
        apply_filter_dev(c, B, op, nvec, dx, dy);
      }
      d2h(c, y, dy, sizeof(double) * len);
      ctx_sync(c);
    } catch (...) {
      dev_free(dx);
      dev_free(dy);
      throw;
    }
    dev_free(dx);
    dev_free(dy);
  });
}

int se_pencil_create(se_ctx* ctx, const se_csr* b, double tol, int max_deg, se_pencil** out) {
  return guard([&] {
    *out = nullptr;
    Ctx& c = C(ctx);
    const DevCsr& B = M(b);
    if (B.n < 1) fail(SE_EINVAL, "pencil: empty B");
    // B's spectrum (the reference bounds its pencils the same way, lanczos.hpp:148-277), widened
    // so the B^-1/2 fit covers it; B must be SPD
    double lo = 0.0, hi = 0.0;
    lan_tr_bounds(c, B, 1e-4, 60, 40, 1234, lo, hi);
    if (!(lo > 0.0)) fail(SE_EINVAL, "pencil: B is not positive definite");
    auto h = std::make_unique<se_pencil>();
    h->bmin = 0.9 * lo;
    h->bmax = 1.05 * hi;
    const ChebFit f = ls_pol_approx(true, h->bmin, h->bmax, tol > 0.0 ? tol : 1e-13,
                                    max_deg > 0 ? max_deg : 300);
    h->achieved = f.achieved;
    h->p.B = &B;
    h->p.P.plain = false;
    h->p.P.k = (int)f.coeff.size() - 1;
    h->p.P.mu = f.coeff;
    h->p.P.c = 0.5 * (h->bmax + h->bmin);
    h->p.P.invd = 1.0 / (0.5 * (h->bmax - h->bmin));
    if (h->p.P.k < 1) {  // keep at least one recurrence degree for the fused kernel
      h->p.P.k = 1;
      h->p.P.mu.push_back(0.0);
    }
    *out = h.release();
  });
}

int se_pencil_info(const se_pencil* p, int* degree, double* bmin, double* bmax, double* achieved) {
  return guard([&] {
    if (!p) fail(SE_EINVAL, "null se_pencil");
    if (degree) *degree = p->p.P.k;
    if (bmin) *bmin = p->bmin;
    if (bmax) *bmax = p->bmax;
    if (achieved) *achieved = p->achieved;
  });
}

int se_pencil_free(se_pencil* p) {
  delete p;
  return SE_OK;
}

int se_lan_tr_bounds_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p, double tol,
                            int restart_dim, int max_restarts, uint64_t seed, double* lmin,
                            double* lmax) {
  return guard([&] {
    if (!p) fail(SE_EINVAL, "null se_pencil");
    lan_tr_bounds(C(ctx), M(a), tol, restart_dim, max_restarts, seed, *lmin, *lmax, &p->p);
  });
}

int se_lan_dos_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p, double lmin, double lmax,
                      int m, int n_vec, int npts, double sigma, uint64_t seed, double* x,
                      double* y, double* nev_est) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& mat = M(a);
    if (!p) fail(SE_EINVAL, "null se_pencil");
    if (!(lmin < lmax)) fail(SE_EINVAL, "dos: empty spectral interval");
    if (m < 1 || n_vec < 1 || npts < 2) fail(SE_EINVAL, "dos: need m >= 1, n_vec >= 1, npts >= 2");
    // dos_generalized (dos.hpp:160-184): Lanczos on S = P A P from Gaussian probes (the
    // reference's L^-T g start is a Gaussian probe of the equivalent standard problem too)
    const double sg = sigma > 0.0 ? sigma : 0.4 * (lmax - lmin) / std::sqrt((double)m);
    Curve cv;
    cv.n = mat.n;
    cv.x = dos_grid(lmin, lmax, npts);
    cv.y.assign(npts, 0.0);
    Rng rng(seed);
    Vec start(mat.n);
    for (int l = 0; l < n_vec; ++l) {
      rng.normal_fill(start.data(), mat.n);
      const LanczosRun r = lanczos_run(c, mat, start.data(), m, false, &p->p);
      Vec vals, vecs;
      sym_tridiag_eig(r.alpha, r.beta, true, vals, vecs);
      const int steps = (int)vals.size();
      Vec tau2(steps);
      for (int i = 0; i < steps; ++i) tau2[i] = vecs[(size_t)i * steps] * vecs[(size_t)i * steps];
      add_ritz_gaussians(vals, tau2, cv.x, sg, cv.y);
    }
    dos_finalize(cv);
    std::copy(cv.x.begin(), cv.x.end(), x);
    std::copy(cv.y.begin(), cv.y.end(), y);
    *nev_est = cv.nev_est;
  });
}

int se_cheb_lan_pencil(se_ctx* ctx, const se_csr* a, const se_pencil* p, const se_poly_filter* f,
                       double xi, double eta, const se_solver_cfg* cfg, int solver,
                       se_results** out) {
  return guard([&] {
    *out = nullptr;
    if (!p) fail(SE_EINVAL, "null se_pencil");
    const char* who = solver == 1 ? "cheb_lan_tr" : "cheb_lan_nr";
    Ctx& c = C(ctx);
    if (M(a).n != p->p.B->n) fail(SE_EINVAL, std::string(who) + ": pencil size mismatch");
    if (!(eta > xi)) fail(SE_EINVAL, std::string(who) + ": degenerate interval");
    const SolverCfg sc = resolve_config(cfg, who);
    auto res = std::make_unique<se_results>();
    res->device = c.device;
    res->r = cheb_lan(c, M(a), to_filter(f), xi, eta, sc, solver == 1, 0, nullptr, nullptr, who,
                      &p->p);
    *out = res.release();
  });
}

int se_results_count(const se_results* r, int* nev) {
  return guard([&] {
    if (!r) fail(SE_EINVAL, "null results");
    *nev = (int)r->r->eigenvalues.size();
  });
}

int se_results_copy(const se_results* r, double* eigenvalues, double* residuals, double* vectors) {
  return guard([&] {
    if (!r) fail(SE_EINVAL, "null results");
    const SliceResult& s = *r->r;
    if (eigenvalues) std::copy(s.eigenvalues.begin(), s.eigenvalues.end(), eigenvalues);
    if (residuals) std::copy(s.residuals.begin(), s.residuals.end(), residuals);
    if (vectors && !s.eigenvalues.empty()) {
      SE_CUDA(cudaSetDevice(r->device));
      SE_CUDA(cudaMemcpy(vectors, s.vectors.p, sizeof(double) * (size_t)s.n * s.eigenvalues.size(),
                         cudaMemcpyDeviceToHost));
    }
  });
}

int se_results_vector(const se_results* r, int index, double* vector) {
  return guard([&] {
    if (!r || !vector) fail(SE_EINVAL, "se_results_vector: null argument");
    const SliceResult& s = *r->r;
    if (index < 0 || index >= (int)s.eigenvalues.size())
      fail(SE_ERANGE, "se_results_vector: eigenpair index out of range");
    SE_CUDA(cudaSetDevice(r->device));
    SE_CUDA(cudaMemcpy(vector, s.vectors.col(index), sizeof(double) * (size_t)s.n,
                       cudaMemcpyDeviceToHost));
  });
}

int se_results_info(const se_results* r, long* niter, int* hit_max_its, se_counters* counters) {
  return guard([&] {
    if (!r) fail(SE_EINVAL, "null results");
    if (niter) *niter = r->r->niter;
    if (hit_max_its) *hit_max_its = r->r->hit_max_its;
    if (counters) *counters = r->r->counters;
  });
}

int se_results_orth(const se_results* r, long long* passes, long long* cols, double* bytes) {
  return guard([&] {
    if (!r) fail(SE_EINVAL, "null results");
    if (passes) *passes = r->r->orth_passes;
    if (cols) *cols = r->r->orth_cols;
    if (bytes) *bytes = r->r->orth_bytes;
  });
}

int se_results_free(se_results* r) {
  return guard([&] {
    if (!r) return;
    cudaSetDevice(r->device);
    devmat_free(r->r->vectors);  // stream-ordered if this thread's context is on the device
    delete r;
  });
}

// ---- checks ---------------------------------------------------------------------------------------
int se_rayleigh_residual(se_ctx* ctx, const se_csr* a, const double* u, double* lambda,
                         double* residual) {
  return guard([&] {
    Ctx& c = C(ctx);
    const DevCsr& m = M(a);
    double* du = dev_alloc<double>(m.n);
    double* dau = dev_alloc<double>(m.n);
    double* st = dev_alloc<double>(3);
    SE_CUDA(cudaMemcpyAsync(du, u, sizeof(double) * m.n, cudaMemcpyHostToDevice, c.stream));
    StepOp op;
    apply_filter_dev(c, m, op, 1, du, dau);
    k::candidate_stats(c, m.n, 1, du, dau, st, m.resw);
    double h[3];
    SE_CUDA(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    ctx_sync(c);
    for (void* p : {(void*)du, (void*)dau, (void*)st}) dev_free(p);
    if (!(h[2] > 0.0)) fail(SE_EINVAL, "rayleigh_and_residual: zero (or B-degenerate) vector");
    *lambda = h[0];
    // candidate_stats reports ||Au - lambda u|| / sqrt(uu); rayleigh_and_residual does not scale
    *residual = h[1] * std::sqrt(h[2]);
  });
}

}  // extern "C"
