// Multi-GPU KPM inside one process (SURVEY.md §8e "KPM probes: one exchange"): the C++ callers
// (the facade's kpm_dos_devices, the CLI's --gpus N) run the probe split with one host thread per
// GPU and combine the per-probe moments with ONE ncclAllReduce over NVLink/NVSwitch.
//
// Determinism: rank g owns probes [first_g, first_g + count_g) and writes only those rows of an
// n_vec x (m+1) array that is zero elsewhere, so the all-reduce sums each entry with exact zeros
// (x + 0 = x in any order) and returns the full per-probe matrix bit for bit.  The host then sums
// the rows in probe order (dos.hpp:100-106), so the curve equals se_kpm_dos on one GPU exactly,
// for any GPU count.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring a copy already loaded in the
// process): a Python process shares torch's NCCL, and the library has no link-time NCCL
// dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"
#include "host_algos.hpp"

namespace {

struct Nccl {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*version)(int*) = nullptr;
  std::string load_error;
};

const Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  std::call_once(once, [] {
    // An NCCL already in the process (e.g. the one torch links) wins: a second copy under the
    // same soname would shadow it for libraries loaded later.  SLICEEIG_NCCL names a specific
    // library; else the loader's libnccl.so.2.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* path = std::getenv("SLICEEIG_NCCL")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if (!h) h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.load_error = std::string("NCCL not found: ") + dlerror();
      return;
    }
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.version = reinterpret_cast<decltype(api.version)>(dlsym(h, "ncclGetVersion"));
    if (!api.comm_init_all || !api.all_reduce || !api.comm_destroy || !api.error_string)
      api.load_error = "NCCL library lacks the expected entry points";
  });
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    se::fail(SE_ENUMERIC, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

namespace se {
void set_last_error(const std::string& msg);  // capi.cpp: the se_last_error() slot
}

namespace {
struct ErrSlot {
  ErrSlot& operator=(const std::string& m) {
    se::set_last_error(m);
    return *this;
  }
} t_err;
}  // namespace

extern "C" {

SE_API int se_nccl_version(int* version) {
  const Nccl& api = nccl();
  if (!api.load_error.empty() || !api.version) {
    t_err = api.load_error.empty() ? "ncclGetVersion missing" : api.load_error;
    if (version) *version = 0;
    return SE_ECUDA;
  }
  int v = 0;
  api.version(&v);
  if (version) *version = v;
  return SE_OK;
}

SE_API int se_kpm_moments_multi(int ngpu, const int* devices, int n, const int* row_ptr,
                                const int* col_idx, const double* vals, double lmin, double lmax,
                                int m, int n_vec, int probe_kind, uint64_t seed, double* per_probe) {
  if (ngpu < 1 || !devices || n < 1 || !row_ptr || !per_probe) {
    t_err = "se_kpm_moments_multi: bad arguments";
    return SE_EINVAL;
  }
  if (m < 1 || n_vec < 1) {
    t_err = "dos: need m >= 1, n_vec >= 1, npts >= 2";
    return SE_EINVAL;
  }
  const Nccl& api = nccl();
  if (!api.load_error.empty()) {
    t_err = api.load_error;
    return SE_ECUDA;
  }
  // contiguous probe ranges in whole blocks of 16 where possible (the device block size)
  std::vector<int> first(ngpu), count(ngpu);
  {
    const int blocks = (n_vec + 15) / 16;
    if (blocks >= ngpu) {
      for (int g = 0, b0 = 0; g < ngpu; ++g) {
        const int nb = blocks / ngpu + (g < blocks % ngpu);
        first[g] = std::min(n_vec, b0 * 16);
        count[g] = std::min(n_vec, (b0 + nb) * 16) - first[g];
        b0 += nb;
      }
    } else {
      for (int g = 0, p0 = 0; g < ngpu; ++g) {
        const int np = n_vec / ngpu + (g < n_vec % ngpu);
        first[g] = p0;
        count[g] = np;
        p0 += np;
      }
    }
  }
  const size_t row = (size_t)m + 1, total = (size_t)n_vec * row;
  std::vector<ncclComm_t> comms(ngpu, nullptr);
  {
    ncclResult_t r = api.comm_init_all(comms.data(), ngpu, devices);
    if (r != ncclSuccess) {
      t_err = std::string("ncclCommInitAll: ") + api.error_string(r);
      return SE_ECUDA;
    }
  }
  std::vector<int> rc(ngpu, SE_OK);
  std::vector<std::string> err(ngpu);
  std::vector<std::thread> pool;
  std::mutex out_mu;
  for (int g = 0; g < ngpu; ++g)
    pool.emplace_back([&, g] {
      se_ctx* ctx = nullptr;
      se_csr* a = nullptr;
      double* buf = nullptr;
      auto bail = [&](int code, std::string msg) {
        rc[g] = code;
        err[g] = std::move(msg);
      };
      int code = se_ctx_create(devices[g], &ctx);
      if (code == SE_OK) code = se_csr_upload(ctx, n, row_ptr, col_idx, vals, &a);
      std::vector<double> mine((size_t)count[g] * row);
      if (code == SE_OK && count[g] > 0)
        code = se_kpm_moments_probes(ctx, a, lmin, lmax, m, n_vec, probe_kind, seed, first[g],
                                     count[g], mine.data());
      if (code != SE_OK) bail(code, se_last_error());
      // every rank joins the all-reduce even after a local failure (a failed rank contributes
      // zeros and the call reports its error), so no peer waits forever
      cudaStream_t st = nullptr;
      try {
        SE_CUDA(cudaSetDevice(devices[g]));
        SE_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        SE_CUDA(cudaMalloc(&buf, sizeof(double) * total));
        SE_CUDA(cudaMemsetAsync(buf, 0, sizeof(double) * total, st));
        if (rc[g] == SE_OK && count[g] > 0)
          SE_CUDA(cudaMemcpyAsync(buf + (size_t)first[g] * row, mine.data(),
                                  sizeof(double) * mine.size(), cudaMemcpyHostToDevice, st));
        nccl_ok(api.all_reduce(buf, buf, total, ncclFloat64, ncclSum, comms[g], st), "ncclAllReduce");
        if (g == 0) {
          std::lock_guard<std::mutex> lk(out_mu);
          SE_CUDA(cudaMemcpyAsync(per_probe, buf, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
        }
        SE_CUDA(cudaStreamSynchronize(st));
      } catch (const se::Error& e) {
        if (rc[g] == SE_OK) bail(e.code, e.what());
      } catch (const std::exception& e) {
        if (rc[g] == SE_OK) bail(SE_ENUMERIC, e.what());
      }
      if (buf) cudaFree(buf);
      if (st) cudaStreamDestroy(st);
      if (a) se_csr_free(a);
      if (ctx) se_ctx_destroy(ctx);
    });
  for (auto& t : pool) t.join();
  for (ncclComm_t c : comms)
    if (c) api.comm_destroy(c);
  for (int g = 0; g < ngpu; ++g)
    if (rc[g] != SE_OK) {
      t_err = "GPU " + std::to_string(devices[g]) + ": " + err[g];
      return rc[g];
    }
  return SE_OK;
}

SE_API int se_kpm_dos_multi(int ngpu, const int* devices, int n, const int* row_ptr,
                            const int* col_idx, const double* vals, double lmin, double lmax, int m,
                            int n_vec, int npts, uint64_t seed, int probe_kind, double* x, double* y,
                            double* nev_est) {
  if (!(lmin < lmax)) {
    t_err = "dos: empty spectral interval";
    return SE_EINVAL;
  }
  if (m < 1 || n_vec < 1 || npts < 2) {
    t_err = "dos: need m >= 1, n_vec >= 1, npts >= 2";
    return SE_EINVAL;
  }
  std::vector<double> pp((size_t)n_vec * (m + 1));
  int rc = se_kpm_moments_multi(ngpu, devices, n, row_ptr, col_idx, vals, lmin, lmax, m, n_vec,
                                probe_kind, seed, pp.data());
  if (rc != SE_OK) return rc;
  std::vector<double> zeta(m + 1, 0.0);
  for (int l = 0; l < n_vec; ++l)  // probe order (dos.hpp:100-106)
    for (int k = 0; k <= m; ++k) zeta[k] += pp[(size_t)l * (m + 1) + k];
  for (double& q : zeta) q /= (double)n_vec * n;  // dos.hpp:110
  return se_kpm_curve(m, zeta.data(), n, lmin, lmax, npts, x, y, nev_est);
}

}  // extern "C"

