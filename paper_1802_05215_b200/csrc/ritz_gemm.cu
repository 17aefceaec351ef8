// Rayleigh-Ritz dense contractions (K6 of SURVEY.md §2.1) on the fp64 tensor cores:
//   * Ritz combinations  U = W Y      (eigensolvers.hpp:275-283 via mult_cols, vecops.hpp:81-89;
//                                      thick-restart vectors eigensolvers.hpp:600-612)
//   * subspace iteration  G = T^T (A T), Y = T V   (eigensolvers.hpp:838-871)
//   * deflation-set Gram  L^T L        (eigensolvers.hpp:160-176)
// These are the only dense fp64 contractions of the path (2 n s c flop against 8 n s bytes: far
// above the HBM ridge), so they run on DMMA (mma.sync.m8n8k4.f64, the one f64 tensor-core shape;
// tcgen05 has no f64 kind).  One kernel covers all of them:
//
//   C[M x N] (column-major, ldc) = A[M x K] B[K x N],   B[k + col ldb],
//   A[row lda + k]  (K-contiguous: the row-major Krylov basis, or X^T for a column-major X), or
//   A[row + k lda]  (M-contiguous: a column-major block),
//
// with an optional split of K over blockIdx.z (tall-skinny Gram products; partials are reduced in
// split order by k_splitk_reduce, so results are deterministic).
//
// CTA = 128 x 64 tile, 8 warps (4 x 2), warp tile 32 x 32 = 4 x 4 DMMA tiles; K advances 16 at a
// time through a 3-stage cp.async ring (24 KB a stage).  Shared rows are padded to a stride of
// 4 (mod 16) doubles so the fragment loads (lane -> row lane / 4, k lane % 4) are conflict-free.
// CTAs that share an A row block (different column tiles) are adjacent in launch order, so the
// basis is fetched from HBM once and re-read from L2.
#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace se {
namespace k {

namespace {

constexpr int kBM = 128, kBN = 64, kBK = 16, kStages = 3;
constexpr int kLdK = kBK + 4;    // K-contiguous tiles: [row][k], stride 20 doubles
constexpr int kLdM = kBM + 4;    // M-contiguous A tile: [k][row], stride 132 doubles
constexpr int kGemmThreads = 256;

__device__ __forceinline__ void cp_async_16(void* smem, const void* g, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* g, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

struct GemmArgs {
  int M, N, K;
  const double* A;
  long lda;
  const double* B;
  long ldb;
  double* C;
  long ldc;
  int ksplit;       // K elements per blockIdx.z (multiple of kBK); == K when unsplit
  long cz_stride;   // C offset per split (partials)
};

// AK: A is K-contiguous (A[row lda + k]); else M-contiguous (A[row + k lda]).
// A16: every A row start / k0 offset is 16-byte aligned (16-byte copies), else 8-byte copies.
template <bool AK, bool A16>
__global__ void __launch_bounds__(kGemmThreads, 2) k_ritz_gemm(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  constexpr int kASz = AK ? kBM * kLdK : kBK * kLdM;
  constexpr int kBSz = kBN * kLdK;
  double* sA = smem;
  double* sB = smem + kStages * kASz;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;      // warp tile origin: rows 32 wm, cols 32 wn
  const int col0 = blockIdx.x * kBN;             // column tile fastest: neighbours share A rows
  const long row0 = (long)blockIdx.y * kBM;
  const int kbeg = blockIdx.z * g.ksplit;
  const int kend = min(g.K, kbeg + g.ksplit);
  const int nk = (kend - kbeg + kBK - 1) / kBK;
  double* __restrict__ C = g.C + (long)blockIdx.z * g.cz_stride;

  auto load_stage = [&](int st, int kt) {
    const int k0 = kbeg + kt * kBK;
    double* a = sA + st * kASz;
    double* b = sB + st * kBSz;
    if (AK) {
      if (A16) {  // 128 rows x 8 chunks of 2 doubles
        for (int q = tid; q < kBM * (kBK / 2); q += kGemmThreads) {
          const int r = q >> 3, c2 = (q & 7) * 2;
          const bool ok = row0 + r < g.M && k0 + c2 < kend;
          // K tail: an odd kend copies one double (the rest of the chunk is zero-filled)
          cp_async_16(a + r * kLdK + c2, g.A + (ok ? (row0 + r) * g.lda + k0 + c2 : 0),
                      ok ? min(16, 8 * (kend - k0 - c2)) : 0);
        }
      } else {
        for (int q = tid; q < kBM * kBK; q += kGemmThreads) {
          const int r = q >> 4, c = q & 15;
          const bool ok = row0 + r < g.M && k0 + c < kend;
          cp_async_8(a + r * kLdK + c, g.A + (ok ? (row0 + r) * g.lda + k0 + c : 0), ok);
        }
      }
    } else {  // 16 k x 128 rows, rows contiguous
      for (int q = tid; q < kBK * kBM; q += kGemmThreads) {
        const int kk = q >> 7, r = q & 127;
        const bool ok = row0 + r < g.M && k0 + kk < kend;
        cp_async_8(a + kk * kLdM + r, g.A + (ok ? (long)(k0 + kk) * g.lda + row0 + r : 0), ok);
      }
    }
    for (int q = tid; q < kBN * kBK; q += kGemmThreads) {
      const int cc = q >> 4, kk = q & 15;
      const bool ok = col0 + cc < g.N && k0 + kk < kend;
      cp_async_8(b + cc * kLdK + kk, g.B + (ok ? (long)(col0 + cc) * g.ldb + k0 + kk : 0), ok);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;  // fragment coordinates
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();  // stage kt landed for everyone; stage kt-1's readers are done
    if (kt + kStages - 1 < nk) load_stage((kt + kStages - 1) % kStages, kt + kStages - 1);
    cp_commit();
    const double* a = sA + (kt % kStages) * kASz;
    const double* b = sB + (kt % kStages) * kBSz;
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 32 * wm + 8 * i + fr;
        af[i] = AK ? a[r * kLdK + k4 + fk] : a[(k4 + fk) * kLdM + r];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b[(32 * wn + 8 * j + fr) * kLdK + k4 + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_wait<0>();
  // epilogue: lane holds C[row fr][cols 2 fk, 2 fk + 1] of each 8 x 8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long r = row0 + 32 * wm + 8 * i + fr;
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = col0 + 32 * wn + 8 * j + 2 * fk;
      if (cc < g.N) C[(long)cc * g.ldc + r] = acc[i][j][0];
      if (cc + 1 < g.N) C[(long)(cc + 1) * g.ldc + r] = acc[i][j][1];
    }
  }
}

// C = sum over splits of the partials, in split order (deterministic).
__global__ void k_splitk_reduce(int M, int N, int splits, const double* __restrict__ part,
                                long pz, double* __restrict__ C, long ldc) {
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long)M * N) return;
  const int r = (int)(e % M), cc = (int)(e / M);
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += part[(long)z * pz + (long)cc * M + r];
  C[(long)cc * ldc + r] = s;
}

template <bool AK, bool A16>
void launch(Ctx& c, const GemmArgs& g, dim3 grid) {
  constexpr int kASz = AK ? kBM * kLdK : kBK * kLdM;
  constexpr size_t smem = sizeof(double) * kStages * (kASz + kBN * kLdK);
  static bool once = false;  // per instantiation
  if (!once) {
    SE_CUDA(cudaFuncSetAttribute(k_ritz_gemm<AK, A16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    once = true;
  }
  k_ritz_gemm<AK, A16><<<grid, kGemmThreads, smem, c.stream>>>(g);
  SE_CUDA(cudaGetLastError());
  ++c.launches;
}

}  // namespace

void ritz_gemm(Ctx& c, int M, int N, int K, const double* A, long lda, bool a_kcontig,
               const double* B, long ldb, double* C, long ldc) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    for (int j = 0; j < N; ++j) SE_CUDA(cudaMemsetAsync(C + (long)j * ldc, 0, sizeof(double) * M, c.stream));
    return;
  }
  GemmArgs g{M, N, K, A, lda, B, ldb, C, ldc, K, 0};
  const unsigned mt = (unsigned)((M + kBM - 1) / kBM), nt = (unsigned)((N + kBN - 1) / kBN);
  // tall-skinny in K (Gram products: K = n rows, M, N = block width): split K so the grid fills
  // the device (at least two waves of CTAs), partials reduced in order
  int splits = 1;
  const long tiles = (long)mt * nt;
  if (tiles < 2L * c.num_sms && K >= 64 * kBK) {
    splits = (int)std::min<long>((2L * c.num_sms + tiles - 1) / tiles, K / (8 * kBK));
    splits = std::max(1, std::min(splits, 512));
  }
  double* part = nullptr;
  if (splits > 1) {
    g.ksplit = (((K + splits - 1) / splits) + kBK - 1) / kBK * kBK;
    splits = (K + g.ksplit - 1) / g.ksplit;
    part = dev_alloc<double>((size_t)splits * M * N);
    g.C = part;
    g.ldc = M;
    g.cz_stride = (long)M * N;
  }
  if (mt > 65535u) fail(SE_EINVAL, "ritz_gemm: more than 8M rows");  // grid.y limit
  const dim3 grid(nt, mt, (unsigned)splits);
  const bool a16 = a_kcontig && (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                   (g.ksplit % 2 == 0);
  if (a_kcontig) {
    if (a16)
      launch<true, true>(c, g, grid);
    else
      launch<true, false>(c, g, grid);
  } else {
    launch<false, false>(c, g, grid);
  }
  if (splits > 1) {
    const long tot = (long)M * N;
    k_splitk_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, c.stream>>>(M, N, splits, part,
                                                                         (long)M * N, C, ldc);
    SE_CUDA(cudaGetLastError());
    ++c.launches;
    dev_free(part);  // stream-ordered
  }
}

}  // namespace k
}  // namespace se
