// Feasibility probe (experiment, not shipped): do green-context SM partitions hold for kernels
// launched directly, for graphs captured on a green stream, and for a fork/join capture spanning
// two green contexts?  Prints the distinct SM ids each launch ran on.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("CU err %s at %d\n", s, __LINE__); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("RT err %s at %d\n", cudaGetErrorString(r), __LINE__); return 1; } } while (0)

__global__ void k_smid(int* out, long long spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}

static std::set<int> sms(int* h, int n) { return std::set<int>(h, h + n); }

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs total %u\n", all.sm.smCount);
  CUdevResource part[1], rest;
  unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(part, &ng, &all, &rest, 0, 72));
  printf("split: group %u SMs, remaining %u SMs\n", part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dA, dB;
  CK(cuDevResourceGenerateDesc(&dA, &part[0], 1));
  CK(cuDevResourceGenerateDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  const int N = 1024;
  int *dA_out, *dB_out;
  RK(cudaMalloc(&dA_out, N * sizeof(int)));
  RK(cudaMalloc(&dB_out, N * sizeof(int)));
  std::vector<int> h(N);
  // 1) direct launches
  k_smid<<<N, 128, 0, (cudaStream_t)sA>>>(dA_out, 20000);
  k_smid<<<N, 128, 0, (cudaStream_t)sB>>>(dB_out, 20000);
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), dA_out, N * 4, cudaMemcpyDeviceToHost));
  auto a1 = sms(h.data(), N);
  RK(cudaMemcpy(h.data(), dB_out, N * 4, cudaMemcpyDeviceToHost));
  auto b1 = sms(h.data(), N);
  int ov = 0; for (int s : a1) ov += b1.count(s);
  printf("direct: A on %zu SMs, B on %zu SMs, overlap %d\n", a1.size(), b1.size(), ov);
  // 2) graph captured on green stream A, replayed on A and on a plain stream
  cudaGraph_t g; cudaGraphExec_t ge;
  RK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
  k_smid<<<N, 128, 0, (cudaStream_t)sA>>>(dA_out, 20000);
  RK(cudaStreamEndCapture((cudaStream_t)sA, &g));
  RK(cudaGraphInstantiate(&ge, g, 0));
  cudaStream_t plain; RK(cudaStreamCreateWithFlags(&plain, cudaStreamNonBlocking));
  RK(cudaMemset(dA_out, 0xff, N * 4));
  RK(cudaGraphLaunch(ge, plain));
  RK(cudaDeviceSynchronize());
  RK(cudaMemcpy(h.data(), dA_out, N * 4, cudaMemcpyDeviceToHost));
  auto a2 = sms(h.data(), N);
  int in_a = 0; for (int s : a2) in_a += a1.count(s);
  printf("graph(captured on A) replayed on plain stream: %zu SMs, %d of them in A's set\n", a2.size(), in_a);
  // 3) fork/join capture: A kernel -> event -> B kernel, one graph
  cudaEvent_t e1, e2; RK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming)); RK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
  cudaGraph_t g2; cudaGraphExec_t ge2;
  cudaError_t rc = cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal);
  printf("begin capture: %s\n", cudaGetErrorString(rc));
  k_smid<<<N, 128, 0, (cudaStream_t)sA>>>(dA_out, 20000);
  rc = cudaEventRecord(e1, (cudaStream_t)sA); printf("record on A: %s\n", cudaGetErrorString(rc));
  rc = cudaStreamWaitEvent((cudaStream_t)sB, e1, 0); printf("B waits: %s\n", cudaGetErrorString(rc));
  k_smid<<<N, 128, 0, (cudaStream_t)sB>>>(dB_out, 20000);
  rc = cudaEventRecord(e2, (cudaStream_t)sB); printf("record on B: %s\n", cudaGetErrorString(rc));
  rc = cudaStreamWaitEvent((cudaStream_t)sA, e2, 0); printf("A joins: %s\n", cudaGetErrorString(rc));
  rc = cudaStreamEndCapture((cudaStream_t)sA, &g2); printf("end capture: %s\n", cudaGetErrorString(rc));
  if (rc == cudaSuccess) {
    RK(cudaGraphInstantiate(&ge2, g2, 0));
    RK(cudaMemset(dA_out, 0xff, N * 4)); RK(cudaMemset(dB_out, 0xff, N * 4));
    RK(cudaGraphLaunch(ge2, plain));
    RK(cudaDeviceSynchronize());
    RK(cudaMemcpy(h.data(), dA_out, N * 4, cudaMemcpyDeviceToHost));
    auto a3 = sms(h.data(), N);
    RK(cudaMemcpy(h.data(), dB_out, N * 4, cudaMemcpyDeviceToHost));
    auto b3 = sms(h.data(), N);
    int ia = 0, ib = 0; for (int s : a3) ia += a1.count(s); for (int s : b3) ib += b1.count(s);
    printf("fork/join graph: A-node on %zu SMs (%d in A), B-node on %zu SMs (%d in B)\n", a3.size(), ia, b3.size(), ib);
  }
  // 4) overlap timing: two long kernels concurrently on A and B
  cudaEvent_t t0, t1; RK(cudaEventCreate(&t0)); RK(cudaEventCreate(&t1));
  RK(cudaEventRecord(t0, plain)); RK(cudaStreamWaitEvent((cudaStream_t)sA, t0, 0)); RK(cudaStreamWaitEvent((cudaStream_t)sB, t0, 0));
  k_smid<<<N, 128, 0, (cudaStream_t)sA>>>(dA_out, 2000000);
  k_smid<<<N, 128, 0, (cudaStream_t)sB>>>(dB_out, 2000000);
  cudaEvent_t ea, eb; RK(cudaEventCreate(&ea)); RK(cudaEventCreate(&eb));
  RK(cudaEventRecord(ea, (cudaStream_t)sA)); RK(cudaEventRecord(eb, (cudaStream_t)sB));
  RK(cudaStreamWaitEvent(plain, ea, 0)); RK(cudaStreamWaitEvent(plain, eb, 0));
  RK(cudaEventRecord(t1, plain)); RK(cudaEventSynchronize(t1));
  float ms; RK(cudaEventElapsedTime(&ms, t0, t1));
  printf("two 2M-cycle kernels on A and B: %.3f ms\n", ms);
  return 0;
}
