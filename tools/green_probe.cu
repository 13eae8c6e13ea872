// green_probe.cu — feasibility probe: can the forward's CUDA graphs and
// runtime launches target an SM partition (green context) while the memory
// and graphs live in the primary context? Records the SM id of every CTA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/green_probe tools/green_probe.cu
//   /tmp/green_probe [dense_sms=16]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <set>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)
#define CD(x)                                                         \
  do {                                                                \
    CUresult r = (x);                                                 \
    if (r != CUDA_SUCCESS) {                                          \
      printf("%s:%d %s -> CUresult %d\n", __FILE__, __LINE__, #x, r); \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

__global__ void smid_kernel(int* out, const float4* src, float4* dst, long n) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)smid;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    float4 v = src[i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  dst[(long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !p) {
    printf("missing %s\n", name);
    exit(1);
  }
  return reinterpret_cast<F>(p);
}

int main(int argc, char** argv) {
  const unsigned dense_sms = argc > 1 ? atoi(argv[1]) : 16;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  auto getRes = entry<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
  auto split = entry<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*,
                                  unsigned, unsigned)>("cuDevSmResourceSplitByCount");
  auto genDesc = entry<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
  auto gCreate = entry<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
  auto gStream = entry<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");

  CUdevResource all;
  CD(getRes(0, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  CUdevResource grp[1], rest;
  unsigned ng = 1;
  CD(split(grp, &ng, &all, &rest, 0, dense_sms));
  printf("dense group: %u SMs, rest: %u SMs\n", grp[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dA, dB;
  CD(genDesc(&dA, grp, 1));
  CD(genDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CD(gCreate(&gA, dA, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CD(gCreate(&gB, dB, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CD(gStream(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
  CD(gStream(&sB, gB, CU_STREAM_NON_BLOCKING, 0));

  const long n = 1l << 28;  // 4 GiB of float4
  float4 *src, *dst;
  int* smids;
  const int grid = 148 * 4, block = 256;
  CK(cudaMalloc(&src, n * 16));
  CK(cudaMemset(src, 0, n * 16));
  CK(cudaMalloc(&dst, (size_t)grid * block * 16));
  CK(cudaMallocManaged(&smids, grid * sizeof(int)));

  // a graph captured in the primary context
  cudaStream_t cap;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  smid_kernel<<<grid, block, 0, cap>>>(smids, src, dst, n);
  CK(cudaStreamEndCapture(cap, &g));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));

  auto report = [&](const char* what, cudaStream_t s, bool graph) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0, s));
      if (graph) CK(cudaGraphLaunch(ge, s));
      else smid_kernel<<<grid, block, 0, s>>>(smids, src, dst, n);
      CK(cudaGetLastError());
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
    }
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::set<int> u(smids, smids + grid);
    printf("%-28s distinct SMs %3zu  [%d..%d]  %.3f ms  %.0f GB/s\n", what, u.size(), *u.begin(),
           *u.rbegin(), ms, n * 16 / (ms * 1e-3) / 1e9);
  };
  report("primary stream, launch", cap, false);
  report("primary stream, graph", cap, true);
  report("green B stream, launch", (cudaStream_t)sB, false);
  report("green B stream, graph", (cudaStream_t)sB, true);
  report("green A stream, launch", (cudaStream_t)sA, false);
  report("green A stream, graph", (cudaStream_t)sA, true);
  // (a) capture on the green stream itself, primary context current
  {
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    CK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
    smid_kernel<<<grid, block, 0, (cudaStream_t)sA>>>(smids, src, dst, n);
    CK(cudaStreamEndCapture((cudaStream_t)sA, &g2));
    CK(cudaGraphInstantiate(&ge2, g2, 0));
    CK(cudaGraphLaunch(ge2, (cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    std::set<int> u(smids, smids + grid);
    printf("(a) captured on green A, launched on A: distinct SMs %zu\n", u.size());
  }
  // (b) green context current during capture + instantiate
  {
    auto fromGreen = entry<CUresult (*)(CUcontext*, CUgreenCtx)>("cuCtxFromGreenCtx");
    auto setCur = entry<CUresult (*)(CUcontext)>("cuCtxSetCurrent");
    auto getCur = entry<CUresult (*)(CUcontext*)>("cuCtxGetCurrent");
    CUcontext prim, cA;
    CD(getCur(&prim));
    CD(fromGreen(&cA, gA));
    CD(setCur(cA));
    cudaGraph_t g3;
    cudaGraphExec_t ge3;
    CK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeThreadLocal));
    smid_kernel<<<grid, block, 0, (cudaStream_t)sA>>>(smids, src, dst, n);
    CK(cudaStreamEndCapture((cudaStream_t)sA, &g3));
    CK(cudaGraphInstantiate(&ge3, g3, 0));
    CK(cudaGraphLaunch(ge3, (cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    std::set<int> u(smids, smids + grid);
    printf("(b) green A current at capture: distinct SMs %zu\n", u.size());
    CD(setCur(prim));
    CK(cudaGraphLaunch(ge3, (cudaStream_t)sA));
    CK(cudaStreamSynchronize((cudaStream_t)sA));
    std::set<int> u2(smids, smids + grid);
    printf("(b') same exec launched with primary current: distinct SMs %zu\n", u2.size());
    CK(cudaGraphLaunch(ge3, cap));
    CK(cudaStreamSynchronize(cap));
    std::set<int> u3(smids, smids + grid);
    printf("(b'') same exec launched on a primary stream: distinct SMs %zu\n", u3.size());
  }
  // (c) one graph whose nodes live on two partitions: capture on B, fork to A
  {
    int* smids2;
    CK(cudaMallocManaged(&smids2, grid * sizeof(int)));
    cudaEvent_t fork, join;
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    cudaGraph_t g4;
    cudaGraphExec_t ge4;
    CK(cudaStreamBeginCapture((cudaStream_t)sB, cudaStreamCaptureModeThreadLocal));
    CK(cudaEventRecord(fork, (cudaStream_t)sB));
    CK(cudaStreamWaitEvent((cudaStream_t)sA, fork, 0));
    smid_kernel<<<grid, block, 0, (cudaStream_t)sA>>>(smids2, src, dst, n / 8);
    CK(cudaEventRecord(join, (cudaStream_t)sA));
    smid_kernel<<<grid, block, 0, (cudaStream_t)sB>>>(smids, src, dst, n);
    CK(cudaStreamWaitEvent((cudaStream_t)sB, join, 0));
    CK(cudaStreamEndCapture((cudaStream_t)sB, &g4));
    CK(cudaGraphInstantiate(&ge4, g4, 0));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaGraphLaunch(ge4, cap));
      CK(cudaStreamSynchronize(cap));
    }
    std::set<int> u(smids, smids + grid), u2(smids2, smids2 + grid);
    printf("(c) mixed graph on a primary stream: B-node SMs %zu, A-node SMs %zu\n", u.size(),
           u2.size());
  }
  // cross-partition event dependency
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaGraphLaunch(ge, (cudaStream_t)sB));
  CK(cudaEventRecord(ev, (cudaStream_t)sB));
  CK(cudaStreamWaitEvent((cudaStream_t)sA, ev, 0));
  smid_kernel<<<grid, block, 0, (cudaStream_t)sA>>>(smids, src, dst, 1024);
  CK(cudaStreamSynchronize((cudaStream_t)sA));
  printf("cross-partition event wait: ok\n");
  return 0;
}
