// Host->device for query-sized transfers: copy engine (cudaMemcpyAsync, back to
// back on one stream) vs SMs pulling the pinned host buffer over the link
// (UVA: a cudaHostAlloc'd buffer is device-addressable) with 16-byte loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 h2d_pull.cu -o h2d_pull
//   ./h2d_pull [bytes=1437696] [reps=400]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void pull(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  constexpr int U = 8;  // 16-byte loads in flight per thread
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < n16; base += stride * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * stride;
      if (i < n16) v[u] = __ldcs(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * stride;
      if (i < n16) dst[i] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? strtoull(argv[1], 0, 10) : 1437696;
  const int reps = argc > 2 ? atoi(argv[2]) : 400;
  const int nbuf = 8;
  void* h[nbuf];
  for (int i = 0; i < nbuf; ++i) {
    cudaHostAlloc(&h[i], bytes, cudaHostAllocDefault);
    memset(h[i], 1, bytes);
  }
  void* d;
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int w = 0; w < 2; ++w) {
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) cudaMemcpyAsync(d, h[r % nbuf], bytes, cudaMemcpyHostToDevice, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy engine: %zu B x %d: %.1f GB/s (%.2f us each)\n", bytes, reps,
         reps * (double)bytes / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
  const size_t n16 = bytes / 16;
  for (int ctas : {8, 16, 32, 64, 148, 296}) {
    for (int thr : {256, 512}) {
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(e0, s);
        for (int r = 0; r < reps; ++r)
          pull<<<ctas, thr, 0, s>>>(static_cast<const int4*>(h[r % nbuf]), static_cast<int4*>(d), n16);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("SM pull %3d CTAs x %d: %.1f GB/s (%.2f us each)%s\n", ctas, thr,
             reps * (double)bytes / (ms * 1e-3) / 1e9, ms * 1e3 / reps,
             cudaGetLastError() == cudaSuccess ? "" : " ERROR");
    }
  }
  // both at once: the copy engine on one stream, SM pulls on another (half each)
  cudaStream_t s2;
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (int w = 0; w < 2; ++w) {
    cudaEventRecord(e0, s);
    cudaStreamWaitEvent(s2, e0, 0);
    for (int r = 0; r < reps; ++r) {
      cudaMemcpyAsync(d, h[r % nbuf], bytes / 2, cudaMemcpyHostToDevice, s);
      pull<<<64, 256, 0, s2>>>(static_cast<const int4*>(h[(r + 1) % nbuf]) + n16 / 2,
                              static_cast<int4*>(d) + n16 / 2, n16 / 2);
    }
    cudaEventRecord(e1, s2);
    cudaStreamWaitEvent(s, e1, 0);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1);
  printf("split CE + SM pull: %.1f GB/s (%.2f us per query)\n",
         reps * (double)bytes / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
  return 0;
}
