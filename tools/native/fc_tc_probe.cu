// Direct (non-graph) launch of one tcgen05 FC layer through the library's
// internal planner: error codes and max |err| vs an fp64 host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I../../include -I../../paper_2001_02772_b200/csrc \
//     fc_tc_probe.cu -L../../paper_2001_02772_b200 -lrecsys_b200 -o fc_tc_probe
//   RS_TC2=1 ./fc_tc_probe M N K [batch] [reps]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels/common.cuh"
#include "kernels/kernels.hpp"

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));     \
      return 2;                                                                       \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 512, N = argc > 2 ? atoi(argv[2]) : 512,
            K = argc > 3 ? atoi(argv[3]) : 1024, B = argc > 4 ? atoi(argv[4]) : 1,
            reps = argc > 5 ? atoi(argv[5]) : 20;
  std::vector<float> hA((size_t)B * M * K), hW((size_t)B * N * K), hb((size_t)B * N);
  srand(1);
  for (auto& v : hA) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto& v : hW) v = ((float)rand() / RAND_MAX - 0.5f) * 0.1f;
  for (auto& v : hb) v = (float)rand() / RAND_MAX - 0.5f;
  float *A, *W, *bias, *C;
  rs::QDesc* qd;
  CK(cudaMalloc(&A, hA.size() * 4));
  CK(cudaMalloc(&W, hW.size() * 4));
  CK(cudaMalloc(&bias, hb.size() * 4));
  CK(cudaMalloc(&C, (size_t)B * M * N * 4));
  CK(cudaMalloc(&qd, sizeof(rs::QDesc)));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(W, hW.data(), hW.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(bias, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  rs::QDesc h{};
  h.S = M;
  CK(cudaMemcpy(qd, &h, sizeof(h), cudaMemcpyHostToDevice));
  rs::FcArgs a{};
  a.A = A; a.lda = K; a.sAz = B > 1 ? (int64_t)M * K : 0;
  a.W = W; a.ldw = K; a.sWz = (int64_t)N * K;
  a.bias = bias; a.sbz = N;
  a.C = C; a.ldc = N; a.sCz = (int64_t)M * N;
  a.N = N; a.K = K; a.relu = 1; a.batch = B;
  rs::TcPlan p;
  if (!rs::tc_plan(&p, a, M, M)) {
    printf("plan failed\n");
    return 1;
  }
  printf("cfg %d block_n %d grid %d x %d x %d\n", p.cfg, p.block_n, p.n_tiles, p.m_tiles, B);
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  rs::launch_fc_tc(qd, p, a, s);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  std::vector<float> hC((size_t)B * M * N);
  CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
  double maxrel = 0;
  for (int z = 0; z < B; ++z)
    for (int m = 0; m < M; m += 7)
      for (int n = 0; n < N; ++n) {
        double acc = hb[(size_t)z * N + n], mag = fabs(acc);
        for (int k = 0; k < K; ++k) {
          const double t = (double)hA[((size_t)z * M + m) * K * (B > 1) + (size_t)m * K * (B == 1) + k] *
                           hW[((size_t)z * N + n) * K + k];
          acc += t;
          mag += fabs(t);
        }
        if (acc < 0) acc = 0;
        const double d = fabs(acc - hC[((size_t)z * M + m) * N + n]) / mag;
        if (d > maxrel) maxrel = d;
      }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps; ++r) rs::launch_fc_tc(qd, p, a, s);
  cudaEventRecord(e1, s);
  CK(cudaStreamSynchronize(s));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / reps;
  printf("max |d|/mag %.3g (tf32 bound 2^-10 = %.3g)  %.2f us/launch  %.1f TFLOP/s\n", maxrel,
         1.0 / 1024, us, 2.0 * B * M * N * K / us * 1e-6);
  return maxrel <= 1.0 / 1024 ? 0 : 1;
}
