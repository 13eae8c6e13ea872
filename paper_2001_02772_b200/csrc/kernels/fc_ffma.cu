// fc_ffma.cu — fp32 FFMA path for the FC stacks (DenseFC, PredictFC;
// proj/src/model_zoo.cpp:187-190, 240-243). This is the tight-parity path and
// the small-batch path: every output is one sequential fmaf chain over k,
// then + bias, then ReLU (hidden layers) or identity (last predict layer).
//
// Tile 32 (items) x 64 (outputs) per 128-thread CTA, 4x4 register micro-tile
// per thread laid out strided (rows ty + 8i, cols tx + 16j) so that the
// 128-bit shared-memory reads along k are conflict-free (row pitch 36 floats
// = 9 x 16 B). K advances 32 at a time through a 3-stage cp.async ring, so up
// to two K slabs are in flight while one is consumed: the K loop is bound
// by FMA issue, not by global-memory latency. Batched over predict stacks on
// grid.z; the item count M is read from the device query descriptor so one
// captured graph serves every query size (blocks past S exit immediately).
#include "common.cuh"
#include "kernels.hpp"

namespace rs {
namespace {

constexpr int BM = 32, BN = 64, BK = 32, STAGES = 3, PITCH = BK + 4;
constexpr int THREADS = 128;

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(THREADS)
fc_ffma_kernel(const QDesc* __restrict__ qd, FcArgs a) {
  __shared__ __align__(16) float As[STAGES][BM][PITCH];
  __shared__ __align__(16) float Bs[STAGES][BN][PITCH];
  const int64_t M = qd->S;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN, z = blockIdx.z;
  if (m0 >= M) return;
  pdl_wait();  // A is the previous layer's output
  const float* __restrict__ A = a.A + (int64_t)z * a.sAz;
  const float* __restrict__ W = a.W + (int64_t)z * a.sWz;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 8
  const int Kp = (a.K + 3) & ~3;
  const int nk = (Kp + BK - 1) / BK;

  // Loader: A slab = 32 rows x 8 float4 (2 per thread), W slab = 64 x 8 (4 per thread).
  auto load = [&](int stage, int kb) {
    const int k0 = kb * BK;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + r * THREADS;
      const int row = e >> 3, c4 = (e & 7) * 4;
      const int64_t m = m0 + row;
      const bool ok = m < M && k0 + c4 < Kp;
      cp_async16(&As[stage][row][c4], ok ? A + m * a.lda + k0 + c4 : A, ok);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * THREADS;
      const int row = e >> 3, c4 = (e & 7) * 4;
      const int n = n0 + row;
      const bool ok = n < a.N && k0 + c4 < Kp;
      cp_async16(&Bs[stage][row][c4], ok ? W + (int64_t)n * a.ldw + k0 + c4 : W, ok);
    }
  };

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_async_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // refill the slot consumed in the previous iteration
    const int nxt = kb + STAGES - 1;
    if (nxt < nk) load(nxt % STAGES, nxt);
    cp_async_commit();
    const int st = kb % STAGES;
#pragma unroll
    for (int k = 0; k < BK; k += 4) {
      float4 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(&As[st][ty + 8 * i][k]);
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(&Bs[st][tx + 16 * j][k]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float c = acc[i][j];
          c = fmaf(av[i].x, bv[j].x, c);
          c = fmaf(av[i].y, bv[j].y, c);
          c = fmaf(av[i].z, bv[j].z, c);
          c = fmaf(av[i].w, bv[j].w, c);
          acc[i][j] = c;
        }
    }
  }
  cp_async_wait<0>();
  // trigger late: the next layer's CTAs launch during this epilogue instead
  // of holding registers and shared memory through the whole main loop
  pdl_trigger();

  float* __restrict__ C = ((a.c_desc && qd->out) ? qd->out : a.C) + (int64_t)z * a.sCz;
  const float* __restrict__ bias = a.bias + (int64_t)z * a.sbz;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty + 8 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= a.N) continue;
      float y = acc[i][j] + __ldg(bias + n);
      if (a.relu) y = fmaxf(y, 0.f);
      C[m * a.ldc + n] = y;
    }
  }
}

}  // namespace

void launch_fc_ffma(const QDesc* qd, const FcArgs& a, int64_t max_items, cudaStream_t s) {
  const dim3 grid((a.N + BN - 1) / BN, (unsigned)((max_items + BM - 1) / BM), a.batch);
  launch_pdl(fc_ffma_kernel, grid, dim3(THREADS), 0, s, qd, a);
}

}  // namespace rs
