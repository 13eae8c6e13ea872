// fc_ffma.cu — fp32 FFMA path for the FC stacks (DenseFC, PredictFC;
// proj/src/model_zoo.cpp:187-190, 240-243). This is the tight-parity path and
// the small-batch path: every output is one sequential fmaf chain over k,
// then + bias, then ReLU (hidden layers) or identity (last predict layer).
//
// 64x64 output tile per 256-thread CTA, 4x4 register micro-tile per thread,
// K staged 16 at a time through double-buffered shared memory with register
// prefetch of the next slab. Batched over predict stacks on grid.z; the item
// count M is read from the device query descriptor so one captured graph
// serves every query size (blocks past S exit immediately).
#include "common.cuh"
#include "kernels.hpp"

namespace rs {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256)
fc_ffma_kernel(const QDesc* __restrict__ qd, FcArgs a) {
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int64_t M = qd->S;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN, z = blockIdx.z;
  if (m0 >= M) return;
  const float* __restrict__ A = a.A + (int64_t)z * a.sAz;
  const float* __restrict__ W = a.W + (int64_t)z * a.sWz;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int lrow = tid >> 2, lk = (tid & 3) * 4;
  const int Kp = (a.K + 3) & ~3;

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  auto load_a = [&](int k0) -> float4 {
    const int64_t m = m0 + lrow;
    const int k = k0 + lk;
    if (m < M && k < Kp) return __ldg(reinterpret_cast<const float4*>(A + m * a.lda + k));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto load_w = [&](int k0) -> float4 {
    const int n = n0 + lrow;
    const int k = k0 + lk;
    if (n < a.N && k < Kp) return __ldg(reinterpret_cast<const float4*>(W + (int64_t)n * a.ldw + k));
    return make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto store = [&](int buf, const float4& va, const float4& vw) {
    As[buf][lk + 0][lrow] = va.x; As[buf][lk + 1][lrow] = va.y;
    As[buf][lk + 2][lrow] = va.z; As[buf][lk + 3][lrow] = va.w;
    Bs[buf][lk + 0][lrow] = vw.x; Bs[buf][lk + 1][lrow] = vw.y;
    Bs[buf][lk + 2][lrow] = vw.z; Bs[buf][lk + 3][lrow] = vw.w;
  };

  float4 ra = load_a(0), rw = load_w(0);
  store(0, ra, rw);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < Kp; k0 += BK) {
    const bool more = k0 + BK < Kp;
    if (more) {
      ra = load_a(k0 + BK);
      rw = load_w(k0 + BK);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 av = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float ar[4] = {av.x, av.y, av.z, av.w};
      const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
    if (more) {
      store(buf ^ 1, ra, rw);
      __syncthreads();
      buf ^= 1;
    }
  }

  float* __restrict__ C = a.C + (int64_t)z * a.sCz;
  const float* __restrict__ bias = a.bias + (int64_t)z * a.sbz;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
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
  fc_ffma_kernel<<<grid, 256, 0, s>>>(qd, a);
}

}  // namespace rs
