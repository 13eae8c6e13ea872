// fc_tcgen05.cu — FC layers (DenseFC / PredictFC, proj/src/model_zoo.cpp:187-190,
// 240-243) on the 5th-generation tensor cores.
//
//   C[z][m][n] = act( sum_k A[z][m][k] * W[z][n][k] + bias[z][n] )
//
// kind::tf32: the fp32 activations and weights are consumed straight from
// shared memory (no conversion pass, no second copy of the weights), the
// tensor core rounds operands to tf32 and accumulates in fp32 in TMEM.
// Tolerance for this path is stated in tests/test_gpu_parity.py.
//
// One 128 x BN output tile per CTA, 4 warps (a small CTA: inside the
// pipelined queue these grids share SMs with the gathers of other queries):
//   warp 0  TMEM allocator (BN fp32 columns x 128 lanes); lane 0 is the TMA
//           producer: K slabs of 32 fp32 (=128 B, one SWIZZLE_128B atom row)
//           for A (128 rows) and W (BN rows) into a STAGES-deep ring
//   warp 1  lane 0 issues 4 x tcgen05.mma (K = 8 each) per slab;
//           tcgen05.commit frees the slab / signals the epilogue
//   all 4   epilogue: tcgen05.ld 32x32b.x32 (warp w owns TMEM lanes
//           32w..32w+31 = tile rows), + bias, ReLU, 128-bit stores
// Rows >= S (device query descriptor) are masked at the store; the tile's
// K tail is zero-filled by TMA.
#include <algorithm>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace rs {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per K slab (128 bytes)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm100 format):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major, 1),
// SBO>>4 [32,46) = 1024 B between 8-row groups, version 1 at [46,48),
// layout type SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: D f32 [4,6)=1, A tf32 [7,10)=2, B tf32 [10,13)=2,
// both K-major, N>>3 at [17,23), M>>4 at [24,29).
template <int BN>
__device__ __forceinline__ uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
// kind::f16 with bf16 operands: A bf16 [7,10)=1, B bf16 [10,13)=1, D f32.
template <int BN>
__device__ __forceinline__ uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

// Discard rows [r0, r1) of a row-major buffer (row stride ld bytes) from L2:
// only the 128-byte lines lying entirely inside the range (the partial lines
// at its ends may hold live neighbour rows). All threads of the CTA take part.
__device__ __forceinline__ void discard_rows(const char* base, int64_t ld, int64_t r0,
                                             int64_t r1) {
  if (r1 <= r0) return;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(base + r0 * ld);
  const uintptr_t hi = reinterpret_cast<uintptr_t>(base + r1 * ld);
  const uintptr_t first = (lo + 127) & ~uintptr_t(127), last = hi & ~uintptr_t(127);
  for (uintptr_t p = first + 128 * threadIdx.x; p + 128 <= last; p += 128 * blockDim.x)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// bf16 pair -> one 32-bit word (round to nearest even)
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

template <int BN, int STAGES>
struct TcSmem {
  alignas(1024) float a[STAGES][BM * BK];
  alignas(1024) float b[STAGES][BN * BK];
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full;
  uint32_t tmem_base;
  int last;  // split-K: this CTA completes the tile
};

constexpr int kTcThreads = 128;

// H: bf16 operands (kind::f16, 64 elements = 128 B per k-slab, RS_FC_BF16);
// otherwise fp32 operands rounded to tf32 by the tensor core (32 per slab).
// The k-slab is 128 bytes per row either way, so the shared-memory ring, the
// SW128 descriptors and the 4 MMAs per slab are identical.
template <int BN, int STAGES, bool H = false>
__global__ void __launch_bounds__(kTcThreads, 1)
fc_tc_kernel(const QDesc* __restrict__ qd, const __grid_constant__ CUtensorMap map_a,
             const __grid_constant__ CUtensorMap map_w, FcArgs a, int a_batched) {
  extern __shared__ uint8_t smem_raw[];
  TcSmem<BN, STAGES>& sm = *reinterpret_cast<TcSmem<BN, STAGES>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int64_t M = qd->S;
  // split-K: grid.z = batch x splits; this CTA accumulates k-blocks
  // [kb0, kb0 + nk) of the tile and the last of its splits to arrive sums the
  // partials in split order (deterministic) and runs the epilogue
#if RS_EXPERIMENTS
  const int splits = a.splits > 1 ? a.splits : 1;
#else
  constexpr int splits = 1;
#endif
  const int z = blockIdx.z / splits, sp = blockIdx.z - (blockIdx.z / splits) * splits;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  if (m0 >= M) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KE = H ? 2 * BK : BK;  // operand elements per k-slab
  const int nk_all = (a.K + KE - 1) / KE;
  const int per = (nk_all + splits - 1) / splits;
  const int kb0 = sp * per;
  const int nk = max(0, min(nk_all, kb0 + per) - kb0);
  const int pre = nk < STAGES ? nk : STAGES;  // stages whose weights load before the wait

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  constexpr uint32_t kBytes = (BM + BN) * BK * sizeof(float);
  // Weights do not depend on the previous layer: their first `pre` slabs are
  // in flight before this grid waits on its predecessor (PDL).
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < pre; ++kb) {
      mbar_expect_tx(&sm.full[kb], kBytes);
      tma_load_3d(sm.b[kb], &map_w, &sm.full[kb], (kb0 + kb) * KE, n0, z);
    }
  }
  pdl_wait();  // the activations A are the previous layer's output

  if (warp == 0) {
    // ---- TMA producer (lane 0) ----
    for (int kb = 0; lane == 0 && kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      if (kb >= pre) {
        mbar_wait(&sm.empty[s], ph ^ 1u);
        mbar_expect_tx(&sm.full[s], kBytes);
        tma_load_3d(sm.b[s], &map_w, &sm.full[s], (kb0 + kb) * KE, n0, z);
      }
      if (a_batched) tma_load_3d(sm.a[s], &map_a, &sm.full[s], (kb0 + kb) * KE, m0, z);
      else tma_load_2d(sm.a[s], &map_a, &sm.full[s], (kb0 + kb) * KE, m0);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer (lane 0) ----
    const uint32_t idesc = H ? idesc_bf16<BN>() : idesc_tf32<BN>();
    for (int kb = 0; lane == 0 && kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      mbar_wait(&sm.full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(sm.a[s]), sb = smem_u32(sm.b[s]);
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t da = sw128_desc(sa + kk * 32);
        const uint64_t db = sw128_desc(sb + kk * 32);
        const uint32_t acc = (kb | kk) ? 1u : 0u;
        if constexpr (H)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&sm.empty[s]))
          : "memory");
    }
    if (lane == 0)
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&sm.tmem_full))
          : "memory");
    __syncwarp();
  }
  {
    // ---- epilogue (all warps): TMEM -> registers -> bias/ReLU -> global ----
    mbar_wait(&sm.tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // trigger late (accumulation done): the next layer's CTAs launch during
    // this epilogue instead of squatting on the SM through the main loop
    pdl_trigger();
    if (a.discard_a || a.dz) {
      // every k-slab of this tile's A rows has been consumed (tmem_full): the
      // rows are dead, drop their L2 lines without a DRAM write-back
      const int64_t r1 = min((int64_t)m0 + BM, M);
      if (a.discard_a)
        discard_rows(reinterpret_cast<const char*>(a.A), a.lda * (H ? 2 : 4), m0, r1);
      if (a.dz) discard_rows(reinterpret_cast<const char*>(a.dz), a.dz_ld, m0, r1);
    }
    const int quad = warp;
    const int64_t m = m0 + quad * 32 + lane;
#if RS_EXPERIMENTS
    if (splits > 1) {
      // partial tile -> workspace; the last split to arrive reduces
      const int64_t tile = ((int64_t)z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      const int64_t tiles = (int64_t)(gridDim.z / splits) * gridDim.y * gridDim.x;
      const int rl = quad * 32 + lane;
      float* __restrict__ mine = a.ws + ((int64_t)sp * tiles + tile) * (BM * BN) + rl * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(c * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (m < M) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            __stcg(reinterpret_cast<float4*>(mine + c * 32) + i,
                   make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                               __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
        }
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int old = atomicAdd(a.cnt + tile, 1);
        sm.last = old == splits - 1;
        if (sm.last) a.cnt[tile] = 0;  // ready for the next launch of this graph
      }
      __syncthreads();
      if (sm.last && m < M) {
        __threadfence();
        float* __restrict__ Cb = (a.c_desc && qd->out) ? qd->out : a.C;
        float* __restrict__ C = Cb + (int64_t)z * a.sCz + m * a.ldc;
        const float* __restrict__ bias = a.bias + (int64_t)z * a.sbz;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int nb = n0 + c * 32;
          float y[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) y[i] = 0.f;
          // all splits' loads of a 16-column half in flight before the adds
          // (split order kept: s2 = 0, 1, 2, 3)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float4 t4[4][4];
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
              const float4* src = reinterpret_cast<const float4*>(
                  a.ws + ((int64_t)s2 * tiles + tile) * (BM * BN) + rl * BN + c * 32 + h * 16);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                t4[s2][i] = s2 < splits ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                float* yy = y + h * 16 + 4 * i;
                yy[0] += t4[s2][i].x; yy[1] += t4[s2][i].y; yy[2] += t4[s2][i].z;
                yy[3] += t4[s2][i].w;
              }
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int n = nb + i;
            const float val = y[i] + (n < a.N ? __ldg(bias + n) : 0.f);
            y[i] = a.relu ? fmaxf(val, 0.f) : val;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < a.N) C[nb + i] = y[i];
        }
      }
    } else
#endif  // RS_EXPERIMENTS
    {
    float* __restrict__ Cb = (a.c_desc && qd->out) ? qd->out : a.C;
    float* __restrict__ C = Cb + (int64_t)z * a.sCz + m * a.ldc;
    const float* __restrict__ bias = a.bias + (int64_t)z * a.sbz;
    const bool vec_ok = (a.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(Cb) & 15) == 0) &&
                        (a.sCz % 4 == 0);
    const float* __restrict__ W2 = a.W2 + (int64_t)z * a.sW2z;
    float part[kFuseMaxN2] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(c * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
            "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
            "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
            "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
            "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (m < M) {
        const int nb = n0 + c * 32;
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int n = nb + i;
          float val = __uint_as_float(v[i]) + (n < a.N ? __ldg(bias + n) : 0.f);
          y[i] = a.relu ? fmaxf(val, 0.f) : val;
        }
        if (a.N2 > 0) {
          // fused narrow next layer: this thread owns row m; columns in order
#pragma unroll
          for (int o = 0; o < kFuseMaxN2; ++o) {
            if (o >= a.N2) break;
            const float* __restrict__ w = W2 + (int64_t)o * a.ldw2 + nb;
            float acc2 = part[o];
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (nb + i < a.N) acc2 = fmaf(y[i], __ldg(w + i), acc2);
            part[o] = acc2;
          }
        }
        if (a.skip_c) {
        } else if (a.c16) {
          // bf16 activations for the next bf16 layer: 32 values = 64 bytes
          uint16_t* __restrict__ C16 = reinterpret_cast<uint16_t*>(Cb) + (int64_t)z * a.sCz +
                                       m * a.ldc + nb;
          if (vec_ok && nb + 32 <= a.N && (a.ldc % 8 == 0)) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(C16)[i] =
                  make_uint4(pack_bf16(y[8 * i], y[8 * i + 1]), pack_bf16(y[8 * i + 2], y[8 * i + 3]),
                             pack_bf16(y[8 * i + 4], y[8 * i + 5]),
                             pack_bf16(y[8 * i + 6], y[8 * i + 7]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (nb + i < a.N)
                C16[i] = (uint16_t)(pack_bf16(y[i], 0.f) & 0xFFFFu);
          }
        } else if (vec_ok && nb + 32 <= a.N) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(C + nb)[i] =
                make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (nb + i < a.N) C[nb + i] = y[i];
        }
      }
    }
    if (a.N2 > 0 && m < M) {
      float* __restrict__ C2b = (a.c2_desc && qd->out) ? qd->out : a.C2;
      float* __restrict__ C2 = C2b + (int64_t)z * a.sC2z + m * a.ldc2;
      const float* __restrict__ b2 = a.b2 + (int64_t)z * a.sb2z;
#pragma unroll
      for (int o = 0; o < kFuseMaxN2; ++o) {
        if (o >= a.N2) break;
        const float val = part[o] + __ldg(b2 + o);
        C2[o] = a.relu2 ? fmaxf(val, 0.f) : val;
      }
    }
    }  // splits == 1
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// fc_tc2_kernel: the same layer on a CTA PAIR (cluster of 2 along M = grid x) with
// tcgen05.mma.cta_group::2 — one 256 x BN tile per pair: each CTA stages its
// own 128 rows of A and HALF of the pair's BN weight rows per k-slab, and the
// leader's single MMA thread multiplies the 256-row tile against all BN
// columns, accumulating each CTA's 128 rows in its own TMEM. Per CTA and
// k-slab: 16 KB of A + BN/2 x 128 B of W for 128 x BN x slab flops — half
// the W bytes per flop of a one-CTA tile of the same width, which is what the
// L2 feed bounds for wide layers (§2b). TMA loads of both CTAs complete on
// the LEADER's full barrier (peer bit cleared); the leader's commits arrive
// on both CTAs' empty / tmem_full barriers (multicast mask 0b11).
template <int BN, int STAGES>
struct Tc2Smem {
  alignas(1024) float a[STAGES][BM * BK];
  alignas(1024) float b[STAGES][(BN / 2) * BK];
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full;
  uint32_t tmem_base;
};

constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address of CTA 0

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
               "memory");
}
__device__ __forceinline__ void tma2_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                             int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                             int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void commit2_multicast(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
template <int BN>
__device__ __forceinline__ uint32_t idesc2(bool h) {
  return (1u << 4) | ((h ? 1u : 2u) << 7) | ((h ? 1u : 2u) << 10) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

template <int BN, int STAGES, bool H>
__global__ void __launch_bounds__(kTcThreads, 1)
fc_tc2_kernel(const QDesc* __restrict__ qd, const __grid_constant__ CUtensorMap map_a,
              const __grid_constant__ CUtensorMap map_w, FcArgs a, int a_batched) {
  extern __shared__ uint8_t smem_raw[];
  Tc2Smem<BN, STAGES>& sm = *reinterpret_cast<Tc2Smem<BN, STAGES>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int64_t M = qd->S;
  const uint32_t rank = cluster_rank();
  const int z = blockIdx.z;
  const int n0 = blockIdx.y * BN;
  const int pair_m0 = (int)(blockIdx.x & ~1u) * BM;
  const int m0 = pair_m0 + (int)rank * BM;
  if (pair_m0 >= M) return;  // both CTAs of the pair leave together
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KE = H ? 2 * BK : BK;
  const int nk = (a.K + KE - 1) / KE;
  const int pre = nk < STAGES ? nk : STAGES;
  constexpr uint32_t kBytesPair = 2u * (BM + BN / 2) * BK * sizeof(float);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // barriers of both CTAs initialised before any TMA or commit
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  auto leader_full = [&](int s) { return smem_u32(&sm.full[s]) & kPeerBitMask; };
  const int wrow = n0 + (int)rank * (BN / 2);  // this CTA's half of the weight rows
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < pre; ++kb) {
      if (rank == 0) mbar_expect_tx(&sm.full[kb], kBytesPair);
      tma2_load_3d(smem_u32(sm.b[kb]), &map_w, leader_full(kb), kb * KE, wrow, z);
    }
  }
  pdl_wait();  // A is the previous layer's output

  if (warp == 0) {
    for (int kb = 0; lane == 0 && kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      if (kb >= pre) {
        mbar_wait(&sm.empty[s], ph ^ 1u);
        if (rank == 0) mbar_expect_tx(&sm.full[s], kBytesPair);
        tma2_load_3d(smem_u32(sm.b[s]), &map_w, leader_full(s), kb * KE, wrow, z);
      }
      if (a_batched) tma2_load_3d(smem_u32(sm.a[s]), &map_a, leader_full(s), kb * KE, m0, z);
      else tma2_load_2d(smem_u32(sm.a[s]), &map_a, leader_full(s), kb * KE, m0);
    }
    __syncwarp();
  } else if (warp == 1 && rank == 0) {
    const uint32_t idesc = idesc2<BN>(H);
    for (int kb = 0; lane == 0 && kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
      mbar_wait(&sm.full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(sm.a[s]), sb = smem_u32(sm.b[s]);
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t da = sw128_desc(sa + kk * 32);
        const uint64_t db = sw128_desc(sb + kk * 32);
        const uint32_t acc = (kb | kk) ? 1u : 0u;
        if constexpr (H)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
      }
      commit2_multicast(&sm.empty[s]);
    }
    if (lane == 0) commit2_multicast(&sm.tmem_full);
    __syncwarp();
  }
  {
    // ---- epilogue (all warps of both CTAs: each its own 128 rows) ----
    mbar_wait(&sm.tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pdl_trigger();
    const int64_t m = m0 + warp * 32 + lane;
    float* __restrict__ Cb = (a.c_desc && qd->out) ? qd->out : a.C;
    const float* __restrict__ bias = a.bias + (int64_t)z * a.sbz;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
            "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
            "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
            "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
            "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int nb = n0 + c * 32;
      if (m < M && nb < a.N) {
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int n = nb + i;
          const float val = __uint_as_float(v[i]) + (n < a.N ? __ldg(bias + n) : 0.f);
          y[i] = a.relu ? fmaxf(val, 0.f) : val;
        }
        if (a.c16) {
          uint16_t* __restrict__ C16 =
              reinterpret_cast<uint16_t*>(Cb) + (int64_t)z * a.sCz + m * a.ldc + nb;
          if (nb + 32 <= a.N && a.ldc % 8 == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(C16)[i] = make_uint4(
                  pack_bf16(y[8 * i], y[8 * i + 1]), pack_bf16(y[8 * i + 2], y[8 * i + 3]),
                  pack_bf16(y[8 * i + 4], y[8 * i + 5]), pack_bf16(y[8 * i + 6], y[8 * i + 7]));
          } else {
            for (int i = 0; i < 32; ++i)
              if (nb + i < a.N) C16[i] = (uint16_t)(pack_bf16(y[i], 0.f) & 0xFFFFu);
          }
        } else {
          float* __restrict__ C = Cb + (int64_t)z * a.sCz + m * a.ldc + nb;
          if (nb + 32 <= a.N && a.ldc % 4 == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              reinterpret_cast<float4*>(C)[i] =
                  make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
          } else {
            for (int i = 0; i < 32; ++i)
              if (nb + i < a.N) C[i] = y[i];
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // both CTAs finished with the pair's TMEM and shared memory
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN)
                 : "memory");
  }
}

template <int BN, int STAGES>
size_t tc2_smem_bytes() {
  return sizeof(Tc2Smem<BN, STAGES>) + 1024;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims,
            const cuuint64_t* strides_bytes, const cuuint32_t* box,
            CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B,
            CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dtype, (cuuint32_t)rank, (void*)base, dims,
                  strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int STAGES, bool H = false>
size_t tc_smem_bytes() {
  return sizeof(TcSmem<BN, STAGES>) + 1024;
}

template <int BN, int STAGES, bool H = false>
void set_attr_once() {  // once per device (common.cuh smem_attr)
  smem_attr(reinterpret_cast<const void*>(fc_tc_kernel<BN, STAGES, H>),
            (int)tc_smem_bytes<BN, STAGES>());
}

template <int BN, int STAGES, bool H>
void set_attr2_once() {
  smem_attr(reinterpret_cast<const void*>(fc_tc2_kernel<BN, STAGES, H>),
            (int)tc2_smem_bytes<BN, STAGES>());
}

// launch_pdl plus a (2, 1, 1) cluster: blockIdx.x 2j / 2j+1 form a CTA pair
// (the driver rejects a cta_group::2 kernel whose pair is not along x)
template <typename... KArgs, typename... Args>
cudaError_t launch_pair(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                        cudaStream_t stream, Args&&... args) {
  max_carveout(reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  unsigned n = 0;
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = 2;
  attr[n].val.clusterDim.y = 1;
  attr[n].val.clusterDim.z = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (prio_enabled()) {
    attr[n].id = cudaLaunchAttributePriority;
    attr[n].val.priority = high_priority();
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#if RS_EXPERIMENTS  // measured slower (DESIGN.md Appendix RS_FC_CHAIN)
// ---------------------------------------------------------------------------
// fc_chain_kernel: a whole FC stack per 128-row tile (see TcChainPlan).
// Warps 0-3: epilogue (TMEM lanes 32w..32w+31 = tile rows) and, between
// layers, the writers of the next layer's A operand; warp 4 lane 0: TMA
// producer (layer-0 input, then every layer's weight k-blocks through a
// 2-stage ring, running ahead into the next layer); warp 5 lane 0: MMA issuer.
constexpr int kChainThreads = 192;
constexpr int kChainActAtoms = 8;  // activations up to 256 wide stay in smem
constexpr int kChainMaxStages = 8;
constexpr int kChainRingBytes = 96 * 1024;

// The k-block ring is one byte pool cut into `stages` slots of `slot` bytes
// (planned per stack: [A k-block of the streamed layer-0 input] + the widest
// layer's W k-block), so narrow stacks get a deeper pipeline.
struct ChainSmem {
  alignas(1024) float act[kChainActAtoms][BM * BK];  // SW128 K-major, 16 KB per atom
  alignas(1024) uint8_t ring[kChainRingBytes];
  uint64_t full[kChainMaxStages];
  uint64_t empty[kChainMaxStages];
  uint64_t act_in;     // layer-0 input resident in act
  uint64_t acc_full;   // a layer's accumulation finished
  uint64_t act_ready;  // epilogue wrote the next layer's A (128 arrivals)
  uint32_t tmem_base;
};

// byte offset of fp32 element (row, c) inside a 128-row x 32-col SW128 atom
__device__ __forceinline__ uint32_t chain_sw(int row, int c) {
  return (uint32_t)(row * 128 + ((((c >> 2) ^ row) & 7) << 4) + (c & 3) * 4);
}

__global__ void __launch_bounds__(kChainThreads, 1)
fc_chain_kernel(const QDesc* __restrict__ qd, const __grid_constant__ TcChainPlan p) {
  extern __shared__ uint8_t smem_raw[];
  ChainSmem& sm = *reinterpret_cast<ChainSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int64_t M = qd->S;
  const int m0 = blockIdx.x * BM;
  if (m0 >= M) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.map_a)) : "memory");
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.act_in, 1);
    mbar_init(&sm.acc_full, 1);
    mbar_init(&sm.act_ready, 4 * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  pdl_wait();  // the input rows are the previous kernel's output
  const int L = p.layers;

  if (warp == 4) {
    // ---- TMA producer ----
    if (lane == 0) {
      if (!p.stream_a) {
        const int na = (p.k[0] + BK - 1) / BK;
        mbar_expect_tx(&sm.act_in, (uint32_t)(na * BM * BK * 4));
        for (int a = 0; a < na; ++a) tma_load_2d(sm.act[a], &p.map_a, &sm.act_in, a * BK, m0);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int l = 0; l < L; ++l) {
        const int nk = (p.k[l] + BK - 1) / BK;
        const bool sa = l == 0 && p.stream_a;
        const uint32_t bytes = (uint32_t)(p.np[l] * BK * 4) + (sa ? (uint32_t)(BM * BK * 4) : 0u);
        for (int kb = 0; kb < nk; ++kb) {
          uint8_t* slot = sm.ring + s * p.slot;
          mbar_wait(&sm.empty[s], ph ^ 1u);
          mbar_expect_tx(&sm.full[s], bytes);
          tma_load_2d(slot + p.slot_b, &p.map_w[l], &sm.full[s], kb * BK, 0);
          if (sa) tma_load_2d(slot, &p.map_a, &sm.full[s], kb * BK, m0);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 5) {
    // ---- MMA issuer ----
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int l = 0; l < L; ++l) {
        if (l == 0 && !p.stream_a) mbar_wait(&sm.act_in, 0);
        if (l > 0) mbar_wait(&sm.act_ready, (uint32_t)((l - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                               ((uint32_t)(p.np[l] >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        const bool sa = l == 0 && p.stream_a;
        const int nk = (p.k[l] + BK - 1) / BK;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&sm.full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* slot = sm.ring + s * p.slot;
          const uint32_t sa_addr = smem_u32(sa ? slot : reinterpret_cast<const uint8_t*>(sm.act[kb]));
          const uint32_t sb_addr = smem_u32(slot + p.slot_b);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n}\n" ::"r"(tmem),
                "l"(sw128_desc(sa_addr + kk * 32)), "l"(sw128_desc(sb_addr + kk * 32)),
                "r"(idesc), "r"(acc)
                : "memory");
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  smem_u32(&sm.empty[s]))
              : "memory");
          if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&sm.acc_full))
            : "memory");
      }
    }
  } else {
    // ---- epilogue: warps 0-3, thread = tile row ----
    const int row = warp * 32 + lane;
    const int64_t m = m0 + row;
    for (int l = 0; l < L; ++l) {
      mbar_wait(&sm.acc_full, (uint32_t)(l & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const bool last = l == L - 1;
      if (last) pdl_trigger();
      const float* __restrict__ bias = p.bias[l];
      const int N = p.n[l];
      float part[kFuseMaxN2] = {0.f, 0.f, 0.f, 0.f};
      float* __restrict__ Cb = (p.c_desc && qd->out) ? qd->out : p.C;
      for (int c = 0; c < p.np[l] / 32 + ((p.np[l] & 31) ? 1 : 0); ++c) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32);
        if (c * 32 + 16 < p.np[l]) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(taddr));
        } else {  // a 16-column tail (np % 32 == 16)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(taddr));
#pragma unroll
          for (int i = 16; i < 32; ++i) v[i] = 0u;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int n = c * 32 + i;
          const float val = n < N ? __uint_as_float(v[i]) + __ldg(bias + n) : 0.f;
          y[i] = (p.relu[l] && n < N) ? fmaxf(val, 0.f) : val;
        }
        if (!last) {
          // next layer's A operand: row `row`, columns 32c..32c+31 (zeros past N)
          uint8_t* atom = reinterpret_cast<uint8_t*>(sm.act[c]);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(atom + chain_sw(row, 4 * q)) =
                make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
        } else if (m < M) {
          if (p.N2 > 0) {
#pragma unroll
            for (int o = 0; o < kFuseMaxN2; ++o) {
              if (o >= p.N2) break;
              const float* __restrict__ w = p.W2 + (int64_t)o * p.ldw2 + c * 32;
              float acc2 = part[o];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c * 32 + i < N) acc2 = fmaf(y[i], __ldg(w + i), acc2);
              part[o] = acc2;
            }
          } else {
            float* __restrict__ C = Cb + m * p.ldc;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i < N) C[c * 32 + i] = y[i];
          }
        }
      }
      if (!last) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.act_ready))
                     : "memory");
      } else if (p.N2 > 0 && m < M) {
#pragma unroll
        for (int o = 0; o < kFuseMaxN2; ++o) {
          if (o >= p.N2) break;
          const float val = part[o] + __ldg(p.b2 + o);
          Cb[m * p.ldc + o] = p.relu2 ? fmaxf(val, 0.f) : val;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256)
                 : "memory");
  }
}
#endif  // RS_EXPERIMENTS

}  // namespace

bool tc_available() { return encode_fn() != nullptr; }

// All tables viewed as one [total_rows, D] fp32 matrix; box = one row of D
// elements (the gathered dimension has box extent 1 for tile::gather4).
bool make_row_gather_map(CUtensorMap* map, const float* base, int64_t total_rows, int D) {
  if (total_rows >= (int64_t(1) << 31) || D > 256 || (D * 4) % 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)total_rows};
  cuuint64_t str[1] = {(cuuint64_t)D * 4};
  cuuint32_t box[2] = {(cuuint32_t)D, 1};
  return encode(map, base, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

bool tc_plan(TcPlan* p, const FcArgs& a, int64_t m_cap, int64_t a_rows_per_batch,
             SplitKPool* pool) {
  const int ke = a.ab16 ? 2 * BK : BK;      // operand elements per 128-byte k-slab
  const int esz = a.ab16 ? 2 : 4;          // operand bytes
  const int al = 16 / esz;                 // 16-byte rows for TMA
  if (a.N < 64 || a.K < ke) return false;
  if (a.lda % al || a.ldw % al || (a.sAz % al) || (a.sWz % al)) return false;
  if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(a.W) & 15))
    return false;
  // tile/pipeline configuration: 0 <BN128,3 stages> 1 <64,4> 2 <128,6> 3 <64,8>
  // (RS_TC_CFG overrides, for tools/fc_micro.py). Default: the deep pipelines.
  // A layer CTA is latency-bound (few k-blocks per round trip), and inside the
  // pipelined queue its lifetime is what it costs the concurrent gathers
  // (tools/pipe_micro.py: 44.0 -> 41.4 us/query on cfg3 RMC2 vs <128,3>).
  // Long-K or wide layers (MT-WND's 1640 -> 1024 x 4 stacks) are bound by
  // feeding the tensor cores from L2, not by latency: there two shallower
  // CTAs per SM win (MT-WND 27.0 -> 21.5 us/query), so they keep <128,3>/<64,4>
  // (RS_TC_WIDE_K / RS_TC_WIDE_K1: the K threshold for batched / single stacks).
  const int64_t ctas = (int64_t)((a.N + 127) / 128) * ((m_cap + BM - 1) / BM) * a.batch;
  static const int wide_k = [] {
    const char* e = getenv("RS_TC_WIDE_K");
    return e ? atoi(e) : 1024;
  }();
  // single-stack layers stay deep up to K < 2048: WND's 1640 -> 1024 and
  // 1024 -> 512 run 25% faster pipelined on <128,6> (73.6K -> 91.9K QPS),
  // RMC3's 2560 -> 512 2.4% slower (45.9K -> 44.7K), so it keeps <128,3>
  static const int wide_k1 = [] {
    const char* e = getenv("RS_TC_WIDE_K1");
    return e ? atoi(e) : 2048;
  }();
  // batched stacks (MT-WND's 4 towers) are feed-bound at every layer: the
  // shallow 2-per-SM tiles also for their narrow last layer (512 -> 256:
  // 14.2 -> 13.2 us/query pipelined at 256 items, tools/env_sweep.py)
  const bool wide = a.K >= (a.batch > 1 ? wide_k : wide_k1) || ctas > 148 || a.batch > 1;
  p->cfg = a.N >= 128 ? (wide ? 0 : 2) : (wide ? 1 : 3);
  // cfg 4 <256,4>: one CTA covers 256 output columns (half the CTAs of a
  // 512-wide layer, same k-block round trips per CTA); RS_TC_WIDE=1 selects it
  // for the latency-bound layers with N >= 256
  if (!wide && a.N >= 256 && getenv("RS_TC_WIDE") && atoi(getenv("RS_TC_WIDE"))) p->cfg = 4;
  // batched tf32 stacks of >= 256 outputs (MT-WND's towers): <256,4> halves
  // the re-reads of the shared A tile per flop (MT-WND 18.0 -> 17.0 us/query,
  // 1024-item queries 49.8 -> 46.8; neutral for bf16 operands, whose k-slabs
  // already carry twice the flops: tools/env_sweep.py, profiles/r2_fc_tiles/)
  if (a.batch > 1 && a.N >= 256 && !a.ab16) p->cfg = 4;
  // cfg 5 <256,4> on a CTA pair (fc_tc2_kernel, cta_group::2): 256-row x
  // 256-column tiles, half the W bytes per flop of cfg 4. Planned for layers
  // of >= 256 outputs in the handle's wide graph (a.pair_ok), which serves the
  // queries that fill whole pairs; RS_TC2=2 forces it into every tcgen05 graph
  const char* tc2e = getenv("RS_TC2");  // read per plan (graph capture): tools/env_sweep.py
  const bool tc2 = a.pair_ok || (tc2e && atoi(tc2e) == 2);
  if (tc2 && a.N >= 256 && m_cap > BM) p->cfg = 5;
  if (const char* e = getenv("RS_TC_CFG")) p->cfg = std::min(5, std::max(0, atoi(e)));
  if (p->cfg == 5 && (a.N < 256 || a.N2 > 0 || a.skip_c)) p->cfg = 4;
  if (p->cfg == 4 && a.N < 256) p->cfg = 2;
  const char* pst = getenv("RS_TC2_STAGES");
  p->pair_stages = pst ? (atoi(pst) == 4 ? 4 : 6) : (a.pair_ok == 2 ? 4 : 6);
  // a shared-memory budget (the handle's uniform carveout): the deep 192 KB
  // pipelines give way to the 96 KB shallow ones — for a CTA pair that is a
  // 3-deep ring of 32 KB k-slabs: a.pair_capped (the handle's choice for
  // gather-bound models with substantial FC work; RS_TC2_CAPPED=0/1
  // overrides) puts layers of >= 256 outputs on pairs, half the weight bytes
  // per flop of <128,3> (cfg3 RMC3 21.5 -> 19.6 us/query)
  const bool capped = a.smem_cap_kb > 0 && a.smem_cap_kb < 192 && !getenv("RS_TC_CFG");
  const char* tcc = getenv("RS_TC2_CAPPED");
  const bool cap_pairs = tcc ? atoi(tcc) != 0 : a.pair_capped != 0;
  if (capped && cap_pairs && a.N >= 256 && a.N2 == 0 && !a.skip_c && m_cap > BM &&
      a.smem_cap_kb * 1024 >= (int)(3 * 32 * 1024 + 2048)) {
    p->cfg = 5;
    p->pair_stages = 3;
  } else if (capped) {
    p->cfg = (p->cfg == 2 || p->cfg == 4 || p->cfg == 5) ? 0 : (p->cfg == 3 ? 1 : p->cfg);
  }
  if (a.single_n_tile && a.N <= 128 && (p->cfg == 1 || p->cfg == 3)) p->cfg -= 1;
  if (a.N < 128 && !a.single_n_tile && (p->cfg == 0 || p->cfg == 2)) p->cfg += 1;
  p->block_n = p->cfg >= 4 ? 256 : (p->cfg == 0 || p->cfg == 2) ? 128 : 64;
  p->m_tiles = (int)((m_cap + BM - 1) / BM);
  if (p->cfg == 5) p->m_tiles = (p->m_tiles + 1) & ~1;  // whole CTA pairs
  p->n_tiles = (a.N + p->block_n - 1) / p->block_n;
  // A: [batch][rows][K] (or shared 2D when sAz == 0)
  const CUtensorMapDataType dt =
      a.ab16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (a.sAz != 0) {
    cuuint64_t dims[3] = {(cuuint64_t)a.K, (cuuint64_t)a_rows_per_batch, (cuuint64_t)a.batch};
    cuuint64_t str[2] = {(cuuint64_t)a.lda * esz, (cuuint64_t)a.sAz * esz};
    cuuint32_t box[3] = {(cuuint32_t)ke, BM, 1};
    if (!encode(&p->map_a, a.A, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B, dt)) return false;
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a_rows_per_batch};
    cuuint64_t str[1] = {(cuuint64_t)a.lda * esz};
    cuuint32_t box[2] = {(cuuint32_t)ke, BM};
    if (!encode(&p->map_a, a.A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B, dt)) return false;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)a.K, (cuuint64_t)a.N, (cuuint64_t)a.batch};
    cuuint64_t str[2] = {(cuuint64_t)a.ldw * esz,
                         (cuuint64_t)(a.sWz ? a.sWz : (int64_t)a.N * a.ldw) * esz};
    // a CTA pair stages half of the tile's weight rows per CTA
    cuuint32_t box[3] = {(cuuint32_t)ke, (cuuint32_t)(p->cfg == 5 ? p->block_n / 2 : p->block_n),
                         1};
    if (!encode(&p->map_w, a.W, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B, dt)) return false;
  }
  p->ab16 = a.ab16;
  if (a.ab16) {
    switch (p->cfg) {
      case 0: set_attr_once<128, 3, true>(); break;
      case 1: set_attr_once<64, 4, true>(); break;
      case 2: set_attr_once<128, 6, true>(); break;
      case 4: set_attr_once<256, 4, true>(); break;
      case 5: set_attr2_once<256, 3, true>(); set_attr2_once<256, 4, true>();
              set_attr2_once<256, 6, true>(); break;
      default: set_attr_once<64, 8, true>(); break;
    }
  } else {
    switch (p->cfg) {
      case 0: set_attr_once<128, 3>(); break;
      case 1: set_attr_once<64, 4>(); break;
      case 2: set_attr_once<128, 6>(); break;
      case 4: set_attr_once<256, 4>(); break;
      case 5: set_attr2_once<256, 3, false>(); set_attr2_once<256, 4, false>();
              set_attr2_once<256, 6, false>(); break;
      default: set_attr_once<64, 8>(); break;
    }
  }
  // Split-K for long reductions (K >= 1024: RMC3's 2560 -> 512, MT-WND/WND's
  // 1640 -> 1024), RS_SPLITK=n (2..4) enables: a tile's k-blocks are spread
  // over n CTAs and the last to arrive sums the partials in split order. Off
  // by default: measured slower at every split count (tools/fc_micro.py, K=2560
  // -> 512: 36 us unsplit vs 42-44 us split, independent of n — the layer's
  // time is not in the per-CTA k-block chain). Not with a fused narrow layer.
  p->splits = 1;
  p->ws = nullptr;
  p->cnt = nullptr;
#if RS_EXPERIMENTS
  const char* sk = getenv("RS_SPLITK");
  const int nk = (a.K + BK - 1) / BK;
  if (pool && !a.ab16 && a.N2 == 0 && p->cfg != 5 && nk >= 32 && sk && atoi(sk) > 1) {
    int splits = std::min(std::min(4, atoi(sk)), nk / 16);
    while (splits > 1 && (splits - 1) * ((nk + splits - 1) / splits) >= nk) --splits;
    const size_t tiles = (size_t)a.batch * p->m_tiles * p->n_tiles;
    const size_t ws = (size_t)splits * tiles * BM * p->block_n;
    if (splits > 1 && pool->ws_used + ws <= pool->ws_cap && pool->cnt_used + tiles <= pool->cnt_cap) {
      p->splits = splits;
      p->ws = pool->ws + pool->ws_used;
      p->cnt = pool->cnt + pool->cnt_used;
      pool->ws_used += ws;
      pool->cnt_used += tiles;
    }
  }
#else
  (void)pool;
#endif
  return true;
}

bool tc_chain_plan(TcChainPlan* p, const FcArgs* ly, int L, int64_t m_cap, int64_t a_rows) {
  // Off by default (RS_FC_CHAIN=1 enables): measured slower than one kernel
  // per layer at the zoo/cfg shapes (cfg1 RMC1 9.4 -> 10.3 us/query pipelined,
  // 52 -> 67 us alone): a chain CTA must own whole rows, so a 256-wide layer
  // runs on half the CTAs the per-layer kernels use, and the launches saved
  // do not pay for the lost parallelism.
#if !RS_EXPERIMENTS
  (void)p; (void)ly; (void)L; (void)m_cap; (void)a_rows;
  return false;
#else
  if (!tc_available() || L < 1) return false;
  const char* e = getenv("RS_FC_CHAIN");
  if (!e || !atoi(e)) return false;
  std::memset(p, 0, sizeof(*p));
  // a final layer of <= 4 outputs after a <= 256-wide layer runs in the epilogue
  int nl = L;
  const bool narrow = L >= 2 && ly[L - 1].N <= kFuseMaxN2 && ly[L - 2].N <= 256;
  if (narrow) nl = L - 1;
  if (nl > kChainMaxLayers) return false;
  for (int l = 0; l < L; ++l) {
    const FcArgs& a = ly[l];
    if (a.batch != 1) return false;
    if (a.ldw % 4 || (reinterpret_cast<uintptr_t>(a.W) & 15)) return false;
  }
  if (ly[0].lda % 4 || (reinterpret_cast<uintptr_t>(ly[0].A) & 15)) return false;
  for (int l = 0; l < nl; ++l) {
    if (ly[l].N > 256 || ly[l].N < 16 || ly[l].K < 4) return false;
    if (l > 0 && ly[l].K > kChainActAtoms * BK) return false;
  }
  p->layers = nl;
  p->stream_a = ly[0].K > kChainActAtoms * BK ? 1 : 0;
  {
    cuuint64_t dims[2] = {(cuuint64_t)ly[0].K, (cuuint64_t)a_rows};
    cuuint64_t str[1] = {(cuuint64_t)ly[0].lda * 4};
    cuuint32_t box[2] = {BK, BM};
    if (!encode(&p->map_a, ly[0].A, 2, dims, str, box)) return false;
  }
  for (int l = 0; l < nl; ++l) {
    const FcArgs& a = ly[l];
    p->n[l] = a.N;
    p->np[l] = (a.N + 15) / 16 * 16;
    p->k[l] = a.K;
    p->relu[l] = a.relu;
    p->bias[l] = a.bias;
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.N};
    cuuint64_t str[1] = {(cuuint64_t)a.ldw * 4};
    cuuint32_t box[2] = {BK, (cuuint32_t)p->np[l]};
    if (!encode(&p->map_w[l], a.W, 2, dims, str, box)) return false;
  }
  const FcArgs& out = ly[L - 1];
  p->C = out.C;
  p->ldc = out.ldc;
  p->c_desc = out.c_desc;
  if (narrow) {
    p->W2 = out.W; p->ldw2 = out.ldw; p->b2 = out.bias; p->N2 = out.N; p->relu2 = out.relu;
  }
  int wmax = 0;
  for (int l = 0; l < nl; ++l) wmax = std::max(wmax, p->np[l] * BK * 4);
  p->slot_b = p->stream_a ? BM * BK * 4 : 0;           // 1 KB multiples: SW128 atoms
  p->slot = p->slot_b + (wmax + 1023) / 1024 * 1024;
  p->stages = std::min(kChainMaxStages, kChainRingBytes / p->slot);
  if (p->stages < 2) return false;
  p->m_tiles = (int)((m_cap + BM - 1) / BM);
  smem_attr(reinterpret_cast<const void*>(fc_chain_kernel), (int)(sizeof(ChainSmem) + 1024));
  return true;
#endif  // RS_EXPERIMENTS
}

void launch_fc_chain(const QDesc* qd, const TcChainPlan& p, cudaStream_t s) {
#if RS_EXPERIMENTS
  launch_pdl(fc_chain_kernel, dim3(p.m_tiles), dim3(kChainThreads), sizeof(ChainSmem) + 1024, s,
             qd, p);
#else
  (void)qd; (void)p; (void)s;
#endif
}

void launch_fc_tc(const QDesc* qd, const TcPlan& p, const FcArgs& a0, cudaStream_t s) {
  FcArgs a = a0;
  a.splits = p.splits;
  a.ws = p.ws;
  a.cnt = p.cnt;
  const dim3 grid(p.n_tiles, p.m_tiles, a.batch * std::max(1, p.splits));
  const int a_batched = a.sAz != 0 ? 1 : 0;
#define RS_TC(BN, ST, H)                                                                    \
  launch_pdl(fc_tc_kernel<BN, ST, H>, grid, dim3(kTcThreads), tc_smem_bytes<BN, ST>(), s, qd, \
             p.map_a, p.map_w, a, a_batched)
  if (p.cfg == 5) {
    const dim3 grid2(p.m_tiles, p.n_tiles, a.batch);  // pairs along x
    // a CTA of the pair stages 32 KB per k-slab (16 KB of A + half of the
    // 256 weight rows), so the ring runs 6 deep in 192 KB (RS_TC2_STAGES=4:
    // 4), or 3 deep in the 96 KB of a carveout-capped graph
#define RS_TC2L(ST, H)                                                                   \
  launch_pair(fc_tc2_kernel<256, ST, H>, grid2, dim3(kTcThreads), tc2_smem_bytes<256, ST>(), \
              s, qd, p.map_a, p.map_w, a, a_batched)
#define RS_TC2S(H)                                  \
  switch (p.pair_stages) {                          \
    case 3: RS_TC2L(3, H); break;                   \
    case 4: RS_TC2L(4, H); break;                   \
    default: RS_TC2L(6, H); break;                  \
  }
    if (p.ab16) {
      RS_TC2S(true)
    } else {
      RS_TC2S(false)
    }
#undef RS_TC2S
#undef RS_TC2L
    return;
  }
  if (p.ab16) {
    switch (p.cfg) {
      case 0: RS_TC(128, 3, true); break;
      case 4: RS_TC(256, 4, true); break;
      case 1: RS_TC(64, 4, true); break;
      case 2: RS_TC(128, 6, true); break;
      default: RS_TC(64, 8, true); break;
    }
  } else {
    switch (p.cfg) {
      case 0: RS_TC(128, 3, false); break;
      case 4: RS_TC(256, 4, false); break;
      case 1: RS_TC(64, 4, false); break;
      case 2: RS_TC(128, 6, false); break;
      default: RS_TC(64, 8, false); break;
    }
  }
#undef RS_TC
}

}  // namespace rs
