// embedding.cu — the HBM-bound half of the offloaded forward pass.
//
//   sls_sum        SparseLengthsSum / embedding-bag Sum pooling
//                  (EmbeddingLookup + Pooling::Sum, proj/src/model_zoo.cpp:192-201)
//   gather_concat  Pooling::Concat gather into the predict-FC input (:202-206)
//   din_pool       DIN local-activation attention pooling (AttentionFC, :207-216)
//   interaction    DLRM pairwise dots + summed embedding (Interaction, :231-238;
//                  feature layout of predict_input_dim, :113-137)
//   init_tables    seeded table fill
//
// Layout in HBM: all T tables of a model in ONE allocation, [T][rows][D]
// fp32 row-major, so a row is one contiguous D*4-byte segment (128 B at the
// zoo's D=32, 256 B at cfg3's D=64). Indices arrive item-major [S][T][L]
// int64 exactly as the reference's byte model ships them
// (proj/src/platform.cpp:105-111), so bag (item, t) is L contiguous int64.
//
// SLS design (measured, tools/sls_micro.py): one warp per bag.
// The warp stages the bag's index list in shared memory, then reads rows with
// 128-bit non-allocating loads: LPR = D/4 lanes cover one row, R = 32/LPR rows
// land per warp instruction and U unrolled instructions keep R*U rows in
// flight per warp (16 rows = 4 KB at D=64; 32 warps/SM). The grid is
// oversubscribed 2x the resident CTAs so late CTAs pick up the bag tail
// dynamically. Lane group g accumulates rows g, g+R, g+2R, ... of the bag in
// order; groups combine by an xor-shuffle tree. That order is the canonical
// SLS order oracle/forward.c restates, so pooled sums are bit-identical to the
// oracle and run to run. Alternatives measured and rejected: 32-lookup chunk
// units (per-unit latency beats the balance gain), a device work queue
// (atomic + reset cost), deeper unrolling (fewer warps), and a TMA
// tile::gather4 landing zone (kept below as variant 1: bit-identical, but
// shared-memory capacity caps bytes in flight; 3.8 vs 5.2 TB/s at S=323).
#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.hpp"

namespace rs {

namespace {

constexpr int kWarps = 8;      // warps per CTA for warp-per-bag kernels
constexpr int kIdxChunk = 256; // staged indices per warp per pass

template <int LPR, int VPL, int U>
__global__ void __launch_bounds__(kWarps * 32)
sls_sum_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables, int64_t rows,
               int T, int L, float* __restrict__ out, int64_t ld_out, int* __restrict__ err,
               int hint) {
  // No early PDL trigger in the embedding-stage kernels: a dependent grid
  // launched early would squat on the SM slots this grid's tail frees, which
  // the next query's gather (another lane) should get. Dependents launch at
  // completion.
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  __shared__ int64_t sidx[kWarps][kIdxChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  const uint64_t pol = l2_evict_first_policy();
  for (int64_t bag = (int64_t)blockIdx.x * kWarps + warp; bag < bags;
       bag += (int64_t)gridDim.x * kWarps) {
    const int t = (int)(bag % T);
    const float4* __restrict__ tab =
        reinterpret_cast<const float4*>(tables + (int64_t)t * rows * D);
    const int64_t* __restrict__ bidx = idx + bag * L;
    float4 acc[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < L; c0 += kIdxChunk) {
      const int n = min(kIdxChunk, L - c0);
      __syncwarp();
      for (int l = lane; l < n; l += 32) sidx[warp][l] = __ldg(bidx + c0 + l);
      __syncwarp();
      for (int j = 0; j < n; j += R * U) {
        float4 v[U][VPL];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int l = j + u * R + g;
          ok[u] = false;
          if (l < n) {
            const int64_t r = sidx[warp][l];
            if ((uint64_t)r < (uint64_t)rows) {
              ok[u] = true;
              const float4* p = tab + r * (D / 4) + c;
#pragma unroll
              for (int k = 0; k < VPL; ++k)
                v[u][k] = hint ? ldg_stream_hint(p + k * LPR, pol) : ldg_stream(p + k * LPR);
            } else {
              atomicOr(err, kErrIndex);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u]) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) add4(acc[k], v[u][k]);
          }
      }
    }
#pragma unroll
    for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
      for (int k = 0; k < VPL; ++k) add4(acc[k], shfl_xor4(acc[k], off));
    if (g == 0) {
      float4* o = reinterpret_cast<float4*>(out + (bag / T) * ld_out + (int64_t)t * D) + c;
#pragma unroll
      for (int k = 0; k < VPL; ++k) o[k * LPR] = acc[k];
    }
  }
}

#if RS_EXPERIMENTS  // measured-slower SLS variant 1
// Variant 1 (RS_SLS_VARIANT=1): TMA tile::gather4. One warp per CTA; the warp walks its bags
// in sub-chunks of up to LB rows. For each sub-chunk, lane i loads lookups
// 4i..4i+3, turns them into rows of the stacked [T*rows, D] tensor and issues
// ONE cp.async.bulk.tensor.2d...tile::gather4 that lands those 4 rows in
// shared memory and completes bytes on the buffer's mbarrier. NBUF buffers
// keep NBUF-1 sub-chunks in flight while the warp sums the current one from
// shared memory in the R-interleaved order of the bag variant (so results are
// bit-identical to it and to the oracle). No register cost for in-flight
// data: memory-level parallelism is set by shared memory, not by unrolling.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int LPR, int VPL, int NBUF>
__global__ void __launch_bounds__(32)
sls_tma_kernel(const QDesc* __restrict__ qd, const __grid_constant__ CUtensorMap tmap,
               int64_t rows, int T, int L, int LB, float* __restrict__ out, int64_t ld_out,
               int* __restrict__ err) {
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  extern __shared__ __align__(128) uint8_t sm_raw[];
  float* buf = reinterpret_cast<float*>(sm_raw);                           // [NBUF][LB][D]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm_raw + NBUF * LB * D * 4);  // [NBUF]
  uint32_t* okmask = reinterpret_cast<uint32_t*>(bar + NBUF);              // [NBUF][MW]
  const int MW = (LB + 31) / 32;                                           // LB <= 128
  const int lane = threadIdx.x;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t S = qd->S;
  const int64_t* __restrict__ idx = qd->idx;
  const int64_t bags = S * T;
  const int nsub = (L + LB - 1) / LB;
  // this warp's stream of sub-chunks: bags blockIdx.x, +gridDim.x, ...; nsub each
  const int64_t my_bags = bags > blockIdx.x ? (bags - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t nk = my_bags * nsub;
  if (nk == 0) return;
  if (lane == 0) {
    for (int b = 0; b < NBUF; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar + b)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](int64_t k) {
    const int b = (int)(k % NBUF);
    const int64_t bag = (int64_t)blockIdx.x + (k / nsub) * gridDim.x;
    const int l0 = (int)(k % nsub) * LB;
    const int n = min(LB, L - l0);
    const int ng = (n + 3) / 4;              // gather4 instructions
    const int t = (int)(bag % T);
    int crd[4] = {0, 0, 0, 0};
    uint32_t okbits = 0;
    if (lane < ng) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int l = 4 * lane + j;
        if (l < n) {
          const int64_t r = __ldg(idx + bag * L + l0 + l);
          if ((uint64_t)r < (uint64_t)rows) {
            crd[j] = (int)(t * rows + r);
            okbits |= 1u << j;
          } else {
            atomicOr(err, kErrIndex);
          }
        }
      }
    }
    // row-validity bits of this sub-chunk: lane i owns rows 4i..4i+3
    uint32_t* mk = okmask + b * MW;
    for (int w = 0; w < MW; ++w) {
      // rows 32w..32w+31 live in lanes 8w..8w+7
      uint32_t word = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) word |= __shfl_sync(0xffffffffu, okbits, (8 * w + q) & 31) << (4 * q);
      if (lane == 0) mk[w] = word;
    }
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)ng * 4u * D * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar + b)),
                   "r"(bytes)
                   : "memory");
    }
    __syncwarp();
    if (lane < ng) {
      float* dst = buf + ((size_t)b * LB + 4 * lane) * D;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_addr(dst)),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(smem_addr(bar + b)), "r"(0), "r"(crd[0]),
          "r"(crd[1]), "r"(crd[2]), "r"(crd[3])
          : "memory");
    }
  };

  for (int64_t k = 0; k < NBUF - 1 && k < nk; ++k) issue(k);
  float4 acc[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t k = 0; k < nk; ++k) {
    if (k + NBUF - 1 < nk) issue(k + NBUF - 1);
    const int b = (int)(k % NBUF);
    const uint32_t parity = (uint32_t)((k / NBUF) & 1);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_addr(bar + b)),
        "r"(parity)
        : "memory");
    const int l0 = (int)(k % nsub) * LB;
    const int n = min(LB, L - l0);
    const float4* src = reinterpret_cast<const float4*>(buf + (size_t)b * LB * D);
    const uint32_t* mk = okmask + b * MW;
    for (int j = g; j < n; j += R) {
      if ((mk[j >> 5] >> (j & 31)) & 1u) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) add4(acc[q], src[j * (D / 4) + c + q * LPR]);
      }
    }
    __syncwarp();  // every lane is done with buffer b before it is refilled
    if (k % nsub == nsub - 1) {
      const int64_t bag = (int64_t)blockIdx.x + (k / nsub) * gridDim.x;
      const int t = (int)(bag % T);
#pragma unroll
      for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
        for (int q = 0; q < VPL; ++q) add4(acc[q], shfl_xor4(acc[q], off));
      if (g == 0) {
        float4* o = reinterpret_cast<float4*>(out + (bag / T) * ld_out + (int64_t)t * D) + c;
#pragma unroll
        for (int q = 0; q < VPL; ++q) o[q * LPR] = acc[q];
      }
#pragma unroll
      for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

#endif  // RS_EXPERIMENTS

// Variant 2 (RS_SLS_VARIANT=2): warp-per-bag with the two serial latencies of
// a bag hidden — the NEXT bag's index list is loaded into registers while this
// bag's rows stream, and row batch j+1 is in flight while batch j accumulates.
// Same per-lane accumulation order as sls_sum_kernel (bit-identical results).
// Bags of up to 32*IPL lookups; longer bags use sls_sum_kernel.
// DYN: bags handed out by a ticket counter in the query descriptor instead of
// a static stride — a warp that finishes early takes the next bag, so a launch
// ends when the LAST BAG ends, not when the warp with the most bags does
// (static striding gives 1.49 bags per warp at 330 items x 32 tables over the
// 7104-warp grid: half the warps idle for a whole bag at the end). The order
// inside a bag is untouched (bit-identical).
template <int LPR, int VPL, int U, int IPL, bool HOT, bool EF = false, bool DYN = false>
__global__ void __launch_bounds__(kWarps * 32)
sls_pipe_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables, int64_t rows,
                int T, int L, float* __restrict__ out, int64_t ld_out, int* __restrict__ err,
                const float* __restrict__ hot, int64_t hot_rows) {
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  constexpr int B = R * U;  // rows per batch
  __shared__ int64_t sidx[kWarps][32 * IPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  const int nw = blockDim.x >> 5;  // warps per CTA (<= kWarps; RS_SLS_WPC)
  const int64_t stride = (int64_t)gridDim.x * nw;
  // EF: table rows marked evict-first in L2, so the once-touched gather stream
  // does not push the dense stages' reused data (weights, X, pooled) out
  const uint64_t pol = EF ? l2_evict_first_policy() : 0;
  int64_t nidx[IPL];
  auto fetch_idx = [&](int64_t bag) {
#pragma unroll
    for (int q = 0; q < IPL; ++q) {
      const int l = q * 32 + lane;
      nidx[q] = (bag < bags && l < L) ? __ldg(idx + bag * L + l) : 0;
    }
  };
  unsigned int* work = const_cast<unsigned int*>(qd->work);
  auto ticket = [&]() -> int64_t {
    unsigned int v = 0;
    if (lane == 0) v = atomicAdd(work, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  int64_t bag = DYN ? ticket() : (int64_t)blockIdx.x * nw + warp;
  fetch_idx(bag);
  for (int64_t next; bag < bags; bag = next) {
    __syncwarp();
#pragma unroll
    for (int q = 0; q < IPL; ++q) sidx[warp][q * 32 + lane] = nidx[q];
    __syncwarp();
    next = DYN ? ticket() : bag + stride;
    fetch_idx(next);  // next bag's indices fly with this bag's rows
    const int t = (int)(bag % T);
    const float4* __restrict__ tab =
        reinterpret_cast<const float4*>(tables + (int64_t)t * rows * D);
    // HOT: rows [0, hot_rows) of every table also live in the L2-persisting
    // hot block [T][hot_rows][D] (an exact copy); a separate instantiation so
    // the default kernel carries no extra work
    const float4* __restrict__ htab =
        HOT ? reinterpret_cast<const float4*>(hot + (int64_t)t * hot_rows * D) : nullptr;
    auto load_batch = [&](int j, float4 (&v)[U][VPL], bool (&ok)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = j + u * R + g;
        ok[u] = false;
        if (l < L) {
          const int64_t r = sidx[warp][l];
          if ((uint64_t)r < (uint64_t)rows) {
            ok[u] = true;
            const float4* p = (HOT && r < hot_rows ? htab : tab) + r * (D / 4) + c;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
              v[u][k] = EF ? ldg_stream_hint(p + k * LPR, pol) : ldg_stream(p + k * LPR);
          } else {
            atomicOr(err, kErrIndex);
          }
        }
      }
    };
    float4 acc[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto consume = [&](const float4 (&v)[U][VPL], const bool (&ok)[U]) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) {
#pragma unroll
          for (int k = 0; k < VPL; ++k) add4(acc[k], v[u][k]);
        }
    };
    float4 va[U][VPL], vb[U][VPL];
    bool oa[U], ob[U];
    load_batch(0, va, oa);
    for (int j = 0; j < L; j += 2 * B) {
      if (j + B < L) load_batch(j + B, vb, ob);
      consume(va, oa);
      if (j + B < L) {
        if (j + 2 * B < L) load_batch(j + 2 * B, va, oa);
        consume(vb, ob);
      }
    }
#pragma unroll
    for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
      for (int k = 0; k < VPL; ++k) add4(acc[k], shfl_xor4(acc[k], off));
    if (g == 0) {
      float4* o = reinterpret_cast<float4*>(out + (bag / T) * ld_out + (int64_t)t * D) + c;
#pragma unroll
      for (int k = 0; k < VPL; ++k) o[k * LPR] = acc[k];
    }
  }
  if (DYN && lane == 0) {
    // the last warp to retire leaves the counters at zero for the next launch
    // of this slot's graph (descriptor rewrites zero them too)
    const unsigned int total = gridDim.x * (unsigned int)nw;
    if (atomicAdd(work + 1, 1u) == total - 1) {
      atomicExch(work, 0u);
      atomicExch(work + 1, 0u);
    }
  }
}

#if RS_EXPERIMENTS  // measured-slower SLS variants 4 and 3
// Variant 4 (RS_SLS_VARIANT=4): variant 2 without the bubble between bags.
// A warp's bags are one continuous stream of row batches: batch t+1 is issued
// before batch t is summed even when t+1 is the first batch of the warp's
// next bag, so the rows in flight per warp never drop to zero at a bag
// boundary (variant 2 pays one dependent round trip per bag there, and at
// the end of a launch every warp's last bags are exactly that chain).
// Index lists are double-buffered in shared memory; bag k's list is staged
// when its first batch is issued, from registers fetched one bag earlier.
// Same per-lane accumulation order as sls_sum_kernel: bit-identical.
template <int LPR, int VPL, int U, int IPL>
__global__ void __launch_bounds__(kWarps * 32)
sls_stream_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables, int64_t rows,
                  int T, int L, float* __restrict__ out, int64_t ld_out, int* __restrict__ err) {
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  constexpr int B = R * U;  // rows per batch
  __shared__ int64_t sidx[kWarps][2][32 * IPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  const int64_t stride = (int64_t)gridDim.x * kWarps;
  const int64_t bag0 = (int64_t)blockIdx.x * kWarps + warp;
  if (bag0 >= bags) return;
  const int64_t nbags = (bags - bag0 + stride - 1) / stride;
  const int nb = (L + B - 1) / B;  // batches per bag
  const int64_t total = nbags * nb;
  int64_t nidx[IPL];
  auto fetch_idx = [&](int64_t bag) {
#pragma unroll
    for (int q = 0; q < IPL; ++q) {
      const int l = q * 32 + lane;
      nidx[q] = (bag < bags && l < L) ? __ldg(idx + bag * L + l) : 0;
    }
  };
  fetch_idx(bag0);
  // issue batch t into v (t = k*nb + jb: rows jb*B.. of the warp's k-th bag)
  auto load = [&](int64_t t, float4 (&v)[U][VPL], bool (&ok)[U]) {
    const int64_t k = t / nb;
    const int jb = (int)(t - k * nb);
    const int64_t bag = bag0 + k * stride;
    int64_t* si = sidx[warp][k & 1];
    if (jb == 0) {
      __syncwarp();
#pragma unroll
      for (int q = 0; q < IPL; ++q) si[q * 32 + lane] = nidx[q];
      __syncwarp();
      fetch_idx(bag + stride);  // flies while this bag's rows stream
    }
    const int t_ = (int)(bag % T);
    const float4* __restrict__ tab =
        reinterpret_cast<const float4*>(tables + (int64_t)t_ * rows * D);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int l = jb * B + u * R + g;
      ok[u] = false;
      if (l < L) {
        const int64_t r = si[l];
        if ((uint64_t)r < (uint64_t)rows) {
          ok[u] = true;
          const float4* p = tab + r * (D / 4) + c;
#pragma unroll
          for (int q = 0; q < VPL; ++q) v[u][q] = ldg_stream(p + q * LPR);
        } else {
          atomicOr(err, kErrIndex);
        }
      }
    }
  };
  float4 acc[VPL];
  // sum batch t; at a bag's last batch reduce across lane groups and store
  auto consume = [&](int64_t t, const float4 (&v)[U][VPL], const bool (&ok)[U]) {
    const int64_t k = t / nb;
    const int jb = (int)(t - k * nb);
    if (jb == 0) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) add4(acc[q], v[u][q]);
      }
    if (jb == nb - 1) {
      float4 r[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) r[q] = acc[q];
#pragma unroll
      for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
        for (int q = 0; q < VPL; ++q) add4(r[q], shfl_xor4(r[q], off));
      if (g == 0) {
        const int64_t bag = bag0 + k * stride;
        const int t_ = (int)(bag % T);
        float4* o = reinterpret_cast<float4*>(out + (bag / T) * ld_out + (int64_t)t_ * D) + c;
#pragma unroll
        for (int q = 0; q < VPL; ++q) o[q * LPR] = r[q];
      }
    }
  };
  float4 va[U][VPL], vb[U][VPL];
  bool oa[U], ob[U];
  load(0, va, oa);
  for (int64_t t = 0; t < total; t += 2) {
    if (t + 1 < total) load(t + 1, vb, ob);
    consume(t, va, oa);
    if (t + 1 < total) {
      if (t + 2 < total) load(t + 2, va, oa);
      consume(t + 1, vb, ob);
    }
  }
}

// Variant 3 (RS_SLS_VARIANT=3): warp-per-bag with whole bags staged in shared
// memory by cp.async. A warp issues 16-byte cp.async copies for EVERY row of
// its next bag (nbuf-1 bags ahead) before it sums the current one, so a bag's
// rows are all in flight at once and memory-level parallelism costs shared
// memory instead of registers. That shortens the kernel's ramp and tail: the
// last bags of a launch complete in about one memory latency instead of
// L/(rows in flight) latencies. Rows with an out-of-range index are zero-filled
// (acc + 0.0f is exact: the accumulator starts at +0 and can never become -0),
// and are flagged in the error word. Summation order per lane is the one of
// sls_sum_kernel (rows g, g+R, g+2R, ...; then the xor tree): bit-identical.
template <int LPR, int VPL, int IPL>
__global__ void __launch_bounds__(512)
sls_stage_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables, int64_t rows,
                 int T, int L, int nbuf, float* __restrict__ out, int64_t ld_out,
                 int* __restrict__ err) {
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  constexpr int C4 = D / 4;  // 16-byte chunks per row
  extern __shared__ __align__(16) float4 sbuf[];  // [warps][nbuf][L][C4]
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  const int64_t stride = (int64_t)gridDim.x * nw;
  const int64_t first = (int64_t)blockIdx.x * nw + warp;
  float4* wbuf = sbuf + (size_t)warp * nbuf * L * C4;
  int64_t nidx[IPL];
  auto fetch_idx = [&](int64_t bag) {
#pragma unroll
    for (int q = 0; q < IPL; ++q) {
      const int l = q * 32 + lane;
      nidx[q] = (bag < bags && l < L) ? __ldg(idx + bag * L + l) : 0;
    }
  };
  // copy bag `bag`'s rows into stage st (indices in nidx)
  auto issue = [&](int64_t bag, int st) {
    const int t = (int)(bag % T);
    const float4* __restrict__ tab = reinterpret_cast<const float4*>(tables + (int64_t)t * rows * D);
    float4* dst = wbuf + (size_t)st * L * C4;
    bool bad = false;
#pragma unroll
    for (int q = 0; q < IPL; ++q) {
#pragma unroll
      for (int i = 0; i < 32 / R; ++i) {
        const int src = i * R + g;
        const int64_t r = __shfl_sync(0xffffffffu, nidx[q], src);
        const int l = q * 32 + src;
        if (l < L) {
          float4* d = dst + (size_t)l * C4 + c;
          if ((uint64_t)r < (uint64_t)rows) {
            const float4* p = tab + r * C4 + c;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(d + k * LPR)),
                           "l"(p + k * LPR)
                           : "memory");
          } else {
#pragma unroll
            for (int k = 0; k < VPL; ++k) d[k * LPR] = make_float4(0.f, 0.f, 0.f, 0.f);
            bad = true;
          }
        }
      }
    }
    if (bad) atomicOr(err, kErrIndex);
  };
  int64_t bag = first;
  fetch_idx(bag);
  for (int s = 0; s < nbuf - 1; ++s) {
    const int64_t b = first + s * stride;
    if (b < bags) {
      issue(b, s);
      fetch_idx(b + stride);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t k = 0; bag < bags; ++k, bag += stride) {
    const int64_t ahead = bag + (int64_t)(nbuf - 1) * stride;
    if (ahead < bags) {
      issue(ahead, (int)((k + nbuf - 1) % nbuf));
      fetch_idx(ahead + stride);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // groups complete in order: all but the newest nbuf-1 are done -> bag k landed
    switch (nbuf) {
      case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
      case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
      default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    }
    __syncwarp();
    const float4* src = wbuf + (size_t)(k % nbuf) * L * C4;
    float4 acc[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int l = g; l < L; l += R) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) add4(acc[q], src[(size_t)l * C4 + c + q * LPR]);
    }
#pragma unroll
    for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
      for (int q = 0; q < VPL; ++q) add4(acc[q], shfl_xor4(acc[q], off));
    if (g == 0) {
      const int t = (int)(bag % T);
      float4* o = reinterpret_cast<float4*>(out + (bag / T) * ld_out + (int64_t)t * D) + c;
#pragma unroll
      for (int q = 0; q < VPL; ++q) o[q * LPR] = acc[q];
    }
    __syncwarp();  // stage k % nbuf is refilled by the next iteration's issue
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

#endif  // RS_EXPERIMENTS

// Any D (not a power of two in [8,256]): lane-per-column, sequential in l.
__global__ void __launch_bounds__(kWarps * 32)
sls_sum_scalar_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables,
                      int64_t rows, int T, int L, int D, float* __restrict__ out,
                      int64_t ld_out, int* __restrict__ err) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  for (int64_t bag = (int64_t)blockIdx.x * kWarps + warp; bag < bags;
       bag += (int64_t)gridDim.x * kWarps) {
    const int t = (int)(bag % T);
    const float* tab = tables + (int64_t)t * rows * D;
    for (int c = lane; c < D; c += 32) {
      float acc = 0.f;
      for (int l = 0; l < L; ++l) {
        const int64_t r = __ldg(idx + bag * L + l);
        if ((uint64_t)r < (uint64_t)rows) acc += ldg_stream1(tab + r * D + c);
        else if (c == lane) atomicOr(err, kErrIndex);
      }
      out[(bag / T) * ld_out + (int64_t)t * D + c] = acc;
    }
  }
}

// Concat gather: out[item, col_off + (t*L + l)*D + c] = E_t[idx[item,t,l], c].
__global__ void __launch_bounds__(256)
gather_concat_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables,
                     int64_t rows, int T, int L, int D, float* __restrict__ out,
                     int64_t ld_out, int64_t col_off, int vec, int* __restrict__ err) {
  const int64_t S = qd->S;
  const int64_t* __restrict__ idx = qd->idx;
  const int64_t TL = (int64_t)T * L;
  const int W = vec ? D / 4 : D;  // work units per row
  const int64_t total = S * TL * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowi = i / W;      // flat (item, t, l)
    const int w = (int)(i - rowi * W);
    const int64_t item = rowi / TL;
    const int64_t tl = rowi - item * TL;
    const int t = (int)(tl / L);
    const int64_t r = __ldg(idx + rowi);
    float* dst = out + item * ld_out + col_off + tl * D;
    if ((uint64_t)r >= (uint64_t)rows) {
      if (w == 0) atomicOr(err, kErrIndex);
      continue;
    }
    const float* src = tables + ((int64_t)t * rows + r) * D;
    if (vec) {
      reinterpret_cast<float4*>(dst)[w] = ldg_stream(reinterpret_cast<const float4*>(src) + w);
    } else {
      dst[w] = ldg_stream1(src + w);
    }
  }
}

// DIN attention pooling, one warp per (item, table) bag:
//   q = e_0 (the bag's first lookup is the candidate), weight
//   a_l = sigmoid(q^T W_t e_l), pooled = sum_l a_l e_l (unnormalised, as DIN).
// Computed as u = W_t^T q once per bag, then a_l = sigmoid(<u, e_l>): the same
// bilinear form with 2D flops per lookup instead of 2D^2, which turns the
// reference's FFMA-bound Attention category (model_zoo.cpp:207-216) into a
// pure gather at HBM speed.
template <int LPR, int VPL, int U>
__global__ void __launch_bounds__(kWarps * 32, 4)
din_pool_kernel(const QDesc* __restrict__ qd, const float* __restrict__ tables, int64_t rows,
                int T, int L, const float* __restrict__ att_w, float* __restrict__ out,
                int64_t ld_out, int64_t col_off, int* __restrict__ err) {
  constexpr int R = 32 / LPR;
  constexpr int D = LPR * 4 * VPL;
  __shared__ int64_t sidx[kWarps][kIdxChunk];
  __shared__ float sq[kWarps][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / LPR, c = lane % LPR;
  const int64_t bags = qd->S * T;
  const int64_t* __restrict__ idx = qd->idx;
  for (int64_t bag = (int64_t)blockIdx.x * kWarps + warp; bag < bags;
       bag += (int64_t)gridDim.x * kWarps) {
    const int t = (int)(bag % T);
    const float4* __restrict__ tab =
        reinterpret_cast<const float4*>(tables + (int64_t)t * rows * D);
    const int64_t* __restrict__ bidx = idx + bag * L;
    // candidate q = row of lookup 0
    const int64_t r0 = __ldg(bidx);
    const bool q_ok = (uint64_t)r0 < (uint64_t)rows;
    if (!q_ok && lane == 0) atomicOr(err, kErrIndex);
    __syncwarp();
    for (int i = lane; i < D; i += 32)
      sq[warp][i] = q_ok ? __ldg(reinterpret_cast<const float*>(tab + r0 * (D / 4)) + i) : 0.f;
    __syncwarp();
    // u = W_t^T q for this lane's columns (W_t row-major [D][D], L2-resident)
    float4 u[VPL];
    const float* W = att_w + (int64_t)t * D * D;
#pragma unroll
    for (int k = 0; k < VPL; ++k) u[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < D; ++i) {
      const float qi = sq[warp][i];
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(W + (int64_t)i * D) + c + k * LPR);
        u[k].x = fmaf(qi, w.x, u[k].x);
        u[k].y = fmaf(qi, w.y, u[k].y);
        u[k].z = fmaf(qi, w.z, u[k].z);
        u[k].w = fmaf(qi, w.w, u[k].w);
      }
    }
    float4 acc[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < L; c0 += kIdxChunk) {
      const int n = min(kIdxChunk, L - c0);
      __syncwarp();
      for (int l = lane; l < n; l += 32) sidx[warp][l] = __ldg(bidx + c0 + l);
      __syncwarp();
      // Software-pipelined: batch j+1's row loads are in flight while batch j
      // is scored and accumulated (the score -> shuffle -> sigmoid chain per
      // row would otherwise leave the memory system idle).
      auto load_batch = [&](int j, float4 (&v)[U][VPL], bool (&ok)[U]) {
#pragma unroll
        for (int u2 = 0; u2 < U; ++u2) {
          const int l = j + u2 * R + g;
          ok[u2] = false;
#pragma unroll
          for (int k = 0; k < VPL; ++k) v[u2][k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (l < n) {
            const int64_t r = sidx[warp][l];
            if ((uint64_t)r < (uint64_t)rows) {
              ok[u2] = true;
              const float4* p = tab + r * (D / 4) + c;
#pragma unroll
              for (int k = 0; k < VPL; ++k) v[u2][k] = ldg_stream(p + k * LPR);
            } else {
              atomicOr(err, kErrIndex);
            }
          }
        }
      };
      auto consume = [&](const float4 (&v)[U][VPL], const bool (&ok)[U]) {
#pragma unroll
        for (int u2 = 0; u2 < U; ++u2) {
          float s = 0.f;
#pragma unroll
          for (int k = 0; k < VPL; ++k) {
            s = fmaf(u[k].x, v[u2][k].x, s);
            s = fmaf(u[k].y, v[u2][k].y, s);
            s = fmaf(u[k].z, v[u2][k].z, s);
            s = fmaf(u[k].w, v[u2][k].w, s);
          }
#pragma unroll
          for (int off = LPR / 2; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          s = __fdividef(1.0f, 1.0f + __expf(-s));  // activation-unit weight (SFU)
          if (ok[u2]) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
              acc[k].x = fmaf(s, v[u2][k].x, acc[k].x);
              acc[k].y = fmaf(s, v[u2][k].y, acc[k].y);
              acc[k].z = fmaf(s, v[u2][k].z, acc[k].z);
              acc[k].w = fmaf(s, v[u2][k].w, acc[k].w);
            }
          }
        }
      };
      constexpr int B = R * U;  // rows per batch
      float4 va[U][VPL], vb[U][VPL];
      bool oa[U], ob[U];
      load_batch(0, va, oa);
      for (int j = 0; j < n; j += 2 * B) {
        if (j + B < n) load_batch(j + B, vb, ob);
        consume(va, oa);
        if (j + B < n) {
          if (j + 2 * B < n) load_batch(j + 2 * B, va, oa);
          consume(vb, ob);
        }
      }
    }
#pragma unroll
    for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
      for (int k = 0; k < VPL; ++k) add4(acc[k], shfl_xor4(acc[k], off));
    if (g == 0) {
      float* o = out + (bag / T) * ld_out + col_off + (int64_t)t * D;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int cc = (c + k * LPR) * 4;
        o[cc + 0] = acc[k].x; o[cc + 1] = acc[k].y; o[cc + 2] = acc[k].z; o[cc + 3] = acc[k].w;
      }
    }
  }
}

// DLRM interaction, one CTA per item (grid-stride):
//   X[item, sum_off + c]  = sum_{t=1..T} v_t[c]              (sequential in t)
//   X[item, dot_off + p]  = <v_i, v_j>, i = 1..T, j = 0..i-1  (p = i(i-1)/2 + j)
// with v_0 = X[item, 0:D] (bottom-MLP output already written there) and
// v_t = pooled[item, t-1, :]. Pairs exist only when has_dense (the
// reference counts them only for Sum pooling with a dense stack).
constexpr int kInterRegs = 8;  // float4 loads in flight per thread per round

// kInterThreads = 256, or 64 for strongly gather-bound models (the handle's
// choice; RS_INTER_THREADS overrides): a 2-warp CTA capped at 64 registers
// per thread fits in the 4K registers three gather CTAs leave free on an SM,
// so the interaction co-runs with the gathers instead of taking SM slots they
// would refill (cfg3 RMC2 35.4 -> 34.1 us/query, zoo RMC2 -3.9%; cfg3 RMC3,
// whose FC work is 60% of its gather time, +4..9%: profiles/r2_inter64.txt).
template <int kInterThreads>
__global__ void __launch_bounds__(kInterThreads, 65536 / (kInterThreads * 64))
interaction_kernel(const QDesc* __restrict__ qd, const float* __restrict__ pooled,
                   int64_t ld_pooled, int T, int D, float* __restrict__ X, int64_t ld_x,
                   int64_t sum_off, int64_t dot_off, int has_dense, int discard) {
  pdl_wait();  // pooled (SLS) and X[:, 0:D] (bottom MLP) are predecessors' outputs
  extern __shared__ float sv[];  // [(T+1)][D+1]
  const int P = has_dense ? (T + 1) * T / 2 : 0;
  const int ldv = D + 1;
  const bool vec = (D & 3) == 0;
  const int D4 = D / 4;
  const int units = (T + 1) * D4;       // float4 units: v0 then pooled rows
  for (int64_t item = blockIdx.x; item < qd->S; item += gridDim.x) {
    __syncthreads();
    if (!vec) {
      for (int i = threadIdx.x; i < (T + 1) * D; i += blockDim.x) {
        const int v = i / D, c = i - v * D;
        sv[v * ldv + c] = v == 0 ? (has_dense ? X[item * ld_x + c] : 0.f)
                                 : pooled[item * ld_pooled + (int64_t)(v - 1) * D + c];
      }
    }
    // All of a round's 128-bit loads are issued before any shared store, so a
    // CTA pays one memory latency per round instead of one per element.
    for (int base = 0; vec && base < units; base += kInterRegs * kInterThreads) {
      float4 r[kInterRegs];
#pragma unroll
      for (int k = 0; k < kInterRegs; ++k) {
        const int u = base + k * kInterThreads + threadIdx.x;
        r[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (u < units) {
          const int v = u / D4, c4 = u - v * D4;
          if (v == 0) {
            if (has_dense) r[k] = *reinterpret_cast<const float4*>(X + item * ld_x + c4 * 4);
          } else {
            r[k] = __ldg(reinterpret_cast<const float4*>(pooled + item * ld_pooled +
                                                         (int64_t)(v - 1) * D) + c4);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kInterRegs; ++k) {
        const int u = base + k * kInterThreads + threadIdx.x;
        if (u < units) {
          const int v = u / D4, c = (u - v * D4) * 4;
          float* d = sv + v * ldv + c;
          d[0] = r[k].x; d[1] = r[k].y; d[2] = r[k].z; d[3] = r[k].w;
        }
      }
    }
    __syncthreads();
    if (discard) {
      // the item's pooled sums are dead once staged: drop their L2 lines
      // without a DRAM write-back (discard.global.L2, 128-byte lines)
      const char* row = reinterpret_cast<const char*>(pooled + item * ld_pooled);
      const int lines = (int)((int64_t)T * D * 4 / 128);
      for (int i = threadIdx.x; i < lines; i += blockDim.x)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + 128 * i) : "memory");
    }
    pdl_trigger();  // the predict layer's grid may launch while the dots run
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      float s = 0.f;
      for (int t = 1; t <= T; ++t) s += sv[t * ldv + c];
      X[item * ld_x + sum_off + c] = s;
    }
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      int i = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
      while (i * (i - 1) / 2 > p) --i;
      while ((i + 1) * i / 2 <= p) ++i;
      const int j = p - i * (i - 1) / 2;
      float d = 0.f;
      for (int c = 0; c < D; ++c) d = fmaf(sv[i * ldv + c], sv[j * ldv + c], d);
      X[item * ld_x + dot_off + p] = d;
    }
  }
}

// Warp-per-item interaction (the default when 8 items' operands fit in shared
// memory): 8 warps = 8 items per CTA, so a 300-item query is ~40 CTAs instead
// of 300 — inside the pipelined queue every CTA slot these take is a slot
// the concurrent gathers lose. Same per-output summation order as
// interaction_kernel: sum over t = 1..T in order; each dot sequential in c.
constexpr int kInterWarps = 8;

__global__ void __launch_bounds__(kInterWarps * 32)
interaction_warp_kernel(const QDesc* __restrict__ qd, const float* __restrict__ pooled,
                        int64_t ld_pooled, int T, int D, float* __restrict__ X, int64_t ld_x,
                        int64_t sum_off, int64_t dot_off, int has_dense) {
  pdl_wait();  // pooled (SLS) and X[:, 0:D] (bottom MLP) are predecessors' outputs
  extern __shared__ float smem_int[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ldv = D + 1;
  float* sv = smem_int + (size_t)warp * (T + 1) * ldv;  // [(T+1)][D+1]
  const int P = has_dense ? (T + 1) * T / 2 : 0;
  const int D4 = D / 4;
  const int units = (T + 1) * D4;
  const int64_t S = qd->S;
  for (int64_t item = (int64_t)blockIdx.x * kInterWarps + warp; item < S;
       item += (int64_t)gridDim.x * kInterWarps) {
    __syncwarp();
    // all of the item's 128-bit loads in flight before any shared store
    constexpr int kPer = 9;  // float4 per lane per round (T+1 <= 33, D <= 64: two rounds)
    for (int base = 0; base < units; base += kPer * 32) {
      float4 r[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int u = base + k * 32 + lane;
        r[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (u < units) {
          const int v = u / D4, c4 = u - v * D4;
          if (v == 0) {
            if (has_dense) r[k] = *reinterpret_cast<const float4*>(X + item * ld_x + c4 * 4);
          } else {
            r[k] = __ldg(reinterpret_cast<const float4*>(pooled + item * ld_pooled +
                                                         (int64_t)(v - 1) * D) + c4);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int u = base + k * 32 + lane;
        if (u < units) {
          const int v = u / D4, c = (u - v * D4) * 4;
          float* d = sv + v * ldv + c;
          d[0] = r[k].x; d[1] = r[k].y; d[2] = r[k].z; d[3] = r[k].w;
        }
      }
    }
    __syncwarp();
    if (warp == 0 && item == (int64_t)blockIdx.x * kInterWarps) pdl_trigger();
    for (int c = lane; c < D; c += 32) {
      float sacc = 0.f;
      for (int t = 1; t <= T; ++t) sacc += sv[t * ldv + c];
      X[item * ld_x + sum_off + c] = sacc;
    }
    for (int p = lane; p < P; p += 32) {
      int i = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
      while (i * (i - 1) / 2 > p) --i;
      while ((i + 1) * i / 2 <= p) ++i;
      const int j = p - i * (i - 1) / 2;
      const float* vi = sv + i * ldv;
      const float* vj = sv + j * ldv;
      float d = 0.f;
#pragma unroll 8
      for (int c = 0; c < D; ++c) d = fmaf(vi[c], vj[c], d);
      X[item * ld_x + dot_off + p] = d;
    }
  }
}

__global__ void init_tables_kernel(float* __restrict__ tables, int64_t T, int64_t rows,
                                   int64_t D, uint64_t seed) {
  const int64_t per_table = rows * D;
  const int64_t total = T * per_table;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < total;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    const int64_t t = i / per_table;
    const int64_t e = i - t * per_table;
    const uint64_t key = stream_key(seed, id_table(t));
    if (i + 3 < total && (e + 3) < per_table) {
      float4 v;
      v.x = param(key, (uint64_t)e + 0, kTableScale);
      v.y = param(key, (uint64_t)e + 1, kTableScale);
      v.z = param(key, (uint64_t)e + 2, kTableScale);
      v.w = param(key, (uint64_t)e + 3, kTableScale);
      *reinterpret_cast<float4*>(tables + i) = v;
    } else {
      for (int64_t k = i; k < i + 4 && k < total; ++k) {
        const int64_t tk = k / per_table;
        tables[k] = param(stream_key(seed, id_table(tk)), (uint64_t)(k - tk * per_table),
                          kTableScale);
      }
    }
  }
}

bool pow2_dim(int64_t D) {
  return D == 8 || D == 16 || D == 32 || D == 64 || D == 128 || D == 256;
}

int grid_for(int64_t units, int per_block, int sm_count, int blocks_per_sm) {
  const int64_t need = (units + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count * blocks_per_sm));
}

}  // namespace

bool sls_vector_path(int64_t D) { return pow2_dim(D); }


// RS_SLS_VARIANT: 2 (default) pipelined warp-per-bag (RS_SLS_UB = rows-per-
// batch unroll, 4 or 8; bags up to 96 lookups, else variant 0), 0 warp-per-bag
// register gather, 1 TMA gather4. All three are bit-identical.
int sls_variant() {
  const char* v = getenv("RS_SLS_VARIANT");
  return v ? atoi(v) : 2;
}
int sls_ub() {
  const char* v = getenv("RS_SLS_UB");
  return v ? atoi(v) : 4;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// RS_SLS_DYN (experiments build): 1 = dynamic bag tickets in the SLS kernel
bool sls_dyn() { return RS_EXPERIMENTS && env_int("RS_SLS_DYN", 0) != 0; }

template <int LPR, int VPL, int U, int IPL>
void launch_sls_pipe(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                     float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                     cudaStream_t s, const float* hot, int64_t hot_rows) {
  const int wpc = std::min(kWarps, std::max(1, env_int("RS_SLS_WPC", kWarps)));
#if RS_EXPERIMENTS
  // RS_SLS_EF=1: gather rows evict-first in L2 (measured +1.3% us/query in the
  // pipelined queue, i.e. slower: tools/env_sweep.py)
  // RS_SLS_DYN=1: bags by ticket (measured slower: one launch 5.16 -> 3.89
  // TB/s at 330 items, pipelined 38.5 -> 40.5 us/query — the ticket atomic
  // sits in front of the next bag's index load)
  const bool ef = env_int("RS_SLS_EF", 0) != 0;
  auto kern = hot_rows > 0 ? sls_pipe_kernel<LPR, VPL, U, IPL, true>
                           : (ef ? sls_pipe_kernel<LPR, VPL, U, IPL, false, true>
                                 : sls_dyn() ? sls_pipe_kernel<LPR, VPL, U, IPL, false, false, true>
                                             : sls_pipe_kernel<LPR, VPL, U, IPL, false>);
#else
  auto kern = hot_rows > 0 ? sls_pipe_kernel<LPR, VPL, U, IPL, true>
                           : sls_pipe_kernel<LPR, VPL, U, IPL, false>;
#endif
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wpc * 32, 0);
  per_sm = std::max(per_sm, 1);
  // grid = waves x resident CTAs: 2 for a single query (the second wave picks
  // up the bag tail), 1 in the pipelined queue's lanes, where the next
  // query's kernels fill the tail instead (cfg3 RMC2 -1.6%, RMC1 -7%
  // us/query; isolated launch -1%); dynamic tickets balance by themselves
  const int waves = env_int("RS_SLS_WAVES", (sls_dyn() && hot_rows == 0) || capture_lane() == 1
                                                ? 1 : 2);
  const int grid = grid_for(max_items * T, wpc, sm_count, waves * per_sm);
  max_carveout(reinterpret_cast<const void*>(kern));
  kern<<<grid, wpc * 32, 0, s>>>(qd, tables, rows, T, L, out, ld_out, err, hot, hot_rows);
}

#if RS_EXPERIMENTS  // variant 4 launcher
template <int LPR, int VPL, int U, int IPL>
void launch_sls_stream(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                       float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                       cudaStream_t s) {
  static const int per_sm = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sls_stream_kernel<LPR, VPL, U, IPL>,
                                                  kWarps * 32, 0);
    return b > 0 ? b : 1;
  }();
  const int grid = grid_for(max_items * T, kWarps, sm_count, env_int("RS_SLS_WAVES", 2) * per_sm);
  max_carveout(reinterpret_cast<const void*>(sls_stream_kernel<LPR, VPL, U, IPL>));
  sls_stream_kernel<LPR, VPL, U, IPL><<<grid, kWarps * 32, 0, s>>>(qd, tables, rows, T, L, out,
                                                                   ld_out, err);
}

template <int LPR, int VPL>
bool try_sls_stream(const QDesc* qd, const float* tables, int64_t rows, int T, int L, float* out,
                    int64_t ld_out, int* err, int64_t max_items, int sm_count, cudaStream_t s) {
  if (L > 96) return false;
  const int ub = sls_ub();
#define RS_STREAM(U, IPL)                                                                \
  launch_sls_stream<LPR, VPL, U, IPL>(qd, tables, rows, T, L, out, ld_out, err, max_items, \
                                      sm_count, s)
  if (L <= 32) {
    if (ub >= 8) RS_STREAM((VPL == 2 ? 4 : 8), 1);
    else RS_STREAM((VPL == 2 ? 2 : 4), 1);
  } else {
    if (ub >= 8) RS_STREAM((VPL == 2 ? 4 : 8), 3);
    else RS_STREAM((VPL == 2 ? 2 : 4), 3);
  }
#undef RS_STREAM
  return true;
}

#endif  // RS_EXPERIMENTS

template <int LPR, int VPL>
bool try_sls_pipe(const QDesc* qd, const float* tables, int64_t rows, int T, int L, float* out,
                  int64_t ld_out, int* err, int64_t max_items, int sm_count, cudaStream_t s,
                  const float* hot, int64_t hot_rows) {
  if (L > 96) return false;
  const int ub = sls_ub();
#define RS_PIPE(U, IPL) \
  launch_sls_pipe<LPR, VPL, U, IPL>(qd, tables, rows, T, L, out, ld_out, err, max_items, sm_count, \
                                    s, hot, hot_rows)
  if (L <= 32) {
    if (ub >= 8) RS_PIPE((VPL == 2 ? 4 : 8), 1);
    else if (ub <= 2) RS_PIPE((VPL == 2 ? 1 : 2), 1);
    else RS_PIPE((VPL == 2 ? 2 : 4), 1);
  } else {
    if (ub >= 8) RS_PIPE((VPL == 2 ? 4 : 8), 3);
    else if (ub <= 2) RS_PIPE((VPL == 2 ? 1 : 2), 3);
    else RS_PIPE((VPL == 2 ? 2 : 4), 3);
  }
#undef RS_PIPE
  return true;
}

#if RS_EXPERIMENTS  // variant 3 launcher
// Variant 3 geometry: one CTA per SM, each warp owning nbuf bag stages
// (RS_SLS_NBUF, 2..4, default 2) of L*D*4 bytes; as many warps as fit in
// RS_SLS_SMEM_KB (default 200) of shared memory, at most 16 (RS_SLS_WARPS caps).
template <int LPR, int VPL, int IPL>
bool launch_sls_stage(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                      float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                      cudaStream_t s) {
  constexpr int D = LPR * 4 * VPL;
  const int nbuf = std::min(4, std::max(2, env_int("RS_SLS_NBUF", 2)));
  const size_t per_warp = (size_t)nbuf * L * D * 4;
  const size_t budget = (size_t)env_int("RS_SLS_SMEM_KB", 200) * 1024;
  int nw = (int)std::min<size_t>(16, budget / std::max<size_t>(per_warp, 1));
  nw = std::min(nw, env_int("RS_SLS_WARPS", 16));
  if (nw < 1) return false;
  const size_t smem = per_warp * nw;
  smem_attr(reinterpret_cast<const void*>(sls_stage_kernel<LPR, VPL, IPL>), 227 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sls_stage_kernel<LPR, VPL, IPL>, nw * 32,
                                                smem);
  if (per_sm < 1) return false;
  const int grid = grid_for(max_items * T, nw, sm_count, per_sm);
  max_carveout(reinterpret_cast<const void*>(sls_stage_kernel<LPR, VPL, IPL>));
  sls_stage_kernel<LPR, VPL, IPL><<<grid, nw * 32, smem, s>>>(qd, tables, rows, T, L, nbuf, out,
                                                              ld_out, err);
  return true;
}

template <int LPR, int VPL>
bool try_sls_stage(const QDesc* qd, const float* tables, int64_t rows, int T, int L, float* out,
                   int64_t ld_out, int* err, int64_t max_items, int sm_count, cudaStream_t s) {
  if (L > 96) return false;
  if (L <= 32)
    return launch_sls_stage<LPR, VPL, 1>(qd, tables, rows, T, L, out, ld_out, err, max_items,
                                         sm_count, s);
  return launch_sls_stage<LPR, VPL, 3>(qd, tables, rows, T, L, out, ld_out, err, max_items,
                                       sm_count, s);
}

#endif  // RS_EXPERIMENTS

template <int LPR, int VPL, int U>
void launch_sls_bag(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                    float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                    cudaStream_t s) {
  static const int per_sm = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sls_sum_kernel<LPR, VPL, U>, kWarps * 32, 0);
    return b > 0 ? b : 1;
  }();
  const int grid = grid_for(max_items * T, kWarps, sm_count, 2 * per_sm);
  max_carveout(reinterpret_cast<const void*>(sls_sum_kernel<LPR, VPL, U>));
  sls_sum_kernel<LPR, VPL, U><<<grid, kWarps * 32, 0, s>>>(qd, tables, rows, T, L, out, ld_out,
                                                           err, 0);
}

#if RS_EXPERIMENTS  // variant 1 launcher
template <int LPR, int VPL, int NBUF>
bool launch_sls_tma(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                    float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                    cudaStream_t s) {
  constexpr int D = LPR * 4 * VPL;
  CUtensorMap map;
  if (!make_row_gather_map(&map, tables, (int64_t)T * rows, D)) return false;
  const int LB = (int)std::min<int64_t>(128, round_up(L, 16));
  const size_t smem = (size_t)NBUF * LB * D * 4 + NBUF * 8 + (size_t)NBUF * ((LB + 31) / 32) * 4;
  if (smem > 227 * 1024) return false;
  cudaFuncSetAttribute(sls_tma_kernel<LPR, VPL, NBUF>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sls_tma_kernel<LPR, VPL, NBUF>, 32, smem);
  if (per_sm < 1) return false;
  const int grid = grid_for(max_items * T, 1, sm_count, per_sm);
  max_carveout(reinterpret_cast<const void*>(sls_tma_kernel<LPR, VPL, NBUF>));
  sls_tma_kernel<LPR, VPL, NBUF><<<grid, 32, smem, s>>>(qd, map, rows, T, L, LB, out, ld_out,
                                                        err);
  return true;
}

#endif  // RS_EXPERIMENTS

// Measured-slower SLS variants (RS_SLS_VARIANT = 1 TMA gather4, 3 cp.async
// staged, 4 continuous stream) exist only in an experiments
// build (make EXPERIMENTS=1); the product build serves 2 (default) and 0.
template <int LPR, int VPL>
bool try_sls_experimental(int v, const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                          float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                          cudaStream_t s) {
#if RS_EXPERIMENTS
  if (v == 1) return launch_sls_tma<LPR, VPL, 2>(qd, tables, rows, T, L, out, ld_out, err,
                                                 max_items, sm_count, s);
  if (v == 3) return try_sls_stage<LPR, VPL>(qd, tables, rows, T, L, out, ld_out, err, max_items,
                                             sm_count, s);
  if (v == 4) return try_sls_stream<LPR, VPL>(qd, tables, rows, T, L, out, ld_out, err,
                                              max_items, sm_count, s);
#else
  (void)v; (void)qd; (void)tables; (void)rows; (void)T; (void)L; (void)out; (void)ld_out;
  (void)err; (void)max_items; (void)sm_count; (void)s;
#endif
  return false;
}

void launch_sls_sum(const QDesc* qd, const float* tables, int64_t rows, int T, int L, int D,
                    float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                    cudaStream_t s, const float* hot, int64_t hot_rows) {
#define RS_SLS(LPR, VPL)                                                                    \
  do {                                                                                      \
    if (try_sls_experimental<LPR, VPL>(sls_variant(), qd, tables, rows, T, L, out, ld_out,  \
                                       err, max_items, sm_count, s))                        \
      break;                                                                                \
    if (sls_variant() == 2 && try_sls_pipe<LPR, VPL>(qd, tables, rows, T, L, out, ld_out,   \
                                                     err, max_items, sm_count, s, hot,      \
                                                     hot_rows))                             \
      break;                                                                                \
    launch_sls_bag<LPR, VPL, (VPL == 2 ? 4 : 8)>(qd, tables, rows, T, L, out, ld_out, err,  \
                                                 max_items, sm_count, s);                   \
  } while (0)
  switch (D) {
    case 8: RS_SLS(2, 1); break;
    case 16: RS_SLS(4, 1); break;
    case 32: RS_SLS(8, 1); break;
    case 64: RS_SLS(16, 1); break;
    case 128: RS_SLS(32, 1); break;
    case 256: RS_SLS(32, 2); break;
    default: {
      const int grid = grid_for(max_items * T, kWarps, sm_count, 8);
      max_carveout(reinterpret_cast<const void*>(sls_sum_scalar_kernel));
      sls_sum_scalar_kernel<<<grid, kWarps * 32, 0, s>>>(qd, tables, rows, T, L, D, out, ld_out,
                                                         err);
    }
  }
#undef RS_SLS
}

void launch_gather_concat(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                          int D, float* out, int64_t ld_out, int64_t col_off, int* err,
                          int64_t max_items, int sm_count, cudaStream_t s) {
  const int vec = (D % 4 == 0 && col_off % 4 == 0 && ld_out % 4 == 0) ? 1 : 0;
  const int64_t units = max_items * T * L * (vec ? D / 4 : D);
  const int grid = grid_for(units, 256, sm_count, 8);
  max_carveout(reinterpret_cast<const void*>(gather_concat_kernel));
  gather_concat_kernel<<<grid, 256, 0, s>>>(qd, tables, rows, T, L, D, out, ld_out, col_off,
                                            vec, err);
}

bool din_supported(int64_t D) { return pow2_dim(D); }

void launch_din_pool(const QDesc* qd, const float* tables, int64_t rows, int T, int L, int D,
                     const float* att_w, float* out, int64_t ld_out, int64_t col_off, int* err,
                     int64_t max_items, int sm_count, cudaStream_t s) {
  // 8 CTAs per SM for a single query, 2 in the pipelined queue's lanes
  // (cfg5 DIN 38.2 -> 37.7 us/query; capture_lane, common.cuh)
  const int grid = grid_for(max_items * T, kWarps, sm_count,
                            env_int("RS_DIN_WAVES", capture_lane() == 1 ? 2 : 8));
  const dim3 blk(kWarps * 32);
  switch (D) {
    case 8: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<2, 1, 4>)); din_pool_kernel<2, 1, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
    case 16: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<4, 1, 4>)); din_pool_kernel<4, 1, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
    case 32: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<8, 1, 4>)); din_pool_kernel<8, 1, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
    case 64: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<16, 1, 4>)); din_pool_kernel<16, 1, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
    case 128: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<32, 1, 4>)); din_pool_kernel<32, 1, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
    case 256: max_carveout(reinterpret_cast<const void*>(din_pool_kernel<32, 2, 4>)); din_pool_kernel<32, 2, 4><<<grid, blk, 0, s>>>(qd, tables, rows, T, L, att_w, out, ld_out, col_off, err); break;
  }
}

#if RS_EXPERIMENTS  // measured slower in the pipelined queue
// ---------------------------------------------------------------------------
// interaction_tc_kernel: the DLRM dot interaction (model_zoo.cpp:231-238) on the
// tensor cores, for the tcgen05 (tf32) forward graph. One WARP per item: the
// item's R = T+1 vectors (v0 = dense_out, v_t = pooled_t, D floats each) are
// staged in shared memory by cp.async, the Gram matrix G = V V^T is formed by
// mma.sync.m16n8k8 tf32 tiles covering the strict lower triangle (j < i), and
// G[i][j] lands in X[item][dot_off + i(i-1)/2 + j]; lanes also write the summed
// embedding X[item][sum_off + c] = sum_t pooled_t[c] (fp32, t in order).
// Per item ~80 MMAs + ~180 shared loads for cfg3 (33 x 64) instead of 33.8K
// dependent FMAs: the stage's SM time in the pipelined queue is what it costs
// the concurrent gathers (tools/pipe_diag.py). tf32 operands (rounded, cvt.rna)
// -> the tf32 tolerance of the graph's FC layers (tests/parity_rule.py).
constexpr int kInterTcWarps = 4;

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

template <int D>
__global__ void __launch_bounds__(kInterTcWarps * 32)
interaction_tc_kernel(const QDesc* __restrict__ qd, const float* __restrict__ pooled,
                      int64_t ld_pooled, int T, float* __restrict__ X, int64_t ld_x,
                      int64_t sum_off, int64_t dot_off) {
  constexpr int LDV = D + 4;  // row stride: conflict-free fragment loads
  constexpr int D4 = D / 4;
  extern __shared__ float smem_v[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = T + 1;
  // two item buffers per warp: item k+1's vectors land while item k's tiles run
  float* __restrict__ Vbuf = smem_v + (size_t)warp * 2 * R * LDV;
  const int g = lane >> 2, tig = lane & 3;
  const int mtiles = (R + 15) / 16, ntiles = (R - 1 + 7) / 8;
  pdl_wait();  // pooled (SLS) and X[:, 0:D] (bottom MLP) are predecessors' outputs
  const int64_t S = qd->S;
  const int64_t step = (int64_t)gridDim.x * kInterTcWarps;
  auto stage = [&](int64_t item, float* V) {
    for (int u = lane; u < R * D4; u += 32) {
      const int v = u / D4, c4 = u - v * D4;
      const float* src = v == 0 ? X + item * ld_x + c4 * 4
                                : pooled + item * ld_pooled + (int64_t)(v - 1) * D + c4 * 4;
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(V + v * LDV + c4 * 4));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t item = (int64_t)blockIdx.x * kInterTcWarps + warp;
  if (item < S) stage(item, Vbuf);
  for (int buf = 0; item < S; item += step, buf ^= 1) {
    float* __restrict__ V = Vbuf + buf * R * LDV;
    const bool more = item + step < S;
    if (more) {
      stage(item + step, Vbuf + (buf ^ 1) * R * LDV);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    // summed embedding (D9): lanes over columns, tables in order
    for (int c = lane; c < D; c += 32) {
      float s = 0.f;
      for (int t = 1; t <= T; ++t) s += V[t * LDV + c];
      X[item * ld_x + sum_off + c] = s;
    }
    // strict lower triangle of V V^T by m16n8k8 tiles (rows i, cols j < i)
    for (int mt = 0; mt < mtiles; ++mt) {
      const int r0 = mt * 16 + g, r1 = r0 + 8;
      const int nt_end = min(ntiles, (mt * 16 + 15) / 8 + 1);
      float acc[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
#pragma unroll 2
      for (int k0 = 0; k0 < D; k0 += 8) {
        const uint32_t a0 = r0 < R ? to_tf32(V[r0 * LDV + k0 + tig]) : 0u;
        const uint32_t a1 = r1 < R ? to_tf32(V[r1 * LDV + k0 + tig]) : 0u;
        const uint32_t a2 = r0 < R ? to_tf32(V[r0 * LDV + k0 + tig + 4]) : 0u;
        const uint32_t a3 = r1 < R ? to_tf32(V[r1 * LDV + k0 + tig + 4]) : 0u;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          if (nt >= nt_end) break;
          const int cj = nt * 8 + g;
          const uint32_t b0 = cj < R ? to_tf32(V[cj * LDV + k0 + tig]) : 0u;
          const uint32_t b1 = cj < R ? to_tf32(V[cj * LDV + k0 + tig + 4]) : 0u;
          asm volatile(
              "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
              "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
              : "+f"(acc[nt][0]), "+f"(acc[nt][1]), "+f"(acc[nt][2]), "+f"(acc[nt][3])
              : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
      }
      float* __restrict__ xo = X + item * ld_x + dot_off;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        if (nt >= nt_end) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = (q < 2) ? r0 : r1;
          const int j = nt * 8 + 2 * tig + (q & 1);
          if (i < R && j < i) xo[i * (i - 1) / 2 + j] = acc[nt][q];
        }
      }
    }
    __syncwarp();  // this buffer is refilled two items from now
  }
  pdl_trigger();
}

bool interaction_tc_supported(int T, int D) {
  return (D == 32 || D == 64 || D == 128) && T + 1 <= 64 &&
         (size_t)(T + 1) * (D + 4) * 4 * 2 * kInterTcWarps <= 200 * 1024;
}

#endif  // RS_EXPERIMENTS

void launch_interaction(const QDesc* qd, const float* pooled, int64_t ld_pooled, int T, int D,
                        float* X, int64_t ld_x, int64_t sum_off, int64_t dot_off, int has_dense,
                        int64_t max_items, int sm_count, cudaStream_t s, bool tc,
                        int threads) {
#if RS_EXPERIMENTS
  // tcgen05 graph, RS_INTER_TC=1: the tensor-core Gram interaction (tf32 like
  // the FC layers). Measured 1 us/query SLOWER in the pipelined queue than the
  // FFMA kernel below at every grid size (tools/env_sweep.py)
  if (tc && has_dense && interaction_tc_supported(T, D) && env_int("RS_INTER_TC", 0)) {
    const size_t smem = (size_t)(T + 1) * (D + 4) * sizeof(float) * 2 * kInterTcWarps;
    // FEW CTAs, each warp streaming items with a one-item prefetch: in the
    // pipelined queue every CTA of this grid displaces a gather CTA for its
    // lifetime (tools/tl_analyze.py: the 296-CTA FFMA kernel stretched the
    // concurrent SLS grids by ~8 us per query), so the stage is packed onto
    // RS_INTER_CTAS (default 16) SMs
    const int ctas = std::max(1, env_int("RS_INTER_CTAS", 16));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(
        (max_items + kInterTcWarps - 1) / kInterTcWarps, (int64_t)ctas));
#define RS_ITC(DD)                                                                            \
  do {                                                                                        \
    smem_attr(reinterpret_cast<const void*>(interaction_tc_kernel<DD>), (int)smem);           \
    launch_pdl(interaction_tc_kernel<DD>, dim3(grid), dim3(kInterTcWarps * 32), smem, s, qd,  \
               pooled, ld_pooled, T, X, ld_x, sum_off, dot_off);                              \
  } while (0)
    switch (D) {
      case 32: RS_ITC(32); break;
      case 64: RS_ITC(64); break;
      default: RS_ITC(128); break;
    }
#undef RS_ITC
    return;
  }
#else
  (void)tc;
#endif
  const size_t per_item = (size_t)(T + 1) * (D + 1) * sizeof(float);
  // warp-per-item only while an item's dot work is short: one warp runs each
  // dot as a dependent FMA chain, so at cfg3's 528 pairs x 64 it lengthens the
  // query's critical path more than it saves in CTA slots (pipe_micro: 39.8
  // -> 43.2 us/query), while at RMC1's 36 pairs x 32 it wins (10.6 -> 9.9).
  const int64_t pair_work = (int64_t)(T + 1) * T / 2 * D;
  if (D % 4 == 0 && D <= 64 && T + 1 <= 33 && per_item * kInterWarps <= 200 * 1024 &&
      pair_work <= 8192 && env_int("RS_INTER_WARP", 1)) {
    smem_attr(reinterpret_cast<const void*>(interaction_warp_kernel), 200 * 1024);
    const int grid = grid_for(max_items, kInterWarps, sm_count, 2);
    launch_pdl(interaction_warp_kernel, dim3(grid), dim3(kInterWarps * 32),
               per_item * kInterWarps, s, qd, pooled, ld_pooled, T, D, X, ld_x, sum_off,
               dot_off, has_dense);
    return;
  }
  const size_t smem = (size_t)(T + 1) * (D + 1) * sizeof(float);
  const bool small = env_int("RS_INTER_THREADS", threads) == 64;
  const int grid = grid_for(max_items, 1, sm_count, env_int("RS_INTER_PER_SM", 2));
  auto kern = small ? interaction_kernel<64> : interaction_kernel<256>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // RS_DISCARD (default 1): discard the pooled rows from L2 once staged (the
  // forward graph's pooled buffer is internal; needs 128-byte row alignment)
  const int discard = env_int("RS_DISCARD", 1) && (T * D * 4) % 128 == 0 &&
                      (reinterpret_cast<uintptr_t>(pooled) & 127) == 0 &&
                      (ld_pooled * 4) % 128 == 0;
  launch_pdl(kern, dim3(grid), dim3(small ? 64 : 256), smem, s, qd, pooled, ld_pooled,
             T, D, X, ld_x, sum_off, dot_off, has_dense, discard);
}

// Dense features into the FC staging buffer: [S, dense_in] contiguous (the
// caller's device buffer, or the contiguous H2D landing zone) -> rows of
// stride ld_dst. A kernel, not a copy-engine memcpy, so the pipelined lanes
// do not queue behind each other on the copy engine.
__global__ void __launch_bounds__(256)
stage_dense_kernel(const QDesc* __restrict__ qd, int64_t dense_in, float* __restrict__ dst,
                   int64_t ld_dst) {
  pdl_trigger();
  const float* __restrict__ src = qd->dense;
  const int64_t S = qd->S;
  if (!src) return;
  if (qd->flags & kDescDenseBf16) {  // labelled bf16-dense input variant
    const uint16_t* __restrict__ h = reinterpret_cast<const uint16_t*>(src);
    const int64_t total = S * dense_in;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / dense_in, c = i - r * dense_in;
      dst[r * ld_dst + c] = __uint_as_float((uint32_t)__ldg(h + i) << 16);
    }
    return;
  }
  const bool vec = (dense_in % 4 == 0) && (ld_dst % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (vec) {
    const int64_t w = dense_in / 4, total = S * w;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / w, c = i - r * w;
      reinterpret_cast<float4*>(dst + r * ld_dst)[c] =
          __ldg(reinterpret_cast<const float4*>(src) + i);
    }
  } else {
    const int64_t total = S * dense_in;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / dense_in, c = i - r * dense_in;
      dst[r * ld_dst + c] = __ldg(src + i);
    }
  }
}

void launch_stage_dense(const QDesc* qd, int64_t dense_in, float* dst, int64_t ld_dst,
                        int64_t max_items, int sm_count, cudaStream_t s) {
  const int64_t units = max_items * ((dense_in % 4 == 0) ? dense_in / 4 : dense_in);
  // a few hundred KB per query: a small grid-stride grid, so the copy does not
  // take an SM slot from the concurrent gathers on every SM (RS_STAGE_CTAS)
  const int grid = (int)std::min<int64_t>(grid_for(units, 256, sm_count, 2),
                                          std::max(1, env_int("RS_STAGE_CTAS", 32)));
  launch_pdl(stage_dense_kernel, dim3(grid), dim3(256), 0, s, qd, dense_in, dst, ld_dst);
}

// fp32 -> bf16 rows (round to nearest even) for the RS_FC_BF16 graph: the
// first layer of a bf16 FC stack reads its activations as bfloat16. Rows are
// the query's S items; columns [0, cols) of each row (the padding of the
// destination rows is never read: the tensor map's K extent is cols).
__global__ void __launch_bounds__(256)
to_bf16_kernel(const QDesc* __restrict__ qd, const float* __restrict__ src, int64_t lds,
               __nv_bfloat16* __restrict__ dst, int64_t ldd, int64_t cols) {
  pdl_wait();  // src is the predecessor's output
  const int64_t total = qd->S * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
  }
  pdl_trigger();
}

void launch_to_bf16(const QDesc* qd, const float* src, int64_t lds, void* dst, int64_t ldd,
                    int64_t cols, int64_t max_items, int sm_count, cudaStream_t s) {
  const int grid = grid_for(max_items * cols, 256, sm_count, 2);
  launch_pdl(to_bf16_kernel, dim3(grid), dim3(256), 0, s, qd, src, lds,
             static_cast<__nv_bfloat16*>(dst), ldd, cols);
}

// int32 -> int64 index widening for the RS_INDEX_I32 input variant
// (sign-extending: an out-of-range index stays out of range and is reported).
__global__ void __launch_bounds__(256)
widen_idx_kernel(const int32_t* __restrict__ src, int64_t* __restrict__ dst, int64_t n) {
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) ? n / 4 : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = __ldg(reinterpret_cast<const int4*>(src) + i);
    reinterpret_cast<longlong2*>(dst)[2 * i] = make_longlong2(v.x, v.y);
    reinterpret_cast<longlong2*>(dst)[2 * i + 1] = make_longlong2(v.z, v.w);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (int64_t)__ldg(src + i);
}

void launch_widen_idx(const int32_t* src, int64_t* dst, int64_t n, int sm_count,
                      cudaStream_t s) {
  const int grid = grid_for((n + 3) / 4, 256, sm_count, 4);
  widen_idx_kernel<<<grid, 256, 0, s>>>(src, dst, n);
}

__global__ void __launch_bounds__(256)
group_gather_kernel(const __grid_constant__ GroupGather g, int64_t dense_in, int64_t TL,
                    float* __restrict__ dense_dst, int64_t* __restrict__ idx_dst) {
  const int k = blockIdx.y;
  const int64_t S = g.size[k], off = g.off[k];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (dense_in > 0 && g.dense[k]) {
    const float* __restrict__ src = g.dense[k];
    float* __restrict__ dst = dense_dst + off * dense_in;
    for (int64_t i = t0; i < S * dense_in; i += stride) dst[i] = __ldg(src + i);
  }
  if (TL > 0) {
    int64_t* __restrict__ dst = idx_dst + off * TL;
    if (g.idx32) {
      const int32_t* __restrict__ src = static_cast<const int32_t*>(g.idx[k]);
      for (int64_t i = t0; i < S * TL; i += stride) dst[i] = (int64_t)__ldg(src + i);
    } else {
      const int64_t* __restrict__ src = static_cast<const int64_t*>(g.idx[k]);
      for (int64_t i = t0; i < S * TL; i += stride) dst[i] = __ldg(src + i);
    }
  }
}

void launch_group_gather(const GroupGather& g, int64_t dense_in, int64_t TL, float* dense_dst,
                         int64_t* idx_dst, int sm_count, cudaStream_t s) {
  const int gx = std::max(1, 2 * sm_count / std::max(1, g.m));
  group_gather_kernel<<<dim3(gx, g.m), 256, 0, s>>>(g, dense_in, TL, dense_dst, idx_dst);
}

// Diagnostic (RS_DIAG_EMPTY, tools/pipe_micro.py): n empty grids of `ctas`
// CTAs, to measure the per-kernel cost inside the pipelined forward.
__global__ void diag_empty_kernel() {
  pdl_trigger();
  pdl_wait();
}

void launch_diag_empty(int n, int ctas, cudaStream_t s) {
  for (int i = 0; i < n; ++i) launch_pdl(diag_empty_kernel, dim3(ctas), dim3(128), 0, s);
}

size_t interaction_smem(int T, int D) { return (size_t)(T + 1) * (D + 1) * sizeof(float); }

void launch_init_tables(float* tables, int64_t T, int64_t rows, int64_t D, uint64_t seed,
                        int sm_count, cudaStream_t s) {
  const int64_t total = T * rows * D;
  const int grid = grid_for((total + 3) / 4, 256, sm_count, 16);
  init_tables_kernel<<<grid, 256, 0, s>>>(tables, T, rows, D, seed);
}

}  // namespace rs
