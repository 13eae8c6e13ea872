// gru_tcgen05.cu — DIEN interest-evolution GRU/AUGRU (AttentionRNN,
// proj/src/model_zoo.cpp:217-227) on the 5th-generation tensor cores.
//
// One CTA owns 128 sequences (items) of one table for all L steps. Per step,
// ONE chain of tcgen05.mma (kind::tf32, M=128, N=4H, K=D+H in 8-wide slices)
// computes every gate pre-activation of every sequence:
//
//   [x_t | h_t] (128 x (D+H), smem, SWIZZLE_128B K-major)
//     x  [ W_ir W_hr ; W_iz W_hz ; W_in 0 ; 0 W_hn ]^T  ((D+H) x 4H, smem)
//   -> TMEM columns [r | z | n_x | n_h], fp32
//
// The epilogue is split over two threads per sequence: warps w and w+4 read
// the same TMEM lanes (sequences 32(w%4)..+31) but different halves of the
// hidden units. Each thread applies the cell (biases folded per
// gate) to its units and writes h_{t+1} straight back into the swizzled A
// operand (generic-proxy writes fenced to the async proxy before the next
// MMA). The next step's embedding rows are prefetched into registers while
// the MMA runs. The recurrence is serial in t: per step one MMA chain and one
// epilogue; the tensor core replaces the 18K FFMA per sequence-step of
// gru.cu's FFMA kernel.
#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace rs {
namespace {

constexpr int kSeq = 128;           // sequences per CTA = UMMA M = TMEM lanes
// Threads per sequence: the hidden units of a sequence are split over TPS
// threads (warps w, w+4, ... share TMEM lanes 32(w%4)..+31). Build knob;
// TPS=4 (512 threads, 128 registers) measured slower for DIEN cfg5
// (126 -> 142 us/query: spills and the per-step barrier over 16 warps).
#ifndef RS_GRU_TPS
#define RS_GRU_TPS 2
#endif
template <int H>
struct GruThreads {
  static constexpr int TPS = H >= 64 ? RS_GRU_TPS : 2;  // >= 16 units per thread
  static constexpr int N = TPS * kSeq;
};

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// byte offset of fp32 element (row, c) inside a 128-row x 32-col SW128 atom
__device__ __forceinline__ uint32_t sw_off(int row, int c) {
  return (uint32_t)(row * 128 + ((((c >> 2) ^ row) & 7) << 4) + (c & 3) * 4);
}
// Cell nonlinearities: one MUFU.TANH each (tanh.approx.f32; sigmoid(x) =
// 0.5 + 0.5 tanh(x/2)). The epilogue of a 128-sequence step is bound by the
// SM's SFU (128 x H units x 3 transcendental ops), and ex2 + rcp pairs took
// twice the SFU issue. tanh.approx's ~2^-11 relative error stays inside the
// tf32 tolerance this path is checked against (tests/test_gpu_parity.py);
// RS_GRU_EXACT_SFU=1 at build time restores the ex2/rcp forms.
#ifndef RS_GRU_EXACT_SFU
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }
#else
__device__ __forceinline__ float sigm(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_fast(float x) {
  return 1.0f - __fdividef(2.0f, __expf(2.0f * x) + 1.0f);
}
#endif

template <int D, int H>
struct GruTcSmem {
  static constexpr int KA = (D + H) / 32;  // K atoms
  static constexpr int N = 4 * H;
  alignas(1024) uint8_t b[KA][N * 128];     // weights, per K atom
  alignas(1024) uint8_t ax[2][D / 32][kSeq * 128];
  alignas(1024) uint8_t ah[H / 32][kSeq * 128];
  alignas(16) float bias[N];
  uint64_t mma_done;
  uint32_t tmem_base;
};

template <int D, int H>
__global__ void __launch_bounds__(GruThreads<H>::N, 1)
gru_tc_kernel(const QDesc* __restrict__ qd, GruArgs g) {
  using SM = GruTcSmem<D, H>;
  constexpr int N = SM::N, KA = SM::KA, DA = D / 32;
  constexpr int kTps = GruThreads<H>::TPS, kThreads = GruThreads<H>::N;
  constexpr int HU = H / kTps;  // hidden units per thread
  constexpr int DX = D / kTps;  // x elements fetched per thread
  static_assert(HU % 8 == 0, "hidden units per thread");
  static_assert(DX % 4 == 0, "x elements per thread");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by offsetting smem_raw itself (not through an integer round trip) so
  // the compiler keeps the shared address space: LDS/STS, not generic LD/ST
  SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024u - (s_u32(smem_raw) & 1023u)) & 1023u));
  const int t = blockIdx.y;
  const int64_t item0 = (int64_t)blockIdx.x * kSeq;
  const int64_t S = qd->S;
  if (item0 >= S) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;  // half = which slice of the units
  const int row = quad * 32 + lane;          // sequence = TMEM lane
  const int u0 = half * HU;                  // this thread's hidden units
  const int64_t item = item0 + row;
  const bool live = item < S;
  const int L = g.L;
  const int64_t* __restrict__ idx = qd->idx;
  const float* __restrict__ tab = g.tables + (int64_t)t * g.rows * D;

  // ---- weights -> swizzled K-major B operand; folded biases; h_0 = 0 ----
  {
    const float* Wih = g.w_ih + (int64_t)t * 3 * H * D;
    const float* Whh = g.w_hh + (int64_t)t * 3 * H * H;
    // 128-bit loads along k (D and H are multiples of 4, so a vector never
    // straddles the x/h boundary), 4 in flight per thread, one 16-byte store
    // each into the swizzled K-major layout (the CTA prologue was ~8% of the
    // kernel with scalar loads)
    constexpr int K4 = (D + H) / 4;
    constexpr int kU = 4;
    for (int e0 = tid; e0 < N * K4; e0 += kThreads * kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kThreads;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < N * K4) {
          const int n = e / K4, k = (e - n * K4) * 4;
          const int gate = n / H, j = n - gate * H;
          if (k < D) {
            if (gate < 3)
              v[u] = __ldg(reinterpret_cast<const float4*>(Wih + (int64_t)(gate * H + j) * D + k));
          } else {
            const int kh = k - D;
            const int row = gate < 2 ? gate * H + j : (gate == 3 ? 2 * H + j : -1);
            if (row >= 0)
              v[u] = __ldg(reinterpret_cast<const float4*>(Whh + (int64_t)row * H + kh));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kThreads;
        if (e < N * K4) {
          const int n = e / K4, k = (e - n * K4) * 4;
          const int atom = k >> 5, c = k & 31;
          *reinterpret_cast<float4*>(sm.b[atom] + n * 128 + ((((c >> 2) ^ n) & 7) << 4)) = v[u];
        }
      }
    }
    const float* bih = g.b_ih + (int64_t)t * 3 * H;
    const float* bhh = g.b_hh + (int64_t)t * 3 * H;
    for (int n = tid; n < N; n += kThreads) {
      const int gate = n / H, j = n - gate * H;
      sm.bias[n] = gate == 0 ? bih[j] + bhh[j]
                 : gate == 1 ? bih[H + j] + bhh[H + j]
                 : gate == 2 ? bih[2 * H + j] : bhh[2 * H + j];
    }
#pragma unroll
    for (int j = 0; j < HU; j += 4)
      *reinterpret_cast<float4*>(sm.ah[(u0 + j) >> 5] + sw_off(row, (u0 + j) & 31)) =
          make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s_u32(&sm.tmem_base)), "r"(2 * N) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&sm.mma_done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // ---- this thread's half of the x row of step l (two steps of lookahead:
  // a random HBM row per sequence per step is the recurrence's only memory
  // traffic, so its latency must hide behind two MMA + epilogue rounds) ----
  float4 xa[DX / 4], xb2[DX / 4];
  // the row index of step l+1 is loaded one step before its row is fetched,
  // so no step waits a memory latency on an index (ncu: long-scoreboard
  // stalls were the largest share before this)
  const int64_t* __restrict__ my_idx = idx + (item * g.T + t) * L;
  auto load_index = [&](int l) -> int64_t { return (live && l < L) ? __ldg(my_idx + l) : 0; };
  int64_t next_r = 0;
  auto fetch = [&](int l, float4* xn, int64_t r) {
#pragma unroll
    for (int q = 0; q < DX / 4; ++q) xn[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!live || l >= L) return;
    if ((uint64_t)r >= (uint64_t)g.rows) {
      if (half == 0) atomicOr(g.err, kErrIndex);
      return;
    }
    const float4* p = reinterpret_cast<const float4*>(tab + r * D + half * DX);
#pragma unroll
    for (int q = 0; q < DX / 4; ++q) xn[q] = ldg_stream(p + q);
  };
  auto stash = [&](int buf, const float4* xn) {
#pragma unroll
    for (int q = 0; q < DX / 4; ++q) {
      const int c = half * DX + 4 * q;
      *reinterpret_cast<float4*>(sm.ax[buf][c >> 5] + sw_off(row, c & 31)) = xn[q];
    }
  };
  fetch(0, xa, load_index(0));
  stash(0, xa);
  fetch(1, xa, load_index(1));
  stash(1, xa);
  next_r = load_index(2);

  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  // AUGRU: ua = W_a^T x_0 (full row, both threads of the sequence)
  float ua[D];
  if (g.augru) {
    const float* Wa = g.w_att + (int64_t)t * D * D;
#pragma unroll
    for (int c = 0; c < D; ++c) ua[c] = 0.f;
    for (int i = 0; i < D; ++i) {
      const float xi = *reinterpret_cast<const float*>(sm.ax[0][i >> 5] + sw_off(row, i & 31));
#pragma unroll
      for (int c = 0; c < D; ++c) ua[c] = fmaf(xi, __ldg(Wa + i * D + c), ua[c]);
    }
  }
  // instruction descriptors by N: the x-part covers gate blocks [r|z|n_x]
  // (3H columns), the h-part [r|z] (2H) and [n_h] (H, at column 3H) — the
  // zero blocks of the packed weights (W_x for n_h, W_h for n_x) are skipped
  auto make_idesc = [](int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(kSeq >> 4) << 24);
  };
  const uint32_t id_x = make_idesc(3 * H), id_rz = make_idesc(2 * H), id_nh = make_idesc(H);

  // Two TMEM accumulators: while step l's cell math runs, the tensor core
  // already computes step l+1's input projection x_{l+1} W_x (it does not
  // depend on h); after the epilogue only the h-part is on the critical path.
  // n0: first gate row / accumulator column of the block, id: its N
  auto issue = [&](uint32_t acc_tmem, int a_begin, int a_end, const uint8_t* ax_buf,
                   bool first_init, int n0, uint32_t id) {
#pragma unroll
    for (int a = a_begin; a < a_end; ++a) {
      const uint32_t abase = a < DA ? s_u32(ax_buf + a * kSeq * 128) : s_u32(sm.ah[a - DA]);
      const uint32_t bbase = s_u32(sm.b[a]) + (uint32_t)n0 * 128;  // 8-row groups: 1024 B
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (first_init && a == a_begin && kk == 0) ? 0u : 1u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                acc_tmem + (uint32_t)n0),
            "l"(sw128(abase + kk * 32)), "l"(sw128(bbase + kk * 32)), "r"(id), "r"(acc)
            : "memory");
      }
    }
  };
  if (tid == 0) issue(tmem, 0, DA, sm.ax[0][0], true, 0, id_x);  // x_0 W_x

  for (int l = 0; l < L; ++l) {
    const int xb = l & 1;
    const uint32_t tcur = tmem + (uint32_t)(xb * N);
    if (tid == 0) {
      issue(tcur, DA, KA, nullptr, false, 0, id_rz);     // [r|z] += h_l W_h
      issue(tcur, DA, KA, nullptr, true, 3 * H, id_nh);  // [n_h]  = h_l W_hn
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              s_u32(&sm.mma_done))
          : "memory");
      if (l + 1 < L)
        issue(tmem + (uint32_t)((xb ^ 1) * N), 0, DA, sm.ax[xb ^ 1][0], true, 0, id_x);
    }
    float att = 1.f;
    if (g.augru) {  // a_l = sigmoid(<ua, x_l>) from the x row in shared memory
      float sc = 0.f;
#pragma unroll
      for (int c = 0; c < D; c += 4) {
        const float4 v = *reinterpret_cast<const float4*>(sm.ax[xb][c >> 5] + sw_off(row, c & 31));
        sc = fmaf(ua[c], v.x, sc); sc = fmaf(ua[c + 1], v.y, sc);
        sc = fmaf(ua[c + 2], v.z, sc); sc = fmaf(ua[c + 3], v.w, sc);
      }
      att = sigm(sc);
    }
    fetch(l + 2, xb2, next_r);  // rows two steps ahead fly during this MMA + epilogue
    next_r = load_index(l + 3);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(s_u32(&sm.mma_done)),
        "r"((uint32_t)(l & 1))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t lane_base = tcur + ((uint32_t)(quad * 32) << 16);
    // units per TMEM batch: 16 (x16 loads) with 2 threads per sequence, 8 with
    // 4 (keeps the 512-thread build under its 128-register cap)
    constexpr int UB = kTps <= 2 ? 16 : 8;
#pragma unroll
    for (int j0 = 0; j0 < HU; j0 += UB) {
      uint32_t v[4][UB];
#pragma unroll
      for (int gte = 0; gte < 4; ++gte) {
        const uint32_t ta = lane_base + (uint32_t)(gte * H + u0 + j0);
        if constexpr (UB == 16) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
              "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[gte][0]), "=r"(v[gte][1]), "=r"(v[gte][2]), "=r"(v[gte][3]),
                "=r"(v[gte][4]), "=r"(v[gte][5]), "=r"(v[gte][6]), "=r"(v[gte][7]),
                "=r"(v[gte][8]), "=r"(v[gte][9]), "=r"(v[gte][10]), "=r"(v[gte][11]),
                "=r"(v[gte][12]), "=r"(v[gte][13]), "=r"(v[gte][14]), "=r"(v[gte][15])
              : "r"(ta));
        } else {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=r"(v[gte][0]), "=r"(v[gte][1]), "=r"(v[gte][2]), "=r"(v[gte][3]),
                "=r"(v[gte][4]), "=r"(v[gte][5]), "=r"(v[gte][6]), "=r"(v[gte][7])
              : "r"(ta));
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < UB / 4; ++q) {
        const int j = u0 + j0 + 4 * q;
        uint8_t* hp = sm.ah[j >> 5] + sw_off(row, j & 31);
        const float4 ho = *reinterpret_cast<const float4*>(hp);
        const float hold[4] = {ho.x, ho.y, ho.z, ho.w};
        // the 4 units' folded biases of each gate: one 128-bit load per gate
        const float4 b4[4] = {*reinterpret_cast<const float4*>(&sm.bias[j]),
                              *reinterpret_cast<const float4*>(&sm.bias[H + j]),
                              *reinterpret_cast<const float4*>(&sm.bias[2 * H + j]),
                              *reinterpret_cast<const float4*>(&sm.bias[3 * H + j])};
        const float bb[4][4] = {{b4[0].x, b4[0].y, b4[0].z, b4[0].w},
                                {b4[1].x, b4[1].y, b4[1].z, b4[1].w},
                                {b4[2].x, b4[2].y, b4[2].z, b4[2].w},
                                {b4[3].x, b4[3].y, b4[3].z, b4[3].w}};
        float hn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jj = 4 * q + u;
          const float r = sigm(__uint_as_float(v[0][jj]) + bb[0][u]);
          const float z = sigm(__uint_as_float(v[1][jj]) + bb[1][u]);
          const float n = tanh_fast(__uint_as_float(v[2][jj]) + bb[2][u] +
                                    r * (__uint_as_float(v[3][jj]) + bb[3][u]));
          if (g.augru) {
            const float uu = att * (1.0f - z);
            hn[u] = (1.0f - uu) * hold[u] + uu * n;
          } else {
            hn[u] = (1.0f - z) * n + z * hold[u];
          }
        }
        *reinterpret_cast<float4*>(hp) = make_float4(hn[0], hn[1], hn[2], hn[3]);
      }
    }
    // x_{l+2} into the buffer x_l used (its MMA finished before step l's h-part)
    if (l + 2 < L) stash(xb, xb2);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }

  if (live) {  // h_L (this thread's units) from the A operand
    float* o = g.out + item * g.ld_out + g.col_off + (int64_t)t * H + u0;
#pragma unroll
    for (int j = 0; j < HU; j += 4) {
      const int jx = u0 + j;
      const float4 h = *reinterpret_cast<const float4*>(sm.ah[jx >> 5] + sw_off(row, jx & 31));
      o[j] = h.x; o[j + 1] = h.y; o[j + 2] = h.z; o[j + 3] = h.w;
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * N)
                 : "memory");
}

template <int D, int H>
void launch_typed(const QDesc* qd, const GruArgs& g, int64_t max_items, cudaStream_t s) {
  const size_t smem = sizeof(GruTcSmem<D, H>) + 1024;
  smem_attr(reinterpret_cast<const void*>(gru_tc_kernel<D, H>), (int)smem);
  const dim3 grid((unsigned)((max_items + kSeq - 1) / kSeq), g.T);
  max_carveout(reinterpret_cast<const void*>(gru_tc_kernel<D, H>));
  gru_tc_kernel<D, H><<<grid, GruThreads<H>::N, smem, s>>>(qd, g);
}

}  // namespace

bool gru_tc_supported(int D, int H) {
  return (D == 32 || D == 64) && (H == 32 || H == 64) && tc_available();
}

bool launch_gru_tc(const QDesc* qd, const GruArgs& g, int64_t max_items, cudaStream_t s) {
  if (!gru_tc_supported(g.D, g.H)) return false;
  if (g.D == 32 && g.H == 64) launch_typed<32, 64>(qd, g, max_items, s);
  else if (g.D == 32 && g.H == 32) launch_typed<32, 32>(qd, g, max_items, s);
  else if (g.D == 64 && g.H == 64) launch_typed<64, 64>(qd, g, max_items, s);
  else launch_typed<64, 32>(qd, g, max_items, s);
  return true;
}

}  // namespace rs
