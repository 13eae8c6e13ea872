// gru.cu — DIEN interest-evolution recurrence (AttentionRNN,
// proj/src/model_zoo.cpp:217-227): one GRU (or AUGRU) per (item, table)
// behaviour sequence of L = lookups_per_table steps, input x_l = E_t[idx_l],
// hidden width h = recurrent_hidden_dim; the final state feeds the predict
// stack (predict_input_dim's T*h sparse width, :126-128).
//
// Cell (PyTorch gate order r, z, n):
//   r = sig(W_ir x + b_ir + W_hr h + b_hr)
//   z = sig(W_iz x + b_iz + W_hz h + b_hz)
//   n = tanh(W_in x + b_in + r * (W_hn h + b_hn))
//   GRU:   h' = (1 - z) * n + z * h
//   AUGRU: a = sig(<W_a^T x_0, x_l>),  u = a * (1 - z),  h' = (1 - u) * h + u * n
//
// Persistent over time: one CTA owns NSEQ sequences of one table for all L
// steps. The table's gate weights sit transposed in shared memory, the
// hidden state in registers plus a transposed shared copy for the next
// step's broadcast reads; thread (j, group) produces hidden unit j for 8
// sequences, so each shared weight read feeds 8 FMAs. The next step's
// embedding rows are gathered into registers while the current step
// computes (the only HBM traffic of the recurrence).
#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace rs {
namespace {

constexpr int SPT = 8;     // sequences per thread
constexpr int MAXPF = 8;   // float4 prefetch registers per thread

int gru_groups(int H) { return std::max(1, 256 / H); }
int gru_threads(int H) { return gru_groups(H) * H; }
int gru_nseq(int H) { return SPT * gru_groups(H); }

size_t gru_smem(int D, int H, bool wsmem) {
  const int nseq = gru_nseq(H);
  size_t f = (size_t)(D + H + D) * nseq + nseq;
  if (wsmem) f += (size_t)(D + H) * 3 * H;
  return f * sizeof(float);
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

template <bool WSMEM>
__global__ void gru_kernel(const QDesc* __restrict__ qd, GruArgs g) {
  const int H = g.H, D = g.D, L = g.L;
  const int G = blockDim.x / H;
  const int NSEQ = SPT * G;
  const int t = blockIdx.y;
  const int64_t item0 = (int64_t)blockIdx.x * NSEQ;
  const int64_t S = qd->S;
  if (item0 >= S) return;
  const int64_t* __restrict__ idx = qd->idx;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int j = tid % H, sg = tid / H;
  const int H3 = 3 * H;

  extern __shared__ __align__(16) float sm[];
  float* xT = sm;                       // [D][NSEQ]
  float* hT = xT + (size_t)D * NSEQ;    // [H][NSEQ]
  float* uaT = hT + (size_t)H * NSEQ;   // [D][NSEQ]
  float* att = uaT + (size_t)D * NSEQ;  // [NSEQ]
  float* wih = att + NSEQ;              // [D][3H]   (WSMEM)
  float* whh = wih + (size_t)D * H3;    // [H][3H]   (WSMEM)

  const float* __restrict__ Wih = g.w_ih + (int64_t)t * H3 * D;
  const float* __restrict__ Whh = g.w_hh + (int64_t)t * H3 * H;
  if (WSMEM) {
    for (int e = tid; e < H3 * D; e += nthr) {
      const int row = e / D, k = e - row * D;
      wih[k * H3 + row] = Wih[e];
    }
    for (int e = tid; e < H3 * H; e += nthr) {
      const int row = e / H, k = e - row * H;
      whh[k * H3 + row] = Whh[e];
    }
  }
  for (int e = tid; e < H * NSEQ; e += nthr) hT[e] = 0.f;

  const float* __restrict__ tab = g.tables + (int64_t)t * g.rows * D;
  const int D4 = D / 4;
  const int units = NSEQ * D4;
  // gather step l's rows into registers
  auto fetch = [&](int l, float4* pf) {
#pragma unroll
    for (int q = 0; q < MAXPF; ++q) {
      const int u = tid + q * nthr;
      pf[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u < units) {
        const int s = u / D4, c4 = u - s * D4;
        const int64_t item = item0 + s;
        if (item < S) {
          const int64_t r = __ldg(idx + (item * g.T + t) * L + l);
          if ((uint64_t)r < (uint64_t)g.rows) {
            pf[q] = ldg_stream(reinterpret_cast<const float4*>(tab + r * D) + c4);
          } else if (c4 == 0) {
            atomicOr(g.err, kErrIndex);
          }
        }
      }
    }
  };
  auto stash = [&](const float4* pf) {
#pragma unroll
    for (int q = 0; q < MAXPF; ++q) {
      const int u = tid + q * nthr;
      if (u < units) {
        const int s = u / D4, c = (u - s * D4) * 4;
        xT[(c + 0) * NSEQ + s] = pf[q].x;
        xT[(c + 1) * NSEQ + s] = pf[q].y;
        xT[(c + 2) * NSEQ + s] = pf[q].z;
        xT[(c + 3) * NSEQ + s] = pf[q].w;
      }
    }
  };

  float4 pf[MAXPF];
  fetch(0, pf);
  stash(pf);
  __syncthreads();

  if (g.augru) {
    // uaT[c][s] = sum_i x0[s][i] * W_a[t][i][c]
    const float* __restrict__ Wa = g.w_att + (int64_t)t * D * D;
    for (int e = tid; e < D * NSEQ; e += nthr) {
      const int c = e / NSEQ, s = e - c * NSEQ;
      float acc = 0.f;
      for (int i = 0; i < D; ++i) acc = fmaf(xT[i * NSEQ + s], __ldg(Wa + (int64_t)i * D + c), acc);
      uaT[e] = acc;
    }
    __syncthreads();
  }

  const float* __restrict__ bih = g.b_ih + (int64_t)t * H3;
  const float* __restrict__ bhh = g.b_hh + (int64_t)t * H3;
  const float bir = bih[j], biz = bih[H + j], bin = bih[2 * H + j];
  const float bhr = bhh[j], bhz = bhh[H + j], bhn = bhh[2 * H + j];
  float h[SPT];
#pragma unroll
  for (int q = 0; q < SPT; ++q) h[q] = 0.f;
  const int s0 = sg * SPT;

  for (int l = 0; l < L; ++l) {
    if (g.augru && tid < NSEQ) {
      float acc = 0.f;
      for (int c = 0; c < D; ++c) acc = fmaf(uaT[c * NSEQ + tid], xT[c * NSEQ + tid], acc);
      att[tid] = sigm(acc);
    }
    if (l + 1 < L) fetch(l + 1, pf);

    float gr[SPT], gz[SPT], gn[SPT], hr[SPT], hz[SPT], hn[SPT];
#pragma unroll
    for (int q = 0; q < SPT; ++q) { gr[q] = gz[q] = gn[q] = hr[q] = hz[q] = hn[q] = 0.f; }
    for (int k = 0; k < D; ++k) {
      float wr, wz, wn;
      if (WSMEM) {
        wr = wih[k * H3 + j]; wz = wih[k * H3 + H + j]; wn = wih[k * H3 + 2 * H + j];
      } else {
        wr = __ldg(Wih + (int64_t)j * D + k);
        wz = __ldg(Wih + (int64_t)(H + j) * D + k);
        wn = __ldg(Wih + (int64_t)(2 * H + j) * D + k);
      }
      const float4 x0 = *reinterpret_cast<const float4*>(xT + k * NSEQ + s0);
      const float4 x1 = *reinterpret_cast<const float4*>(xT + k * NSEQ + s0 + 4);
      const float xs[SPT] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        gr[q] = fmaf(wr, xs[q], gr[q]);
        gz[q] = fmaf(wz, xs[q], gz[q]);
        gn[q] = fmaf(wn, xs[q], gn[q]);
      }
    }
    for (int k = 0; k < H; ++k) {
      float wr, wz, wn;
      if (WSMEM) {
        wr = whh[k * H3 + j]; wz = whh[k * H3 + H + j]; wn = whh[k * H3 + 2 * H + j];
      } else {
        wr = __ldg(Whh + (int64_t)j * H + k);
        wz = __ldg(Whh + (int64_t)(H + j) * H + k);
        wn = __ldg(Whh + (int64_t)(2 * H + j) * H + k);
      }
      const float4 v0 = *reinterpret_cast<const float4*>(hT + k * NSEQ + s0);
      const float4 v1 = *reinterpret_cast<const float4*>(hT + k * NSEQ + s0 + 4);
      const float hs[SPT] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int q = 0; q < SPT; ++q) {
        hr[q] = fmaf(wr, hs[q], hr[q]);
        hz[q] = fmaf(wz, hs[q], hz[q]);
        hn[q] = fmaf(wn, hs[q], hn[q]);
      }
    }
    __syncthreads();  // every read of xT/hT for step l is done; att is visible
#pragma unroll
    for (int q = 0; q < SPT; ++q) {
      const float r = sigm((gr[q] + bir) + (hr[q] + bhr));
      const float z = sigm((gz[q] + biz) + (hz[q] + bhz));
      const float n = tanhf((gn[q] + bin) + r * (hn[q] + bhn));
      float hn1;
      if (g.augru) {
        const float u = att[s0 + q] * (1.0f - z);
        hn1 = (1.0f - u) * h[q] + u * n;
      } else {
        hn1 = (1.0f - z) * n + z * h[q];
      }
      h[q] = hn1;
      hT[j * NSEQ + s0 + q] = hn1;
    }
    if (l + 1 < L) stash(pf);
    __syncthreads();
  }

#pragma unroll
  for (int q = 0; q < SPT; ++q) {
    const int64_t item = item0 + s0 + q;
    if (item < S) g.out[item * g.ld_out + g.col_off + (int64_t)t * H + j] = h[q];
  }
}

bool use_wsmem(const GruArgs& g) { return gru_smem(g.D, g.H, true) <= 200 * 1024; }

}  // namespace

void prepare_gru(const GruArgs& g) {
  const size_t s1 = gru_smem(g.D, g.H, true), s0 = gru_smem(g.D, g.H, false);
  cudaFuncSetAttribute(gru_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::min<size_t>(s1, 227 * 1024));
  cudaFuncSetAttribute(gru_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::min<size_t>(s0, 227 * 1024));
}

bool gru_supported(int D, int H) {
  return D % 4 == 0 && H >= 1 && H <= 1024 &&
         gru_nseq(H) * (D / 4) <= MAXPF * gru_threads(H) &&
         gru_smem(D, H, false) <= 200 * 1024;
}

void launch_gru(const QDesc* qd, const GruArgs& g, int64_t max_items, int sm_count,
                cudaStream_t s) {
  (void)sm_count;
  const int nseq = gru_nseq(g.H);
  const dim3 grid((unsigned)((max_items + nseq - 1) / nseq), g.T);
  const bool ws = use_wsmem(g);
  const size_t smem = gru_smem(g.D, g.H, ws);
  max_carveout(reinterpret_cast<const void*>(gru_kernel<true>));
  max_carveout(reinterpret_cast<const void*>(gru_kernel<false>));
  if (ws) gru_kernel<true><<<grid, gru_threads(g.H), smem, s>>>(qd, g);
  else gru_kernel<false><<<grid, gru_threads(g.H), smem, s>>>(qd, g);
}

}  // namespace rs
