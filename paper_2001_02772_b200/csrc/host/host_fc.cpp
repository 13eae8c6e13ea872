// host_fc.cpp — fully connected layer on the host cores for the CPU side of
// the split (the GEMM half; host_sls.cpp is the gather half).
// The reference costs this work (DenseFC/PredictFC flops of work(),
// proj/src/model_zoo.cpp:177-245, priced by cpu_service_time,
// proj/src/platform.cpp:71-103); this executes it.
//
// y[m][n] = act(b[n] + sum_k x[m][k] * W[n][k]) with W in the device layout
// [out][in]. W is transposed once per call into [in][out] so
// the inner loop runs across n (vectorised by the AVX-512/AVX2 clones without
// reassociating a reduction); a 4 x 32 tile of y stays in vector registers
// across the K loop, so each W^T load feeds four rows of x. Rows of
// x are dealt to std::threads in contiguous blocks. fp32 with FMA
// contraction: parity is the floating-point tolerance rule of DESIGN.md §4,
// not bit identity.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace rs {
namespace {

constexpr int kRows = 4;  // rows of x per pass over W^T

// The register tile is 4 rows x 2 vectors of y held across the K loop: 8
// accumulators + 2 W^T vectors. Its width follows the vector ISA so the tile
// never spills: 2 x 16 floats with AVX-512 (32 zmm), 2 x 8 with AVX2 (16 ymm),
// 2 x 4 otherwise.
template <int W>
__attribute__((always_inline)) inline void fc_rows_body(
    const float* __restrict__ x, int64_t m0, int64_t m1, int K, int N,
    const float* __restrict__ wt, const float* __restrict__ b, int relu, float* __restrict__ y) {
  typedef float vec __attribute__((vector_size(W * 4)));
  constexpr int TW = 2 * W;  // tile columns
  const int nt = N / TW * TW;
  for (int64_t m = m0; m < m1; m += kRows) {
    const int nr = (int)std::min<int64_t>(kRows, m1 - m);
    if (nr == kRows && nt > 0) {
      for (int n0 = 0; n0 < nt; n0 += TW) {
        vec acc[kRows][2];
        for (int r = 0; r < kRows; ++r) {
          acc[r][0] = vec{};
          acc[r][1] = vec{};
          if (b) {
            std::memcpy(&acc[r][0], b + n0, sizeof(vec));
            std::memcpy(&acc[r][1], b + n0 + W, sizeof(vec));
          }
        }
        for (int k = 0; k < K; ++k) {
          vec w0, w1;
          std::memcpy(&w0, wt + (int64_t)k * N + n0, sizeof(vec));
          std::memcpy(&w1, wt + (int64_t)k * N + n0 + W, sizeof(vec));
          for (int r = 0; r < kRows; ++r) {
            const float av = x[(m + r) * K + k];
            acc[r][0] += av * w0;
            acc[r][1] += av * w1;
          }
        }
        for (int r = 0; r < kRows; ++r) {
          if (relu) {
            acc[r][0] = acc[r][0] > 0.0f ? acc[r][0] : vec{};
            acc[r][1] = acc[r][1] > 0.0f ? acc[r][1] : vec{};
          }
          std::memcpy(y + (m + r) * N + n0, &acc[r][0], sizeof(vec));
          std::memcpy(y + (m + r) * N + n0 + W, &acc[r][1], sizeof(vec));
        }
      }
      if (nt == N) continue;
    }
    const int nb = (nr == kRows) ? nt : 0;  // columns already written
    float* __restrict__ yr[kRows];
    for (int r = 0; r < kRows; ++r) yr[r] = y + (m + std::min(r, nr - 1)) * N;
    for (int r = 0; r < nr; ++r)
      for (int n = nb; n < N; ++n) yr[r][n] = b ? b[n] : 0.0f;
    for (int k = 0; k < K; ++k) {
      const float* __restrict__ w = wt + (int64_t)k * N;
      for (int r = 0; r < nr; ++r) {
        const float av = x[(m + r) * K + k];
        float* __restrict__ yy = yr[r];
        for (int n = nb; n < N; ++n) yy[n] += av * w[n];
      }
    }
    if (relu)
      for (int r = 0; r < nr; ++r)
        for (int n = nb; n < N; ++n) yr[r][n] = yr[r][n] > 0.0f ? yr[r][n] : 0.0f;
  }
}

__attribute__((target("avx512f"))) void fc_rows_avx512(const float* x, int64_t m0, int64_t m1,
                                                       int K, int N, const float* wt,
                                                       const float* b, int relu, float* y) {
  fc_rows_body<16>(x, m0, m1, K, N, wt, b, relu, y);
}
__attribute__((target("avx2,fma"))) void fc_rows_avx2(const float* x, int64_t m0, int64_t m1,
                                                      int K, int N, const float* wt,
                                                      const float* b, int relu, float* y) {
  fc_rows_body<8>(x, m0, m1, K, N, wt, b, relu, y);
}
void fc_rows_sse(const float* x, int64_t m0, int64_t m1, int K, int N, const float* wt,
                 const float* b, int relu, float* y) {
  fc_rows_body<4>(x, m0, m1, K, N, wt, b, relu, y);
}

void fc_rows(const float* x, int64_t m0, int64_t m1, int K, int N, const float* wt,
             const float* b, int relu, float* y) {
  static const int isa = [] {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512f")) return 2;
    if (__builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma")) return 1;
    return 0;
  }();
  if (isa == 2) fc_rows_avx512(x, m0, m1, K, N, wt, b, relu, y);
  else if (isa == 1) fc_rows_avx2(x, m0, m1, K, N, wt, b, relu, y);
  else fc_rows_sse(x, m0, m1, K, N, wt, b, relu, y);
}

}  // namespace

void host_fc_rows(const float* x, int64_t m0, int64_t m1, int K, int N, const float* wt,
                  const float* b, int relu, float* y) {
  fc_rows(x, m0, m1, K, N, wt, b, relu, y);
}

}  // namespace rs

extern "C" int rs_host_fc(const float* x, int64_t rows, int32_t in_dim, const float* weight,
                          int64_t ldw, const float* bias, int32_t out_dim, int32_t relu,
                          float* y, int32_t threads) {
  using namespace rs;
  return guarded([&] {
    if (rows < 0 || in_dim < 0 || out_dim < 1) raise(RS_E_INVALID, "rs_host_fc: bad shape");
    if (ldw == 0) ldw = in_dim;
    if (ldw < in_dim) raise(RS_E_INVALID, "rs_host_fc: ldw < in_dim");
    if (rows == 0) return;
    if (!y || (in_dim > 0 && (!x || !weight))) raise(RS_E_INVALID, "rs_host_fc: null buffer");
    // W^T [in][out] (row stride ldw of the caller's [out][ldw] weight: the
    // device layout pads rows to round4(in))
    std::vector<float> wt((size_t)in_dim * out_dim);
    for (int n = 0; n < out_dim; ++n)
      for (int k = 0; k < in_dim; ++k) wt[(size_t)k * out_dim + n] = weight[(size_t)n * ldw + k];
    int nt = threads > 0 ? threads : host_cores();
    nt = (int)std::min<int64_t>(nt, (rows + kRows - 1) / kRows);
    auto run = [&](int i) {
      const int64_t blocks = (rows + kRows - 1) / kRows;
      const int64_t m0 = std::min(rows, blocks * i / nt * kRows);
      const int64_t m1 = std::min(rows, blocks * (i + 1) / nt * kRows);
      fc_rows(x, m0, m1, in_dim, out_dim, wt.data(), bias, relu, y);
    };
    if (nt == 1) {
      run(0);
    } else {
      std::vector<std::thread> pool;
      pool.reserve(nt);
      for (int i = 0; i < nt; ++i) pool.emplace_back(run, i);
      for (auto& th : pool) th.join();
    }
  });
}
