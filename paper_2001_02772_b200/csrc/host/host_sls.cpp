// host_sls.cpp — SparseLengthsSum on the host cores for the CPU side of the
// split: the sub-queries routed to CPU cores by the split/offload
// decision (proj/src/sim.cpp:173-191) gather and pool their embedding bags
// here. The reference only costs this work (cpu_service_time,
// proj/src/platform.cpp:71-103, fed by work()'s EmbeddingLookup/Sum bytes,
// proj/src/model_zoo.cpp:177-245); this is a real implementation of it.
//
// Order: the CANONICAL order of the B200 SLS kernel (oracle/oracle.h,
// or_sls_canonical): a bag's rows go round-robin into R partial sums, combined
// by a pairwise tree, R = 32 / min(32, D/4) for power-of-two D in [8,256], else
// 1. Element c of a bag only ever adds element c of rows, so vectorising across
// c (AVX-512 / AVX2 via target clones, adds only, no contraction) keeps the
// result bit-identical to the GPU path — a query split between host and device
// pools identically on both sides.
//
// Work split: bags are dealt to `threads` std::threads in contiguous ranges;
// the next rows of a bag are prefetched a few lookups ahead (the gather is
// DRAM-latency bound on the host exactly as on the device).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace rs {
namespace {


int canonical_r(int D) {
  if (D == 8 || D == 16 || D == 32 || D == 64 || D == 128 || D == 256) {
    const int lpr = D / 4 < 32 ? D / 4 : 32;
    return 32 / lpr;
  }
  return 1;
}

// Pools bags [b0, b1). Returns the first bad (bag, lookup) as bag*L+l, or -1.
__attribute__((target_clones("avx512f", "avx2", "default")))
int64_t pool_range(const float* __restrict__ tables, int64_t rows, int T, int L, int D, int R,
                   const int64_t* __restrict__ idx, float* __restrict__ pooled, int64_t b0,
                   int64_t b1, int pf) {
  std::vector<float> part_buf((size_t)R * D);
  float* __restrict__ part = part_buf.data();
  for (int64_t bag = b0; bag < b1; ++bag) {
    const int64_t t = bag % T;
    const float* __restrict__ tab = tables + t * rows * (int64_t)D;
    const int64_t* __restrict__ bi = idx + bag * L;
    std::memset(part, 0, sizeof(float) * (size_t)R * D);
    for (int l = 0; l < L; ++l) {
      if (l + pf < L) {
        const int64_t rp = bi[l + pf];
        if ((uint64_t)rp < (uint64_t)rows)
          for (int o = 0; o < D; o += 16) __builtin_prefetch(tab + rp * D + o);
      }
      const int64_t r = bi[l];
      if ((uint64_t)r >= (uint64_t)rows) return bag * L + l;
      const float* __restrict__ e = tab + r * D;
      float* __restrict__ p = part + (size_t)(l % R) * D;
      for (int c = 0; c < D; ++c) p[c] = p[c] + e[c];
    }
    for (int half = R / 2; half >= 1; half /= 2)
      for (int g = 0; g < half; ++g) {
        float* __restrict__ a = part + (size_t)g * D;
        const float* __restrict__ b = part + (size_t)(g + half) * D;
        for (int c = 0; c < D; ++c) a[c] = a[c] + b[c];
      }
    std::memcpy(pooled + bag * D, part, sizeof(float) * (size_t)D);
  }
  return -1;
}

}  // namespace

int64_t host_pool_bags(const float* tables, int64_t rows, int T, int L, int D,
                       const int64_t* idx, float* pooled, int64_t b0, int64_t b1) {
  return pool_range(tables, rows, T, L, D, canonical_r(D), idx, pooled, b0, b1, 8);
}

}  // namespace rs

extern "C" int rs_host_sls(const float* tables, int64_t rows_per_table, int32_t num_tables,
                           int32_t lookups, int32_t dim, int64_t query_size,
                           const int64_t* indices, float* pooled, int32_t threads) {
  using namespace rs;
  return guarded([&] {
  if (query_size < 0 || rows_per_table < 1 || num_tables < 1 || lookups < 0 || dim < 1 ||
      dim > 4096)
    raise(RS_E_INVALID, "rs_host_sls: bad shape");
  const int64_t bags = query_size * num_tables;
  if (bags == 0) return;
  if (!tables || !pooled || (lookups > 0 && !indices))
    raise(RS_E_INVALID, "rs_host_sls: null buffer");
  const int R = canonical_r(dim);
  static const int pf = [] {  // lookups prefetched ahead (RS_HOST_PREFETCH)
    const char* v = getenv("RS_HOST_PREFETCH");
    return v ? std::max(1, atoi(v)) : 8;
  }();
  int nt = threads > 0 ? threads : host_cores();
  nt = (int)std::min<int64_t>(nt, bags);
  std::vector<int64_t> bad(nt, -1);
  auto run = [&](int i) {
    const int64_t b0 = bags * i / nt, b1 = bags * (i + 1) / nt;
    bad[i] = pool_range(tables, rows_per_table, num_tables, lookups, dim, R, indices, pooled,
                        b0, b1, pf);
  };
  if (nt == 1) {
    run(0);
  } else {
    std::vector<std::thread> pool;
    pool.reserve(nt);
    for (int i = 0; i < nt; ++i) pool.emplace_back(run, i);
    for (auto& th : pool) th.join();
  }
  for (int i = 0; i < nt; ++i)
    if (bad[i] >= 0) {
      const int64_t bag = bad[i] / std::max(lookups, 1), l = bad[i] % std::max(lookups, 1);
      raise(RS_E_INDEX, "rs_host_sls: index " + std::to_string(indices[bad[i]]) +
                            " outside [0, " + std::to_string(rows_per_table) + ") at item " +
                            std::to_string(bag / num_tables) + ", table " +
                            std::to_string(bag % num_tables) + ", lookup " + std::to_string(l));
    }
  });
}
