// spec.h — the frozen numeric specification of the forward pass inputs and
// parameters. The reference defines no weights, no init and
// no inputs, so this file IS the contract shared by the
// product (host C++ and CUDA) and restated independently by oracle/forward.c.
//
// Every parameter element is a pure function of (seed, tensor id, element
// index) through one splitmix64 call, so a table of 10M rows can be filled on
// the device at HBM speed and the oracle can regenerate exactly the rows a
// query touches without materialising the table.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD static inline
#endif

namespace rs {

RS_HD uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Per-tensor stream key.
RS_HD uint64_t stream_key(uint64_t seed, uint64_t id) {
  return splitmix64(seed ^ (id * 0xD1B54A32D192ED03ull));
}

// 24-bit signed lattice in [-1, 1): exact in fp32, one multiply to scale.
RS_HD float unit(uint64_t h) {
  return (float)((int32_t)(h >> 40) - 8388608) * (1.0f / 8388608.0f);
}

RS_HD float param(uint64_t key, uint64_t elem, float bound) {
  return unit(splitmix64(key + elem)) * bound;
}

// Tensor ids.
RS_HD uint64_t id_table(int64_t t) { return 0x1000ull + (uint64_t)t; }
RS_HD uint64_t id_dense_w(int64_t l) { return 0x2000ull + 2ull * (uint64_t)l; }
RS_HD uint64_t id_dense_b(int64_t l) { return 0x2001ull + 2ull * (uint64_t)l; }
RS_HD uint64_t id_pred_w(int64_t s, int64_t l) {
  return 0x3000ull + 64ull * (uint64_t)s + 2ull * (uint64_t)l;
}
RS_HD uint64_t id_pred_b(int64_t s, int64_t l) { return id_pred_w(s, l) + 1ull; }
RS_HD uint64_t id_att_w(int64_t t) { return 0x4000ull + (uint64_t)t; }
// GRU per table: 0 W_ih[3H,D], 1 W_hh[3H,H], 2 b_ih[3H], 3 b_hh[3H], 4 W_a[D,D]
RS_HD uint64_t id_gru(int64_t t, int k) { return 0x5000ull + 8ull * (uint64_t)t + (uint64_t)k; }
RS_HD uint64_t id_query_dense(uint64_t q) { return 0x70000000000ull + q; }
RS_HD uint64_t id_query_idx(uint64_t q) { return 0x80000000000ull + q; }

constexpr float kTableScale = 0.05f;

// Uniform index in [0, rows) from a 64-bit hash (multiply-shift).
RS_HD int64_t index_from_hash(uint64_t h, int64_t rows) {
#if defined(__CUDA_ARCH__)
  return (int64_t)__umul64hi(h, (uint64_t)rows);
#else
  return (int64_t)(((unsigned __int128)h * (unsigned __int128)(uint64_t)rows) >> 64);
#endif
}

}  // namespace rs
