// kernels.hpp — host-side launchers for the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rs {

struct QDesc;

// ---- embedding.cu ----
bool sls_vector_path(int64_t D);
// hot/hot_rows: optional exact copy of rows [0, hot_rows) of every table,
// [T][hot_rows][D], kept in the L2 persisting set-aside (rs_init_desc
// l2_persist_mb); the default SLS kernel reads those rows from it.
void launch_sls_sum(const QDesc* qd, const float* tables, int64_t rows, int T, int L, int D,
                    float* out, int64_t ld_out, int* err, int64_t max_items, int sm_count,
                    cudaStream_t s, const float* hot = nullptr, int64_t hot_rows = 0);
void launch_gather_concat(const QDesc* qd, const float* tables, int64_t rows, int T, int L,
                          int D, float* out, int64_t ld_out, int64_t col_off, int* err,
                          int64_t max_items, int sm_count, cudaStream_t s);
bool din_supported(int64_t D);
void launch_din_pool(const QDesc* qd, const float* tables, int64_t rows, int T, int L, int D,
                     const float* att_w, float* out, int64_t ld_out, int64_t col_off, int* err,
                     int64_t max_items, int sm_count, cudaStream_t s);
void launch_diag_empty(int n, int ctas, cudaStream_t s);
void launch_widen_idx(const int32_t* src, int64_t* dst, int64_t n, int sm_count, cudaStream_t s);
// Device-resident inputs of m merged queries gathered back to back in one
// launch (RS_OPT_MERGE_QUERIES): per query k, dense rows -> dense_dst + off_k
// * dense_in and indices -> idx_dst + off_k * TL (int32 sources widened).
constexpr int kMaxGroup = 64;
struct GroupGather {
  const float* dense[kMaxGroup];
  const void* idx[kMaxGroup];
  int64_t size[kMaxGroup];
  int64_t off[kMaxGroup];
  int m;
  int idx32;
};
void launch_group_gather(const GroupGather& g, int64_t dense_in, int64_t TL, float* dense_dst,
                         int64_t* idx_dst, int sm_count, cudaStream_t s);
void launch_stage_dense(const QDesc* qd, int64_t dense_in, float* dst, int64_t ld_dst,
                        int64_t max_items, int sm_count, cudaStream_t s);
// fp32 rows -> bf16 rows (RS_FC_BF16 graphs): dst[r][c] = bf16(src[r][c]),
// r < QDesc::S, c < cols
void launch_to_bf16(const QDesc* qd, const float* src, int64_t lds, void* dst, int64_t ldd,
                    int64_t cols, int64_t max_items, int sm_count, cudaStream_t s);
// threads: 256 (default) or 64 — 2-warp CTAs that fit beside three gather
// CTAs on an SM (the handle picks 64 for strongly gather-bound models)
void launch_interaction(const QDesc* qd, const float* pooled, int64_t ld_pooled, int T, int D,
                        float* X, int64_t ld_x, int64_t sum_off, int64_t dot_off, int has_dense,
                        int64_t max_items, int sm_count, cudaStream_t s, bool tc = false,
                        int threads = 256);
size_t interaction_smem(int T, int D);
void launch_init_tables(float* tables, int64_t T, int64_t rows, int64_t D, uint64_t seed,
                        int sm_count, cudaStream_t s);

// ---- fc_ffma.cu ----
// Batched (over predict stacks, grid z) fp32 FC layer:
//   C[z][m][n] = act( sum_k A[z][m][k] * W[z][n][k] + bias[z][n] ),  m < S (device)
struct FcArgs {
  const float* A; int64_t lda; int64_t sAz;
  const float* W; int64_t ldw; int64_t sWz;
  const float* bias; int64_t sbz;
  float* C; int64_t ldc; int64_t sCz;
  int N; int K; int relu; int batch;
  int c_desc;  // 1: write C into QDesc::out when that is non-null (final layer)
  // Optional narrow next layer fused into the tcgen05 epilogue (the CTA owns
  // whole rows of C when the layer is a single N tile):
  //   C2[z][m][o] = act2( sum_n C[z][m][n] * W2[z][o][n] + b2[z][o] ), o < N2 <= 4
  const float* W2; int64_t ldw2; int64_t sW2z;
  const float* b2; int64_t sb2z;
  float* C2; int64_t ldc2; int64_t sC2z;
  int N2; int relu2; int c2_desc;
  int skip_c;          // 1: C itself is not needed (only C2)
  int single_n_tile;   // planning hint: prefer one N tile (BN = 128) when N <= 128
  int splits; float* ws; int* cnt;  // split-K (set by launch_fc_tc from the plan)
  // RS_FC_BF16: A and W hold bfloat16 (row strides in elements); c16: C is
  // written as bfloat16 (the next bf16 layer's A). tcgen05 only.
  int ab16; int c16;
  // Dead-data discard (discard.global.L2, no DRAM write-back): discard_a = this
  // CTA is the only reader of its A rows (one N tile, batch 1), drop them after
  // the main loop; dz = another dead buffer whose rows [m0, m0+128) this CTA
  // drops too (row stride dz_ld bytes) — e.g. the stack input two layers back.
  int discard_a; const void* dz; int64_t dz_ld;
  int smem_cap_kb;  // planning: tcgen05 tile shared-memory budget (0 = none)
  int pair_ok;      // planning: CTA-pair tiles (fc_tc2_kernel) for N >= 256: 1 = the wide
                    // graph (6-deep ring), 2 = every graph of the handle (4-deep)
  int pair_capped;  // planning: 3-deep CTA-pair tiles within smem_cap_kb for N >= 256
};
constexpr int kFuseMaxN2 = 4;
void launch_fc_ffma(const QDesc* qd, const FcArgs& a, int64_t max_items, cudaStream_t s);

// ---- fc_tcgen05.cu ----
// Same contract on the 5th-gen tensor cores (kind::tf32, fp32 accumulate in
// TMEM, operands staged by TMA). Tensor maps are built once per buffer.
struct TcPlan {
  CUtensorMap map_a;   // A: [batch][M_cap][K] fp32, box 128 x 32
  CUtensorMap map_w;   // W: [batch][N][K] fp32, box BN x 32
  int block_n;         // 64 / 128 / 256
  int pair_stages;     // cfg 5 (CTA pairs): k-slab ring depth (3, 4 or 6)
  int cfg;             // tile/pipeline configuration (fc_tcgen05.cu)
  int m_tiles, n_tiles;
  int splits;          // split-K factor (1 = none)
  float* ws;           // split-K partial tiles [batch*splits][m_tiles][n_tiles][128*BN]
  int* cnt;            // split-K arrival counters [batch][m_tiles][n_tiles] (self-resetting)
  int ab16;            // bf16 operands (kind::f16)
};
// Device scratch the plans of one graph carve split-K workspaces from.
struct SplitKPool {
  float* ws = nullptr; size_t ws_cap = 0, ws_used = 0;    // floats
  int* cnt = nullptr; size_t cnt_cap = 0, cnt_used = 0;   // ints (zeroed)
};
bool tc_available();
bool make_row_gather_map(CUtensorMap* map, const float* base, int64_t total_rows, int D);
bool tc_plan(TcPlan* p, const FcArgs& a, int64_t m_cap, int64_t a_rows_per_batch,
             SplitKPool* pool = nullptr);
void launch_fc_tc(const QDesc* qd, const TcPlan& p, const FcArgs& a, cudaStream_t s);

// A whole FC stack in ONE kernel (fc_tcgen05.cu, fc_chain_kernel): per
// 128-row tile the activations stay in shared memory between layers (as the
// next layer's swizzled K-major A operand), weights stream by TMA, each
// layer accumulates in TMEM. Layers with N <= 256 and hidden widths <= 256;
// an optional final layer of <= 4 outputs runs in the last epilogue.
constexpr int kChainMaxLayers = 4;
struct TcChainPlan {
  CUtensorMap map_a;                   // layer-0 input [rows][K0], box 32 x 128
  CUtensorMap map_w[kChainMaxLayers];  // W_l [N_l][K_l], box 32 x NP_l
  const float* bias[kChainMaxLayers];
  int n[kChainMaxLayers];              // N_l
  int np[kChainMaxLayers];             // N_l rounded up to 16 (UMMA N)
  int k[kChainMaxLayers];              // K_l
  int relu[kChainMaxLayers];
  int layers;
  int stream_a;                        // layer-0 input streamed per k-block (K0 > 256)
  int slot, slot_b, stages;            // k-block ring: slot bytes, W offset in a slot, depth
  float* C; int64_t ldc; int c_desc;   // output of the last layer
  const float* W2; int64_t ldw2; const float* b2; int N2; int relu2;  // fused narrow layer
  int m_tiles;
};
// Plans a chain for layers [0, L) of `layers` (FcArgs of each, batch 1);
// false if some layer does not fit (the caller runs them one by one).
bool tc_chain_plan(TcChainPlan* p, const FcArgs* layers, int L, int64_t m_cap,
                   int64_t a_rows);
void launch_fc_chain(const QDesc* qd, const TcChainPlan& p, cudaStream_t s);

// ---- gru.cu ----
struct GruArgs {
  const float* tables; int64_t rows; int T; int L; int D; int H;
  const float* w_ih;   // [T][3H][D]
  const float* w_hh;   // [T][3H][H]
  const float* b_ih;   // [T][3H]
  const float* b_hh;   // [T][3H]
  const float* w_att;  // [T][D][D] (AUGRU only)
  int augru;
  float* out; int64_t ld_out; int64_t col_off;
  int* err;
};
bool gru_supported(int D, int H);
// gru_tcgen05.cu: tensor-core recurrence (D, H in {32, 64}); false if unsupported
bool gru_tc_supported(int D, int H);
bool launch_gru_tc(const QDesc* qd, const GruArgs& g, int64_t max_items, cudaStream_t s);
void prepare_gru(const GruArgs& g);
void launch_gru(const QDesc* qd, const GruArgs& g, int64_t max_items, int sm_count,
                cudaStream_t s);

}  // namespace rs
