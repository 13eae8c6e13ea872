// common.cuh — device-side shared types and helpers for the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>
#include <map>
#include <set>
#include <utility>

#include "../spec.h"

// Measured-slower alternatives (SLS variants 1/3/4, the whole-stack FC chain
// kernel, split-K, green-context partitions, stream-memop descriptors) are
// compiled only into an experiments build: make EXPERIMENTS=1.
#ifndef RS_EXPERIMENTS
#define RS_EXPERIMENTS 0
#endif

namespace rs {

// Device-resident query descriptor. Every kernel of the forward graph reads
// the item count (and the index pointer) from here, so ONE captured CUDA
// graph per scratch slot serves every query size up to max_query_size:
// the grid is sized for capacity and blocks past S exit at once.
struct QDesc {
  int64_t S;
  const int64_t* idx;  // [S, T, L] int64 (device)
  const float* dense;  // [S, dense_in] fp32 contiguous (device), or null
  float* out;          // final logits [S, out_w] (device) or null: slot buffer
  int64_t flags;       // kDescDenseBf16: `dense` holds bfloat16 values
  // embedding-stage work counters, zero in every descriptor the host writes
  // (so each query starts from 0): [0] next bag ticket, [1] warps retired
  unsigned int work[2];
};
constexpr int64_t kDescDenseBf16 = 1;

// Error bits accumulated by kernels and read back with the logits.
enum : int { kErrIndex = 1 };

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  // Table rows are touched once per query: stream them past L1.
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// L2 policy for data touched once per query (table rows): evict first, so
// the random row stream does not push weights, indices and partials out.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ float4 ldg_stream_hint(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ float ldg_stream1(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}

__device__ __forceinline__ float4 shfl_xor4(const float4& v, int off) {
  float4 r;
  r.x = __shfl_xor_sync(0xffffffffu, v.x, off);
  r.y = __shfl_xor_sync(0xffffffffu, v.y, off);
  r.z = __shfl_xor_sync(0xffffffffu, v.z, off);
  r.w = __shfl_xor_sync(0xffffffffu, v.w, off);
  return r;
}

__host__ __device__ __forceinline__ int64_t round_up(int64_t x, int64_t m) {
  return (x + m - 1) / m * m;
}

// Programmatic dependent launch (PDL). Every kernel of the forward graph is
// launched with programmatic stream serialisation: it lets its successor
// launch as soon as it starts (pdl_trigger), and blocks on its predecessor
// (pdl_wait: full completion + memory visibility) only right before it
// touches data the predecessor wrote. Both are no-ops without a programmatic
// dependency.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// What the graph being captured on this thread serves: 1 = a lane of the
// pipelined queue (rs_forward_many / rs_serve), 0 = single queries, -1 = no
// capture in progress. Kernels launched into a lane graph leave SM slots to
// the other lanes' kernels: no PDL edges, one resident wave
// of gather CTAs.
inline int& capture_lane() {
  thread_local int v = -1;
  return v;
}
// PDL edges are captured unless RS_PDL=0 (read at graph capture); without the
// variable, everywhere but in the queue's lanes: PDL shortens one query's
// kernel chain, but there the early-launched dependent CTAs sit on SM slots
// the other lanes' kernels would use.
inline bool pdl_enabled() {
  const char* v = getenv("RS_PDL");
  if (v) return atoi(v) != 0;
  return capture_lane() != 1;
}

// Node priorities (graphs instantiated with cudaGraphInstantiateFlagUseNodePriority):
// the latency-bound dense kernels (staging, FC layers, interaction) run at the
// device's greatest priority, the HBM-bound gathers at the default. Without
// it, the gathers of the other pipelined lanes refill every SM slot as it
// frees (3 gather CTAs fill an SM's registers) and the larger FC CTAs starve
// (tools/timeline.py). RS_PRIO=0 disables.
inline bool prio_enabled() {
  const char* v = getenv("RS_PRIO");
  return !v || atoi(v) != 0;
}
inline int high_priority() {
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  return greatest;
}

// Experiment knob (RS_CARVEOUT=1): every kernel asks for the maximum
// shared-memory carveout, so gather and tcgen05 CTAs never differ in their
// preferred L1/shared split. Measured off by default: the gathers lose L1
// capacity for in-flight loads (pipelined queue 34.2 -> 39.0 us/query, one
// launch 5.43 -> 4.99 TB/s at 323 items).
// Function attributes belong to the current device's context: a process that
// drives several GPUs (rs_serve over K replicas) sets them once PER DEVICE.
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
// The attribute is a per-function maximum: raised whenever a launch needs more
// than any earlier one on this device (kernels whose shared memory depends on
// the model shape, e.g. the interaction's (T+1) x D staging).
inline void smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  std::lock_guard<std::mutex> g(mu);
  int& cur = done[{current_device(), fn}];
  if (bytes > cur) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cur = bytes;
  }
}

// RS_CARVEOUT_FUNC=<p> (experiment): the carveout as a FUNCTION attribute of
// every kernel (p% of the unified L1/shared array; 1 = maximum shared). The
// product sets it per handle on the graph's kernel nodes instead (accel.cu,
// rs_accel::carveout_pct, RS_CARVEOUT).
inline void max_carveout(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  static const int pct = [] {
    const char* v = getenv("RS_CARVEOUT_FUNC");
    const int p = v ? atoi(v) : 0;
    return p == 1 ? (int)cudaSharedmemCarveoutMaxShared : p;
  }();
  if (pct <= 0) return;
  std::lock_guard<std::mutex> g(mu);
  if (done.insert({current_device(), fn}).second)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

#if defined(__CUDACC__)
// Launch with the programmatic-stream-serialisation attribute (captured into
// a CUDA graph as a programmatic dependency edge).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  max_carveout(reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
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
#endif

}  // namespace rs
