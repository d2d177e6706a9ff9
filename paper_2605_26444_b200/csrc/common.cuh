// Shared device helpers of the NanoSpec CUDA path (sm_100a).  Product code:
// shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace nanospec {

constexpr int kWarp = 32;
constexpr int32_t kFirstSentinel = 0x7f7f7f7f;  // byte-memset value 0x7f: "no occurrence yet"

// Per-sequence scalars of the GPU-resident state (16 bytes).
struct Meta {
  long long total;   // |S| (R1) or pushes (R2)
  int32_t n_active;  // |I|
  int32_t err;       // bit 0: an out-of-range id was dropped
};

// Pointers + geometry of a state workspace (type-major arrays, seq stride =
// the per-sequence length of each array).
struct StateView {
  int32_t vocab, v_local, w_max, words, rank, n_shards, rule, batch;
  Meta* meta;
  uint32_t* bitmap;   // [batch][words]
  int32_t* ids;       // [batch][w_max]
  int32_t* ring;      // [batch][w_max]
  int32_t* cnt;       // [batch][v_local]   (R1 only)
  int32_t* pos;       // [batch][v_local]   (R1 only) slot of each active local id in ids[]
  int32_t* first;     // [batch][vocab]
};

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix, writes the block total to *total.  `sh` needs blockDim/32 + 1 ints.
__device__ __forceinline__ int block_exclusive_scan(int v, int* sh, int* total) {
  const int lane = lane_id(), wid = warp_id(), nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  int base = wid > 0 ? sh[wid - 1] : 0;
  *total = sh[nw - 1];
  __syncthreads();  // sh may be reused right after
  return base + x - v;
}

__device__ __forceinline__ float block_sum(float v, float* sh) {
  const int lane = lane_id(), wid = warp_id(), nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  float s = 0.f;
  if (wid == 0) {
    s = lane < nw ? sh[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sh[0] = s;
  }
  __syncthreads();
  s = sh[0];
  __syncthreads();
  return s;
}

// Order-preserving map float -> uint32 (larger float -> larger key); -0 == +0.
__device__ __forceinline__ uint32_t float_key(float v) {
  if (v == 0.f) v = 0.f;
  uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Optional phase trace (debug): when `trace` is non-null, CTA b writes the
// %globaltimer (ns) of phase e to trace[b * kTraceSlots + e].
constexpr int kTraceSlots = 16;
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_mark(unsigned long long* trace, int e) {
  if (trace) trace[(long long)blockIdx.x * kTraceSlots + e] = globaltimer();
}

}  // namespace nanospec
