// a3+a4+a5 in ONE kernel on the 5th-generation tensor cores (tcgen05.mma,
// accumulators in TMEM):
//
//   z'[b][i][j] = sum_c W[row(ids_b[j])][c] * H[b][i][c]     (Eq. 2 on I)
//   then per (b, i) the top-k of z' by (value desc, id asc) + lse
//
// Gather.  The paper repacks the active rows into a dense buffer on a copy
// stream before a dense GEMM.  Here the gather is fused into the
// contraction's load stage: each 128-row tile of active rows is pulled
// straight from W_head with 16-byte cp.async into 128B-swizzled shared memory
// (the UMMA K-major SW128 layout), so weight bytes cross HBM exactly once.
//
// Contraction.  UMMA M = 128 active rows (A), N = NT >= n nodes (B, zero
// padded), K = 64 per pipeline stage; D in TMEM (NT fp32 columns).  T =
// sum_b ceil(n_active_b / 128) tiles are read from device memory (no host
// sync); every tile is split along K into S = max(1, floor(#SMs / T)) uniform
// chunks so that ~all SMs stream.  Each (tile, chunk) unit writes its fp32
// partial tile to L2-resident scratch.
//
// Top-k, two levels spread over all CTAs.  Level 1: as soon as the S partials
// of a tile are written (per-tile arrival counter; the launch is cooperative so
// all CTAs are co-resident and the spin is safe), the tile's S CTAs split its
// (tile, node) pairs; one warp per pair sums the S partials of the 128 rows in
// split order (fixed order -> equal rows give bit-equal logits) and keeps the
// pair's exact top-k (k arg-max rounds over (value desc, id asc) packed into
// 64-bit keys) plus (max, sum exp) for the lse.  Level 2, after one grid
// barrier: one CTA per (sequence, node) merges the ceil(|I|/128) * k level-1
// candidates the same way and combines the lse partials.
//
// Warp roles (544 threads): warps 0-15 load (cp.async) and drain TMEM (warp w
// reads TMEM lanes 32*(w%4).. and a quarter of the columns); warp 16 allocates
// TMEM and one lane issues the MMAs.  All 17 warps run the top-k phase (enough
// warps per scheduler to hide shared-memory and shuffle latencies).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kBM = 128;          // active rows per tile (UMMA M)
constexpr int kBK = 64;           // K per stage (bf16 -> 128 bytes)
constexpr int kLoadWarps = 16;    // loaders / epilogue / top-k
constexpr int kLoaders = kLoadWarps * 32;
constexpr int kThreads = kLoaders + 32;   // + one MMA-issue warp
constexpr int kWarps = kThreads / 32;
constexpr int kSmemBudget = 192 * 1024;
constexpr int kMaxSMs = 256;
constexpr int kCandCap = 1024;    // candidates kept for the exact ranking
constexpr int kMaxK = 32;

struct TcArgs {
  HeadProblem p;
  float* part;                 // [units][NT][128] fp32 partial tiles (split-K)
  float* zl;                   // [batch][n][max_ids] reduced logits (the debug output when requested)
  unsigned* counters;          // [0] grid arrive, [1] grid done, [2 + tile] tile arrivals (zero between launches)
  float* topk_logit;           // [batch][n][k]
  int32_t* topk_id;
  float* lse;                  // [batch][n] or null
  int k;
  int max_tiles;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled UMMA shared-memory descriptor (SM100): start>>4
// [0,14), LBO>>4 [16,30) (unused for SW128 K-major: 1), SBO>>4 [32,46) = 1024 B
// between 8-row groups, version 1 at [46,48), layout SWIZZLE_128B (2) at [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// Instruction descriptor, kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16
// [10,13)=1, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// ------------------------------------------------------------------ work split
__device__ __forceinline__ int clamp_nact(const HeadProblem& p, int b) {
  int m = p.nact_base[(long long)b * p.nact_stride];
  return m < 0 ? 0 : (m > p.max_ids ? p.max_ids : m);
}
__device__ __forceinline__ int batch_m0(const HeadProblem& p) { return p.batch > 0 ? clamp_nact(p, 0) : 0; }



template <int NT>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr int kBBytes = NT * kBK * 2;   // NT * 128 B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = NT < 32 ? 32 : NT;
  static constexpr int kPipeArea = kStages * kStageBytes;
  static constexpr int kTopkArea = 2 * kCandCap * 4;  // top-k phase staging
  static constexpr int kStageArea = kPipeArea > kTopkArea ? kPipeArea : kTopkArea;
  static constexpr int kSmemBytes = kStageArea + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(2 * kStages + 3 <= 30, "barrier area");
  static constexpr int kHChunks = NT * 8;                 // 16-B chunks of one H stage
  static constexpr int kColGroups = NT / 16 < 4 ? NT / 16 : 4;  // epilogue column groups
};

struct TopkSmem {
  float wmax[kWarps];     // per-warp max, sum exp(v - max), threshold candidate
  float wsum[kWarps];
  float wthr[kWarps];
  float T;                // candidate threshold of the chunk
  int ncand;
  int nbest;
  float best_v[kMaxK];
  int32_t best_g[kMaxK];
};

__device__ __forceinline__ bool ranks_before(float va, int32_t ga, float vb, int32_t gb) {
  const uint32_t ka = float_key(va), kb = float_key(vb);
  return ka > kb || (ka == kb && ga < gb);
}

// k-th largest (k <= 32) of one float per lane, by counting (ties by lane).
__device__ __forceinline__ float warp_kth_largest(float x, int k) {
  const int lane = threadIdx.x & 31;
  int rank = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float o = __shfl_sync(0xffffffffu, x, j);
    rank += (o > x || (o == x && j < lane)) ? 1 : 0;
  }
  const unsigned sel = __ballot_sync(0xffffffffu, rank == k - 1);
  return __shfl_sync(0xffffffffu, x, __ffs(sel) - 1);
}

// Top-k + lse of one (sequence, node), the whole CTA; every phase runs on all
// warps in parallel (a single warp executes ~6 cycles per instruction here):
//  1. each thread cp.async's its rows' S split partials and ids (<= 2 float4
//     groups per chunk) into its own shared-memory slots -- all in flight at
//     once, no registers held -- then sums them in split order (fixed order:
//     equal rows give bit-equal logits) and keeps (max, sum exp) online;
//  2. per-warp (max, sum exp) and, for k > 16, the k-th largest lane maximum;
//  3. warp 0 combines the 17 warp summaries: lse partial and a threshold T that
//     at least k values reach (k <= 16: the k-th largest warp maximum; else the
//     largest per-warp k-th lane maximum);
//  4. values >= T (plus the running best) are compacted into shared memory and
//     ranked by counting (value desc, id asc).
template <int NT>
__device__ void topk_node(const TcArgs& a, int seq, int node, int m, uint8_t* smem, TopkSmem& sh) {
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = a.k;
  const int32_t* ids = p.ids_base + (long long)seq * p.ids_stride;
  const long long ob = ((long long)seq * p.n + node) * k;
  float* cv = reinterpret_cast<float*>(smem);
  int32_t* cg = reinterpret_cast<int32_t*>(cv + kCandCap);
  constexpr int kChunk = 2 * kThreads * 4;  // rows per chunk
  if (tid == 0) sh.nbest = 0;
  float run_max = -INFINITY, run_sum = 0.f;  // online lse over chunks (kept by warp 0 lane 0)
  for (int c0 = 0; c0 < m; c0 += kChunk) {
    const int mc = min(kChunk, m - c0);
    // ---- 1. gather the reduced logits and ids (<= 2 float4 groups per thread, all in flight)
    float v[8];
    int32_t g[8];
    float tm = -INFINITY;
    {
      const float* zrow = a.zl + ((long long)seq * p.n + node) * p.max_ids;
      float4 x[2];
      int4 gi[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = 4 * (tid + h * kThreads);
        const int j = c0 + jj;
        x[h] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        gi[h] = make_int4(0, 0, 0, 0);
        if (jj < mc) {
          if (((((uintptr_t)(zrow + j)) | ((uintptr_t)(ids + j))) & 15) == 0 && j + 3 < m) {
            x[h] = __ldcg(reinterpret_cast<const float4*>(zrow + j));
            gi[h] = __ldcg(reinterpret_cast<const int4*>(ids + j));
          } else {
            x[h].x = __ldcg(zrow + j);
            gi[h].x = __ldg(ids + j);
            if (j + 1 < m) { x[h].y = __ldcg(zrow + j + 1); gi[h].y = __ldg(ids + j + 1); }
            if (j + 2 < m) { x[h].z = __ldcg(zrow + j + 2); gi[h].z = __ldg(ids + j + 2); }
            if (j + 3 < m) { x[h].w = __ldcg(zrow + j + 3); gi[h].w = __ldg(ids + j + 3); }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = 4 * (tid + h * kThreads);
        const float vv[4] = {x[h].x, x[h].y, x[h].z, x[h].w};
        const int32_t gg[4] = {gi[h].x, gi[h].y, gi[h].z, gi[h].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool ok = jj + i < mc;
          v[4 * h + i] = ok ? vv[i] : -INFINITY;
          g[4 * h + i] = gg[i];
          if (ok) tm = fmaxf(tm, vv[i]);
        }
      }
    }
    float ts = 0.f;
    if (tm != -INFINITY) {
#pragma unroll
      for (int i = 0; i < 8; ++i) ts += __expf(v[i] - tm);  // exp(-inf) = 0 for padding
    }
    if (tid == 0 && c0 == 0) trace_mark(p.trace, 7);  // gathered
    // ---- 2. per-warp summaries
    float wm = tm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    float ws = (tm == -INFINITY) ? 0.f : ts * __expf(tm - wm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    const float wt = k > 16 ? warp_kth_largest(tm, k) : -INFINITY;
    if (lane == 0) { sh.wmax[warp] = wm; sh.wsum[warp] = ws; sh.wthr[warp] = wt; }
    if (tid == 0) sh.ncand = sh.nbest;  // the running best go first
    __syncthreads();
    // ---- 3. every warp combines the 17 warp summaries itself (no extra
    //         barrier): lse partial (kept by thread 0) and the threshold T
    float T;
    {
      const float x = lane < kWarps ? sh.wmax[lane] : -INFINITY;
      float M = x;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      if (warp == 0) {
        float es = (lane < kWarps && x != -INFINITY) ? sh.wsum[lane] * __expf(x - M) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
        if (lane == 0 && M != -INFINITY) {
          const float nm = fmaxf(run_max, M);
          run_sum = (run_max == -INFINITY ? 0.f : run_sum * __expf(run_max - nm)) + es * __expf(M - nm);
          run_max = nm;
        }
      }
      if (k <= 16) {
        // k-th largest warp maximum, by counting over the kWarps lanes
        int rank = 0;
#pragma unroll
        for (int j = 0; j < kWarps; ++j) {
          const float o = __shfl_sync(0xffffffffu, x, j);
          rank += (o > x || (o == x && j < lane)) ? 1 : 0;
        }
        const unsigned sel = __ballot_sync(0xffffffffu, lane < kWarps && rank == k - 1);
        T = __shfl_sync(0xffffffffu, x, __ffs(sel) - 1);
      } else {
        T = lane < kWarps ? sh.wthr[lane] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) T = fmaxf(T, __shfl_xor_sync(0xffffffffu, T, o));
      }
      if (sh.nbest == k) T = fmaxf(T, sh.best_v[k - 1]);
    }
    if (tid == 0 && c0 == 0) trace_mark(p.trace, 9);  // threshold
    // ---- 4. compact the values >= T (plus the running best), then rank
    const int nprev = sh.nbest;
    if (tid < nprev) { cv[tid] = sh.best_v[tid]; cg[tid] = sh.best_g[tid]; }
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) cnt += (v[i] != -INFINITY && v[i] >= T) ? 1 : 0;
    if (cnt) {
      int slot = atomicAdd(&sh.ncand, cnt);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (v[i] != -INFINITY && v[i] >= T) {
          if (slot < kCandCap) { cv[slot] = v[i]; cg[slot] = g[i]; }
          ++slot;
        }
    }
    __syncthreads();
    if (tid == 0 && c0 == 0) trace_mark(p.trace, 10);  // compacted
    const int tot = sh.ncand;
    if (tid == 0 && c0 == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 15] = tot;
    if (tot > kCandCap) {
      // Degenerate ties (e.g. h = 0): exact but slow fallback -- one thread
      // re-walks the chunk in row order (= ascending id) with a sorted best-k.
      if (tid == 0) {
        int nb = sh.nbest;
        for (int jj = 0; jj < mc; ++jj) {
          const int j = c0 + jj;
          const float vv = __ldcg(a.zl + ((long long)seq * p.n + node) * p.max_ids + j);
          const int32_t gg = __ldg(ids + j);
          if (nb == k && !ranks_before(vv, gg, sh.best_v[k - 1], sh.best_g[k - 1])) continue;
          int pos = nb < k ? nb : k - 1;
          while (pos > 0 && ranks_before(vv, gg, sh.best_v[pos - 1], sh.best_g[pos - 1])) {
            sh.best_v[pos] = sh.best_v[pos - 1];
            sh.best_g[pos] = sh.best_g[pos - 1];
            --pos;
          }
          sh.best_v[pos] = vv;
          sh.best_g[pos] = gg;
          if (nb < k) ++nb;
        }
        sh.nbest = nb;
      }
      __syncthreads();
      continue;
    }
    for (int e = tid; e < tot; e += kThreads) {
      const float ve = cv[e];
      const int32_t ge = cg[e];
      int r = 0;
      for (int f = 0; f < tot; ++f) r += ranks_before(cv[f], cg[f], ve, ge) ? 1 : 0;
      if (r < k) { sh.best_v[r] = ve; sh.best_g[r] = ge; }
    }
    __syncthreads();
    if (tid == 0) sh.nbest = min(k, tot);
    if (tid == 0 && c0 == 0) trace_mark(p.trace, 11);  // ranked
    __syncthreads();
  }
  if (tid < k) {
    const bool ok = tid < sh.nbest;
    a.topk_logit[ob + tid] = ok ? sh.best_v[tid] : -INFINITY;
    a.topk_id[ob + tid] = ok ? sh.best_g[tid] : -1;
  }
  if (a.lse && tid == 0)
    a.lse[(long long)seq * p.n + node] = run_max == -INFINITY ? -INFINITY : run_max + logf(run_sum);
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) head_tc_kernel(TcArgs a) {
  using C = Cfg<NT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned view that keeps the shared address space visible to the compiler
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStageArea);
  // bars[0..S) full, [S..2S) empty, [2S] tmem_full, [2S+1] tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 2);
  __shared__ int sh_tiles, sh_S, sh_m0;
  __shared__ TopkSmem tsh;

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int KB = p.d / kBK;
  const int G = gridDim.x;

  if (tid == 0) trace_mark(p.trace, 0);  // start
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&bars[s]), kLoaders);          // full: every loader thread arrives
      mbar_init(smem_u32(&bars[C::kStages + s]), 1);    // empty: one tcgen05.commit
    }
    mbar_init(smem_u32(&bars[2 * C::kStages]), 1);              // tmem_full
    mbar_init(smem_u32(&bars[2 * C::kStages + 1]), kLoaders);   // tmem_empty
    fence_proxy_async();
  }
  if (warp == kLoadWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // Everything above overlaps the previous kernel (programmatic dependent
  // launch); the state it produced (n_active, ids) is read only after this.
  pdl_wait();
  // the next kernel on the stream (typically the next state update) may be
  // launched now; it waits for this grid's completion before touching state
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) trace_mark(p.trace, 1);  // dependency resolved

  // Loader pattern: thread t moves 16-B chunk (t & 7) of tile rows lr and
  // lr + 64 (lr = t >> 3) of every W stage, and of H rows lr + 64 i < NT.
  const int lr = tid >> 3;
  const uint32_t swz = (uint32_t)(((tid & 7) ^ (lr & 7)) << 4);
  // Speculative first unit, assuming every sequence holds max_ids active rows:
  // its id loads go out together with the n_active reads (re-issued below if
  // the guess is wrong).
  const int tps_g = (p.max_ids + kBM - 1) / kBM;
  const int tiles_g = p.batch * tps_g;
  const int S_g = (tiles_g >= G) ? 1 : min(KB, G / tiles_g);
  int32_t gid_pre[2] = {0, 0};
  if (warp < kLoadWarps && (int)blockIdx.x < tiles_g * S_g) {
    const int tg = blockIdx.x / S_g;
    const int32_t* idp = p.ids_base + (long long)(tg / tps_g) * p.ids_stride + (tg % tps_g) * kBM;
    const int lim = p.max_ids - (tg % tps_g) * kBM - 1;
    gid_pre[0] = __ldg(idp + min(lr, lim));
    gid_pre[1] = __ldg(idp + min(lr + 64, lim));
  }
  if (warp == 0) {
    int t = 0, m0 = 0;
    for (int b = lane; b < p.batch; b += 32) {
      const int m = clamp_nact(p, b);
      if (b == 0) m0 = m;
      t += (m + kBM - 1) / kBM;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) {
      sh_tiles = t;
      sh_S = (t >= G || t == 0) ? 1 : min(KB, G / t);
      sh_m0 = m0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int tiles = sh_tiles, S = sh_S, units = tiles * S;
  const bool guess_ok = (S == S_g && tiles == tiles_g);
  constexpr uint32_t idesc = make_idesc(kBM, NT);

  int it = 0;      // pipeline iteration counter across units
  int local = 0;   // units processed by this CTA
  int seq = 0, seq_tile0 = 0, seq_m = sh_m0;  // tile -> sequence walk (units are tile-major)
  for (int u = blockIdx.x; u < units; u += G, ++local) {
    const int tile = u / S, split = u - (u / S) * S;
    while (tile - seq_tile0 >= (seq_m + kBM - 1) / kBM) {  // advance to the tile's sequence
      seq_tile0 += (seq_m + kBM - 1) / kBM;
      ++seq;
      seq_m = clamp_nact(p, seq);
    }
    const int row0 = (tile - seq_tile0) * kBM;
    const int rows = min(kBM, seq_m - row0);
    const int kb0 = split * KB / S, kb1 = (split + 1) * KB / S;
    const int nk = kb1 - kb0;

    if (warp < kLoadWarps) {
      // ---------------- producers: gather rows of W_head + H into SW128 stages
      int32_t gid[2];
      if (local == 0 && guess_ok) {
        gid[0] = gid_pre[0];
        gid[1] = gid_pre[1];
      } else {
        const int32_t* idp = p.ids_base + (long long)seq * p.ids_stride + row0;
        gid[0] = __ldg(idp + min(lr, rows - 1));
        gid[1] = __ldg(idp + min(lr + 64, rows - 1));
      }
      const uint16_t* rp[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const long long row = p.n_shards > 1 ? gid[i] / p.n_shards : gid[i];
        rp[i] = (lr + 64 * i < rows) ? p.w + row * p.ldw + (tid & 7) * 8 : nullptr;
      }
      const uint16_t* hp = p.h + (long long)seq * p.n * p.d + (tid & 7) * 8;
      if (tid == 0 && local == 0) trace_mark(p.trace, 2);  // row pointers ready, first loads next
      for (int q = 0; q < nk + C::kStages - 1; ++q) {
        if (q < nk) {
          const int g_it = it + q;
          const int stage = g_it % C::kStages;
          if (g_it >= C::kStages) mbar_wait(smem_u32(&bars[C::kStages + stage]), ((g_it / C::kStages) - 1) & 1);
          const uint32_t sA = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sB = sA + C::kABytes;
          const int kcol = (kb0 + q) * kBK;
#pragma unroll
          for (int i = 0; i < 2; ++i)
            cp_async16(sA + (lr + 64 * i) * 128 + swz, rp[i] ? (const void*)(rp[i] + kcol) : (const void*)p.w,
                       rp[i] ? 16u : 0u);
#pragma unroll
          for (int i = 0; i < (C::kHChunks + kLoaders - 1) / kLoaders; ++i) {
            const int hr = lr + 64 * i;
            if (hr < NT)
              cp_async16(sB + hr * 128 + swz, hr < p.n ? (const void*)(hp + (long long)hr * p.d + kcol) : (const void*)p.h,
                         hr < p.n ? 16u : 0u);
          }
        }
        cp_async_commit();
        if (q >= C::kStages - 1) {
          cp_async_wait<C::kStages - 1>();
          fence_proxy_async();
          mbar_arrive(smem_u32(&bars[(it + q - (C::kStages - 1)) % C::kStages]));
        }
      }
      if (tid == 0 && local == 0) trace_mark(p.trace, 3);  // all loads issued and landed
      // ---------------- epilogue: TMEM -> registers -> partial tile (L2)
      mbar_wait(smem_u32(&bars[2 * C::kStages]), local & 1);
      tc_fence_after();
      if (tid == 0 && local == 0) trace_mark(p.trace, 4);  // last MMA done
      const int lg = warp & 3, cgp = warp >> 2;   // TMEM lane group, column group
      const int r = lg * 32 + lane;               // TMEM lane == tile row
      const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
      float* dst = a.part + (long long)u * NT * kBM + r;
      if (cgp < C::kColGroups) {
#pragma unroll 1
        for (int c0 = cgp * 16; c0 < NT && c0 < p.n; c0 += 16 * C::kColGroups) {
          float v[16];
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < p.n) __stcg(dst + (c0 + c) * kBM, v[c]);
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&bars[2 * C::kStages + 1]));
    } else {
      // ---------------- MMA issuer (warp 16, one lane)
      if (local > 0) {
        mbar_wait(smem_u32(&bars[2 * C::kStages + 1]), (local - 1) & 1);
        tc_fence_after();
      }
      for (int q = 0; q < nk; ++q) {
        const int g_it = it + q;
        const int stage = g_it % C::kStages;
        mbar_wait(smem_u32(&bars[stage]), (g_it / C::kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sB = sA + C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            umma_bf16(tmem, sw128_desc(sA + kk * 32), sw128_desc(sB + kk * 32), idesc, (q | kk) ? 1u : 0u);
          umma_commit(smem_u32(&bars[C::kStages + stage]));
          if (q == nk - 1) umma_commit(smem_u32(&bars[2 * C::kStages]));
        }
        __syncwarp();
      }
    }
    it += nk;

    // ---------------- split-K reduction, distributed over the tile's S CTAs:
    // once all S partials of the tile are written (per-tile arrival counter;
    // the launch is cooperative so the spin is safe), split s sums, in split
    // order, quads [32 s / S, 32 (s+1) / S) of the tile's rows for every node
    // and writes the final logits.
    __threadfence();
    __syncthreads();
    if (S > 1) {
      if (tid == 0) {
        atomicAdd(&a.counters[2 + tile], 1u);
        while (ld_acquire(&a.counters[2 + tile]) < (unsigned)S) __nanosleep(20);
      }
      __syncthreads();
    }
    if (tid == 0 && local == 0) trace_mark(p.trace, 5);  // tile's partials complete
    {
      const int q0 = split * (kBM / 4) / S, q1 = (split + 1) * (kBM / 4) / S;
      const int nq = q1 - q0;
      for (int item = tid; item < p.n * nq; item += kThreads) {
        const int c = item / nq, r = 4 * (q0 + item - (item / nq) * nq);
        if (r >= rows) continue;
        const float* src = a.part + ((long long)tile * S * NT + c) * kBM + r;
        float4 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < S) x[q] = __ldcg(reinterpret_cast<const float4*>(src + (long long)q * NT * kBM));
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < S) { acc.x += x[q].x; acc.y += x[q].y; acc.z += x[q].z; acc.w += x[q].w; }
        for (int q = 8; q < S; ++q) {
          const float4 y = __ldcg(reinterpret_cast<const float4*>(src + (long long)q * NT * kBM));
          acc.x += y.x; acc.y += y.y; acc.z += y.z; acc.w += y.w;
        }
        float* dst = a.zl + ((long long)seq * p.n + c) * p.max_ids + row0 + r;
        if (((uintptr_t)dst & 15) == 0 && r + 4 <= rows) {
          __stcg(reinterpret_cast<float4*>(dst), acc);
        } else {
          const float vv[4] = {acc.x, acc.y, acc.z, acc.w};
          for (int i = 0; i < 4 && r + i < rows; ++i) __stcg(dst + i, vv[i]);
        }
      }
    }
  }

  // ---------------- grid barrier: every logit reduced
  if (tid == 0) trace_mark(p.trace, 6);  // reduction done
  __threadfence();
  tc_fence_before();
  __syncthreads();
  const int tasks = p.batch * p.n;
  if (tid == 0) {
    atomicAdd(&a.counters[0], 1u);
    if ((int)blockIdx.x < tasks)  // CTAs with top-k work wait for everyone
      while (ld_acquire(&a.counters[0]) < (unsigned)G) __nanosleep(32);
    trace_mark(p.trace, 12);  // grid barrier passed
  }
  __syncthreads();

  // ---------------- top-k: (sequence, node) tasks over the CTAs
  {
    int tseq = 0, tm = sh_m0;
    for (int t = blockIdx.x; t < tasks; t += G) {
      const int sq = t / p.n, node = t - (t / p.n) * p.n;
      while (tseq < sq) {
        ++tseq;
        tm = clamp_nact(p, tseq);
      }
      topk_node<NT>(a, sq, node, tm, smem, tsh);
    }
  }

  // ---------------- teardown: last CTA out resets the counters for the next launch
  if (tid == 0) trace_mark(p.trace, 8);  // top-k done
  __syncthreads();
  if (tid == 0) {
    const unsigned old = atomicAdd(&a.counters[1], 1u);
    sh_tiles = (old == (unsigned)G - 1) ? 1 : 0;
  }
  __syncthreads();
  if (sh_tiles) {  // the last CTA: every other CTA has passed all its waits
    for (int t = tid; t < tiles; t += kThreads) a.counters[2 + t] = 0u;
    if (tid == 0) { a.counters[0] = 0u; a.counters[1] = 0u; }
    __threadfence();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kLoadWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
}

struct ScratchLayout {
  size_t counters, part, zl, total;
};

inline ScratchLayout scratch_layout(int batch, int max_ids, int n, int nt) {
  const size_t max_tiles = (size_t)batch * ((max_ids + kBM - 1) / kBM);
  const size_t units_cap = max_tiles > (size_t)kMaxSMs ? max_tiles : (size_t)kMaxSMs;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  ScratchLayout L;
  size_t off = 0;
  L.counters = off; off += al(sizeof(unsigned) * (2 + max_tiles));
  L.part = off;     off += al(units_cap * nt * kBM * sizeof(float));
  L.zl = off;       off += al((size_t)batch * n * max_ids * sizeof(float));
  L.total = off;
  return L;
}

inline int nt_for(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

template <int NT>
cudaError_t launch_nt(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse, void* scratch,
                      size_t scratch_bytes, int num_sms, cudaStream_t stream) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(head_tc_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = num_sms < kMaxSMs ? num_sms : kMaxSMs;
  const ScratchLayout L = scratch_layout(p.batch, p.max_ids, p.n, NT);
  if (L.total > scratch_bytes) return cudaErrorInvalidValue;
  char* sc = (char*)scratch;
  TcArgs a;
  a.p = p;
  a.counters = (unsigned*)(sc + L.counters);
  a.part = (float*)(sc + L.part);
  a.zl = p.logits ? p.logits : (float*)(sc + L.zl);
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.k = k;
  a.max_tiles = p.batch * ((p.max_ids + kBM - 1) / kBM);

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT>, a);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    cfg.numAttrs = 1;  // cooperative only
    e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT>, a);
  }
  return e;
}

}  // namespace

size_t head_tc_scratch_bytes(int batch, int max_ids, int n) {
  return scratch_layout(batch, max_ids, n, nt_for(n)).total;
}

cudaError_t launch_head_tc(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                           void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream) {
  if (p.d % kBK != 0 || p.n < 1 || p.n > 256 || p.ldw % 8 != 0 || k < 1 || k > kMaxK) return cudaErrorNotSupported;
  if (p.n <= 16) return launch_nt<16>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 32) return launch_nt<32>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 64) return launch_nt<64>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 128) return launch_nt<128>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  return launch_nt<256>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
}

}  // namespace nanospec
