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
// padded), K = 64 per pipeline stage; D in TMEM (NT fp32 columns).  A launch
// covers tiles_g = batch * ceil(max_ids / 128) row tiles (tiles past a
// sequence's n_active, read from device memory, exit at once).  With
// tiles_g < #SMs every tile is split along K into S = min(8, #SMs / tiles_g)
// chunks handled by the S CTAs of one thread-block cluster, so ~all SMs stream.
//
// Reduction + top-k, no grid-wide synchronisation:
//  1. each CTA drains its partial tile from TMEM into its own shared memory;
//     after a cluster barrier, CTA s sums -- over distributed shared memory, in
//     split order (fixed order: equal rows give bit-equal logits) -- the 128
//     rows of nodes s, s+S, ...;
//  2. level 1, one warp per (tile, node): exact top-k of the 128 logits
//     (threshold = k-th largest lane maximum, compaction, rank by counting)
//     and (max, sum exp) for the lse, written to L2-resident scratch;
//  3. level 2: a per-(sequence, node) arrival counter; the warp that brings it
//     to ceil(n_active / 128) merges that node's sorted per-tile lists
//     (threshold = k-th largest list head, rank by counting) and combines the
//     lse partials -- the last arriver finishes the node, nobody waits.
//
// Warp roles (544 threads): warps 0-15 load (cp.async) and drain TMEM (warp w
// reads TMEM lanes 32*(w%4).. and a quarter of the columns); warp 16 allocates
// TMEM and one lane issues the MMAs.  All 17 warps run the reduction / top-k.
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
constexpr int kMaxK = 32;
constexpr int kMaxCluster = 8;    // portable cluster size
constexpr int kL2Tiles = 64;      // tiles per sequence whose level-2 inputs are fetched in one round trip

struct TcArgs {
  HeadProblem p;
  uint2* cand;          // [tiles_g][n][k] level-1 lists (float_key, global id), best first
  float2* tstat;        // [tiles_g][n] (max, sum exp(z - max)) over a tile's rows
  unsigned* node_ctr;   // [batch * n] level-1 arrivals per (sequence, node); zero between launches
  float* topk_logit;    // [batch][n][k]
  int32_t* topk_id;
  float* lse;           // [batch][n] or null
  int k;
  int S;                // K splits per tile == cluster size (1: no cluster, persistent CTAs)
  int tps;              // tiles per sequence = ceil(max_ids / 128)
};

// ------------------------------------------------------------------ PTX helpers
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
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared-memory location in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_v4(uint32_t caddr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(caddr)
               : "memory");
  return v;
}
__device__ __forceinline__ int clamp_nact(const HeadProblem& p, int b) {
  int m = p.nact_base[(long long)b * p.nact_stride];
  return m < 0 ? 0 : (m > p.max_ids ? p.max_ids : m);
}

template <int NT>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr int kBBytes = NT * kBK * 2;   // NT * 128 B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = NT < 32 ? 32 : NT;
  static constexpr int kStageArea = kStages * kStageBytes;
  // after the MMAs the stage area holds the partial tile P[NT][128] fp32 and a
  // per-warp scratch for the selections
  static constexpr int kPBytes = NT * kBM * 4;
  static constexpr int kWarpScratch = ((kStageArea - kPBytes) / kWarps) / 8 * 8;  // bytes
  static_assert(kWarpScratch >= kBM * 8, "per-warp scratch");
  static constexpr int kSmemBytes = kStageArea + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(2 * kStages + 3 <= 30, "barrier area");
  static constexpr int kHChunks = NT * 8;                 // 16-B chunks of one H stage
  static constexpr int kColGroups = NT / 16 < 4 ? NT / 16 : 4;  // epilogue column groups
};

__device__ __forceinline__ float key_value(uint32_t kk) {
  if (kk == 0u) return -INFINITY;  // "none"
  return __uint_as_float((kk & 0x80000000u) ? (kk & 0x7fffffffu) : ~kk);
}
// (value desc, id asc): a before b
__device__ __forceinline__ bool key_before(uint32_t ka, int32_t ga, uint32_t kb, int32_t gb) {
  return ka > kb || (ka == kb && ga < gb);
}
// k-th largest (1 <= k <= 32) of one key per lane, by counting (ties by lane).
__device__ __forceinline__ uint32_t warp_kth_key(uint32_t x, int k) {
  const int lane = threadIdx.x & 31;
  int rank = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t o = __shfl_sync(0xffffffffu, x, j);
    rank += (o > x || (o == x && j < lane)) ? 1 : 0;
  }
  const unsigned sel = __ballot_sync(0xffffffffu, rank == k - 1);
  return __shfl_sync(0xffffffffu, x, __ffs(sel) - 1);
}

// Rank `cnt` staged (key, gid) candidates by counting and write the k best
// (best first) to out[0..k); the warp-private scratch holds the candidates.
__device__ __forceinline__ void warp_rank_write(const uint2* cs, int cnt, int k, uint2* out) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < cnt; e += 32) {
    const uint2 me = cs[e];
    int r = 0;
    for (int f = 0; f < cnt; ++f) {
      const uint2 o = cs[f];
      r += key_before(o.x, (int32_t)o.y, me.x, (int32_t)me.y) ? 1 : 0;
    }
    if (r < k) out[r] = me;
  }
}

// Level 1 for one (tile, node): the 128 logits of the tile's rows (4 per lane).
// Writes the tile's sorted top-k (key, gid) -- padded with (0, -1) -- and
// (max, sum exp) of the valid rows.
__device__ __forceinline__ void level1(const float (&v)[4], const int32_t (&g)[4], int r0, int rows, int k,
                                       uint2* scratch, uint2* cand_out, float2* tstat_out) {
  const int lane = threadIdx.x & 31;
  uint32_t key[4];
  uint32_t lmk = 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    key[i] = (r0 + i < rows) ? float_key(v[i]) : 0u;
    lmk = key[i] > lmk ? key[i] : lmk;
  }
  // lse partial
  const float M = key_value(__reduce_max_sync(0xffffffffu, lmk));
  float es = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (key[i]) es += __expf(v[i] - M);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
  // threshold: k-th largest lane maximum (k lanes each own a value >= T)
  const uint32_t T = warp_kth_key(lmk, k);
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool c = key[i] != 0u && key[i] >= T;
    const unsigned bal = __ballot_sync(0xffffffffu, c);
    if (c) scratch[cnt + __popc(bal & ((1u << lane) - 1u))] = make_uint2(key[i], (uint32_t)g[i]);
    cnt += __popc(bal);
  }
  __syncwarp();
  if (lane < k) cand_out[lane] = make_uint2(0u, 0xffffffffu);  // padding when rows < k
  __syncwarp();
  warp_rank_write(scratch, cnt, k, cand_out);
  if (lane == 0) *tstat_out = make_float2(M, es);
}

// Level 2 for one (sequence, node), one warp: merge ntiles sorted lists.
__device__ void level2(const TcArgs& a, int seq, int node, int tile0, int ntiles, uint2* scratch, int cap) {
  const HeadProblem& p = a.p;
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const long long ob = ((long long)seq * p.n + node) * k;
  const uint2* lists = a.cand + ((long long)tile0 * p.n + node) * k;  // list t at lists + t * n * k
  const long long lstride = (long long)p.n * k;
  // one round trip: every lane fetches its tiles' (max, sum exp) and list heads
  float2 st[kL2Tiles / 32];
  uint32_t head[kL2Tiles / 32];
  uint32_t mk = 0u;
#pragma unroll
  for (int c = 0; c < kL2Tiles / 32; ++c) {
    const int t = lane + 32 * c;
    st[c] = make_float2(-INFINITY, 0.f);
    head[c] = 0u;
    if (t < ntiles) {
      st[c] = __ldcg(&a.tstat[(long long)(tile0 + t) * p.n + node]);
      head[c] = __ldcg(&lists[t * lstride]).x;
    }
  }
  for (int t = lane + kL2Tiles; t < ntiles; t += 32) {  // (more than kL2Tiles tiles: rare)
    const float x = __ldcg(&a.tstat[(long long)(tile0 + t) * p.n + node]).x;
    const uint32_t kx = x == -INFINITY ? 0u : float_key(x);
    mk = kx > mk ? kx : mk;
  }
#pragma unroll
  for (int c = 0; c < kL2Tiles / 32; ++c) {
    const uint32_t kx = st[c].x == -INFINITY ? 0u : float_key(st[c].x);
    mk = kx > mk ? kx : mk;
  }
  const float M = key_value(__reduce_max_sync(0xffffffffu, mk));
  float es = 0.f;
#pragma unroll
  for (int c = 0; c < kL2Tiles / 32; ++c)
    if (st[c].x != -INFINITY) es += st[c].y * __expf(st[c].x - M);
  for (int t = lane + kL2Tiles; t < ntiles; t += 32) {
    const float2 s2 = __ldcg(&a.tstat[(long long)(tile0 + t) * p.n + node]);
    if (s2.x != -INFINITY) es += s2.y * __expf(s2.x - M);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
  // threshold: k-th largest list head (k lists each own a value >= T)
  uint32_t T = 0u;
  if (ntiles <= 32 && ntiles >= k) T = warp_kth_key(head[0], k);
  // candidates >= T into the warp scratch; each lane reads its list kChunk
  // entries at a time (all in flight), stopping once a whole row qualifies nowhere
  constexpr int kChunk = 8;
  int cnt = 0;
  bool overflow = false;
  for (int t0 = 0; t0 < ntiles; t0 += 32) {
    const int t = t0 + lane;
    bool more = true;
    for (int j0 = 0; j0 < k && more; j0 += kChunk) {
      uint2 e[kChunk];
#pragma unroll
      for (int jj = 0; jj < kChunk; ++jj)
        e[jj] = (t < ntiles && j0 + jj < k) ? __ldcg(&lists[t * lstride + j0 + jj]) : make_uint2(0u, 0u);
#pragma unroll
      for (int jj = 0; jj < kChunk; ++jj) {
        const bool c = e[jj].x != 0u && e[jj].x >= T;
        const unsigned bal = __ballot_sync(0xffffffffu, c);
        if (!bal) { more = false; break; }  // lists are sorted: nothing further qualifies
        const int slot = cnt + __popc(bal & ((1u << lane) - 1u));
        if (c && slot < cap) scratch[slot] = e[jj];
        cnt += __popc(bal);
      }
    }
  }
  overflow = cnt > cap;
  __syncwarp();
  uint2 res = make_uint2(0u, 0xffffffffu);
  if (!overflow) {
    uint2* best = scratch + cap - kMaxK;  // (cap > kMaxK + candidates: guarded below)
    if (cnt + kMaxK <= cap) {
      if (lane < k) best[lane] = make_uint2(0u, 0xffffffffu);
      __syncwarp();
      warp_rank_write(scratch, cnt, k, best);
      __syncwarp();
      if (lane < k) res = best[lane];
    } else {
      overflow = true;
    }
  }
  if (overflow) {
    // many candidates (e.g. the dense [0, V) comparator): k rounds of a warp
    // arg-max over the list heads (heads kept in the scratch as positions)
    int* hpos = reinterpret_cast<int*>(scratch);
    for (int t = lane; t < ntiles; t += 32) hpos[t] = 0;
    __syncwarp();
    for (int r = 0; r < k; ++r) {
      uint32_t bk = 0u;
      int32_t bg = 0x7fffffff;
      int bt = -1;
      for (int t = lane; t < ntiles; t += 32) {
        if (hpos[t] >= k) continue;
        const uint2 e = __ldcg(&lists[t * lstride + hpos[t]]);
        if (e.x != 0u && key_before(e.x, (int32_t)e.y, bk, bg)) { bk = e.x; bg = (int32_t)e.y; bt = t; }
      }
      const uint32_t wk = __reduce_max_sync(0xffffffffu, bk);
      if (wk == 0u) break;
      const int32_t wg = (int32_t)__reduce_min_sync(0xffffffffu, bk == wk ? (uint32_t)bg : 0x7fffffffu);
      if (bk == wk && bg == wg && bt >= 0) hpos[bt] += 1;
      __syncwarp();
      if (lane == r) res = make_uint2(wk, (uint32_t)wg);
    }
  }
  if (lane < k) {
    a.topk_logit[ob + lane] = res.x ? key_value(res.x) : -INFINITY;
    a.topk_id[ob + lane] = res.x ? (int32_t)res.y : -1;
  }
  if (a.lse && lane == 0) a.lse[(long long)seq * p.n + node] = M == -INFINITY ? -INFINITY : M + logf(es);
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
  __shared__ int32_t ids_s[kBM];   // the unit's row ids
  __shared__ int sh_last[kWarps];

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int KB = p.d / kBK;
  const int S = a.S;

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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = make_idesc(kBM, NT);
  // Loader pattern: thread t moves 16-B chunk (t & 7) of tile rows lr and
  // lr + 64 (lr = t >> 3) of every W stage, and of H rows lr + 64 i < NT.
  const int lr = tid >> 3;
  const uint32_t swz = (uint32_t)(((tid & 7) ^ (lr & 7)) << 4);
  uint2* wscratch = reinterpret_cast<uint2*>(smem + C::kPBytes + warp * C::kWarpScratch);
  const int wcap = C::kWarpScratch / 8;
  const float* Pm = reinterpret_cast<const float*>(smem);  // partial tile [NT][128] after the MMAs

  const int tiles_g = p.batch * a.tps;
  const int split = S > 1 ? (int)cluster_ctarank() : 0;
  const int first = S > 1 ? (int)blockIdx.x / S : (int)blockIdx.x;
  const int step = S > 1 ? tiles_g : (int)gridDim.x;
  int it = 0;      // pipeline iteration counter across units
  int local = 0;   // units processed by this CTA
  for (int tile = first; tile < tiles_g; tile += step) {
    const int seq = tile / a.tps, tin = tile - (tile / a.tps) * a.tps;
    const int m = clamp_nact(p, seq);
    const int row0 = tin * kBM;
    const int rows = min(kBM, m - row0);
    if (rows <= 0) continue;  // the whole cluster (same tile) skips together
    const int ntiles = (m + kBM - 1) / kBM;
    const int kb0 = split * KB / S, kb1 = (split + 1) * KB / S;
    const int nk = kb1 - kb0;
    if (tid < kBM) {
      const int32_t* idp = p.ids_base + (long long)seq * p.ids_stride + row0;
      ids_s[tid] = __ldg(idp + min(tid, rows - 1));
    }
    __syncthreads();

    if (warp < kLoadWarps) {
      // ---------------- producers: gather rows of W_head + H into SW128 stages
      const uint16_t* rp[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int32_t g = ids_s[lr + 64 * i];
        const long long row = p.n_shards > 1 ? g / p.n_shards : g;
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
      // ---------------- epilogue: TMEM -> registers -> partial tile P in shared memory
      mbar_wait(smem_u32(&bars[2 * C::kStages]), local & 1);
      tc_fence_after();
      if (tid == 0 && local == 0) trace_mark(p.trace, 4);  // last MMA done
      const int lg = warp & 3, cgp = warp >> 2;   // TMEM lane group, column group
      const int r = lg * 32 + lane;               // TMEM lane == tile row
      const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
      float* Pw = reinterpret_cast<float*>(smem) + r;
      if (cgp < C::kColGroups) {
#pragma unroll 1
        for (int c0 = cgp * 16; c0 < NT && c0 < p.n; c0 += 16 * C::kColGroups) {
          float v[16];
          tmem_ld16(taddr + c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < p.n) Pw[(c0 + c) * kBM] = v[c];
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
      // the MMA warp joins below once the epilogue has drained TMEM
      mbar_wait(smem_u32(&bars[2 * C::kStages + 1]), local & 1);
    }
    it += nk;

    // ---------------- split-K reduction over the cluster, level-1 top-k
    __syncthreads();  // P complete in this CTA
    if (S > 1) cluster_sync();  // ... and in every CTA of the cluster
    if (tid == 0 && local == 0) trace_mark(p.trace, 5);  // partials complete
    if (lane == 0) sh_last[warp] = 0;
    for (int c = split + S * warp; c < p.n; c += S * kWarps) {
      // node c, rows 4*lane .. 4*lane+3: sum of the S partials in split order
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      const uint32_t la = smem_u32(Pm + c * kBM + 4 * lane);
      if (S == 1) {
        acc = *reinterpret_cast<const float4*>(Pm + c * kBM + 4 * lane);
      } else {
        float4 x[kMaxCluster];
#pragma unroll
        for (int s2 = 0; s2 < kMaxCluster; ++s2)
          if (s2 < S) x[s2] = ld_dsmem_v4(mapa_shared(la, (uint32_t)s2));
#pragma unroll
        for (int s2 = 0; s2 < kMaxCluster; ++s2)
          if (s2 < S) { acc.x += x[s2].x; acc.y += x[s2].y; acc.z += x[s2].z; acc.w += x[s2].w; }
      }
      const float v[4] = {acc.x, acc.y, acc.z, acc.w};
      const int32_t g[4] = {ids_s[4 * lane], ids_s[4 * lane + 1], ids_s[4 * lane + 2], ids_s[4 * lane + 3]};
      if (p.logits) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * lane + i < rows) p.logits[((long long)seq * p.n + c) * p.max_ids + row0 + 4 * lane + i] = v[i];
      }
      uint2* cout = a.cand + ((long long)tile * p.n + c) * a.k;
      level1(v, g, 4 * lane, rows, a.k, wscratch, cout, &a.tstat[(long long)tile * p.n + c]);
      // level 2: the warp whose list completes the node merges it.  The warp's
      // list is published by lane 0's release (after the warp barrier); the
      // last arriver's acquire makes every tile's list visible.
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) {
        last = atom_add_acq_rel(&a.node_ctr[seq * p.n + c], 1u) == (unsigned)(ntiles - 1);
        if (last) a.node_ctr[seq * p.n + c] = 0u;  // every other tile has arrived: reset for the next launch
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) level2(a, seq, c, seq * a.tps, ntiles, wscratch, wcap);
    }
    if (tid == 0 && local == 0) trace_mark(p.trace, 6);  // level 1 (+ merges) done
    if (S > 1) cluster_sync();  // peers are done reading this CTA's partials
    __syncthreads();            // P / scratch free for the next unit
    ++local;
  }

  if (tid == 0) trace_mark(p.trace, 8);  // done
  tc_fence_before();
  __syncthreads();
  if (warp == kLoadWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
}

struct ScratchLayout {
  size_t node_ctr, cand, tstat, total;
};

inline ScratchLayout scratch_layout(int batch, int max_ids, int n) {
  const size_t tiles = (size_t)batch * ((max_ids + kBM - 1) / kBM);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  ScratchLayout L;
  size_t off = 0;
  L.node_ctr = off; off += al(sizeof(unsigned) * (size_t)batch * n);
  L.cand = off;     off += al(tiles * (size_t)n * kMaxK * sizeof(uint2));
  L.tstat = off;    off += al(tiles * (size_t)n * sizeof(float2));
  L.total = off;
  return L;
}

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
  const ScratchLayout L = scratch_layout(p.batch, p.max_ids, p.n);
  if (L.total > scratch_bytes) return cudaErrorInvalidValue;
  char* sc = (char*)scratch;
  TcArgs a;
  a.p = p;
  a.node_ctr = (unsigned*)(sc + L.node_ctr);
  a.cand = (uint2*)(sc + L.cand);
  a.tstat = (float2*)(sc + L.tstat);
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.k = k;
  a.tps = (p.max_ids + kBM - 1) / kBM;
  const int G = num_sms < kMaxSMs ? num_sms : kMaxSMs;
  const int tiles_g = p.batch * a.tps;
  const int KB = p.d / kBK;
  // Largest cluster (K-split) size S <= 8 whose tiles_g clusters are all
  // co-resident in one wave (GPC packing decides, so ask the runtime; cached).
  static int max_clusters[kMaxCluster + 1] = {0};
  int S = 1;
  if (tiles_g < G) {
    for (int s = kMaxCluster; s >= 2; --s) {
      if (s > KB || s * tiles_g > G) continue;
      if (max_clusters[s] == 0) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(s * tiles_g);
        q.blockDim = dim3(kThreads);
        q.dynamicSmemBytes = C::kSmemBytes;
        cudaLaunchAttribute ca;
        ca.id = cudaLaunchAttributeClusterDimension;
        ca.val.clusterDim.x = s;
        ca.val.clusterDim.y = 1;
        ca.val.clusterDim.z = 1;
        q.attrs = &ca;
        q.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, head_tc_kernel<NT>, &q) != cudaSuccess || nc <= 0) {
          (void)cudaGetLastError();
          nc = -1;
        }
        max_clusters[s] = nc;
      }
      if (max_clusters[s] >= tiles_g) { S = s; break; }
    }
  }
  a.S = S;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S > 1 ? tiles_g * S : (tiles_g < G ? tiles_g : G));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  if (S > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = S;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT>, a);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    cfg.attrs = attrs + 1;  // without PDL
    cfg.numAttrs = na - 1;
    e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT>, a);
  }
  return e;
}

}  // namespace

size_t head_tc_scratch_bytes(int batch, int max_ids, int n) { return scratch_layout(batch, max_ids, n).total; }

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
