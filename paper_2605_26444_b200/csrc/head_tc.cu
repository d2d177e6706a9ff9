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
// covers batch * ceil(max_ids / 128) row tiles (tiles past a sequence's
// n_active, read from device memory, are skipped).  Fewer tiles than SMs: every
// tile is split along K over S CTAs; more: persistent CTAs loop over tiles.
//
// Split-K reduction + top-k, one of four modes (chosen by the launchers):
//  * cluster (the headline): the S CTAs of a tile form a thread-block cluster
//    (S = largest <= 8 with every cluster co-resident: 5 at |I| = 3072); each
//    drains its partial tile TMEM -> smem, and after a cluster barrier CTA s
//    sums the nodes s, s+S, ... over DSMEM in K-chunk order (deterministic),
//    one warp per (tile, node) takes the exact level-1 top-k (threshold = k-th
//    largest lane maximum, compaction, rank by counting) + (max, sum exp); a
//    per-node arrival counter (release/acquire) lets the last tile's warp
//    merge the node's lists (level 2, one round trip) -- nobody waits;
//  * poll (> 32 tiles per sequence, one unit per CTA): partials and lists go
//    through L2 as self-validating words (stored XOR a constant no value
//    equals; the consumer re-zeroes), no fences or flags;
//  * finisher (persistent): whole-tile partials to L2 (two tiles per unit when
//    the capacity is >= 2x the SMs, sharing H), a one-word grid barrier, then
//    one finisher CTA per (sequence, node) sums, keeps an online lse and
//    selects the top-k (sorting network + warp arg-max rounds);
//  * fused step (nanospec_step): cluster mode over the pre-update slots plus
//    patch tiles for the update-list ids, with one extra cluster whose CTA 0
//    runs the state update (state_fast.cuh) while everything streams.
// Every mode relies on all CTAs of a launch being co-resident (grid <= #SMs,
// one CTA per SM, cluster counts from cudaOccupancyMaxActiveClusters).
//
// Warp roles (544 threads): warps 0-15 load (cp.async) and drain TMEM (warp w
// reads TMEM lanes 32*(w%4).. and a quarter of the columns); warp 16 allocates
// TMEM and one lane issues the MMAs.  All 17 warps run the reduction / top-k.
#include <math.h>

#include "common.cuh"
#include "internal.h"
#include "state_fast.cuh"
#include "tc_ptx.cuh"

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
constexpr int kMaxSplit = 32;     // K splits per tile
constexpr int kFinRows = 8;       // rows per finisher thread per round
constexpr int kCountBits = 12;    // grid barrier word: arrivals in bits [0, 12), generation above
// Poll mode hands data between CTAs without fences or flags: every 32-bit word
// is stored XOR-ed with a constant that no real value equals, so a word reads
// as 0 exactly until its producer's store has landed; the consumer re-zeroes
// what it consumed (the scratch starts zeroed, ABI).
constexpr uint32_t kEncF = 0x7fbadbadu;  // partial logits / lse floats: a NaN payload arithmetic never makes
constexpr uint32_t kEncK = 0x00000001u;  // list keys: float_key(v) == 1 only for NaN bit patterns
constexpr uint32_t kEncG = 0x7fffffffu;  // list ids: valid ids are < 2^31 - 1, padding is 0xffffffff
constexpr int kModeFinish = 0;   // persistent CTAs, grid barrier, one finisher CTA per (sequence, node)
constexpr int kModeFinishWide = 5;  // the same with two row tiles per unit (capacity >= 2 x #SMs tiles)
constexpr int kModePoll = 1;     // one unit per CTA, split-K partials + lists handed over through L2
constexpr int kModeCluster = 2;  // one unit per CTA, the S splits of a tile form a cluster (DSMEM reduction)
constexpr int kModeFused = 3;    // cluster mode + the state update in the same launch (patch tiles)
constexpr int kModePair = 6;     // opt-in: the pair-split kernel of head_pair.cu
constexpr int kModeSplit = 7;    // the two-kernel head of head_split.cu (also what auto takes first)
constexpr int kMaxCluster = 8;   // portable cluster size
constexpr int kMaxL2Lists = 160;  // poll mode: tiles per sequence (5 lists per lane at level 2)
constexpr long long kSpinLimit = 1ll << 26;  // polls before giving up (a trap beats a hung GPU)

struct TcArgs {
  HeadProblem p;
  unsigned* grid_word;  // grid barrier: (generation << kCountBits) | arrivals
  float* part;          // [tiles_g * S][n][128] partial tiles (split-K partials, or whole tiles for S = 1)
  uint2* cand;          // poll mode: [tiles_g][n][k + 1] level-1 lists (+ lse partial), encoded
  int mode;             // kModeCluster / kModePoll / kModeFinish / kModeFused (see the launchers)
  int l2poll;           // cluster mode: level-1 lists self-validating, level 2 by the tile-0 CTAs polling
  // fused update + head (kModeFused): one sequence, its update and its head in one launch
  AppendArgs upd;       // the state update (fast path) of sequence upd.seq0
  unsigned* step_ctr;   // publication generation of the update's results
  unsigned* arrive_ctr; // CTAs that have read the pre-update ids / n_active
  uint32_t* stale;      // [w_max / 32] slots (pre-update) whose id left I
  int32_t* enter_ids;   // [kFastThreads] global ids entering I
  int* enter_meta;      // {ne, n_new}
  int tps_reg;          // row tiles over the pre-update slots; patch tiles follow
  int n_patch;          // patch tiles (distinct update-list ids, 128 per tile); then the update cluster
  unsigned* node_ctr;   // cluster mode: [batch * n] level-1 arrivals per (sequence, node); zero between launches
  float* topk_logit;    // [batch][n][k]
  int32_t* topk_id;
  float* lse;           // [batch][n] or null
  int k;
  int S;                // K splits per tile (1: persistent CTAs loop over tiles)
  int tps;              // tiles per sequence = ceil(max_ids / 128)
};

// ------------------------------------------------------------------ PTX helpers
// ------------------------------------------------------------------ PTX helpers

template <int NT, int UT = 1>  // UT: 128-row tiles per work unit (the persistent finisher mode takes 2)
struct Cfg {
  static constexpr int kABytes = UT * kBM * kBK * 2;  // UT x 16 KB
  static constexpr int kBBytes = NT * kBK * 2;        // NT * 128 B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = NT * UT < 32 ? 32 : NT * UT;
  static constexpr int kStageArea = kStages * kStageBytes;
  static constexpr int kSmemBytes = kStageArea + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(2 * kStages + 3 <= 30, "barrier area");
  static_assert(kWarps * kMaxK * 8 + kWarps * 8 + kMaxSplit * kBM * 4 + 1024 <= kStageArea, "finisher scratch");
  static constexpr int kHChunks = NT * 8;                 // 16-B chunks of one H stage
  static constexpr int kColGroups = NT / 16 < 4 ? NT / 16 : 4;  // epilogue column groups
};

// Sort 8 entries (19-comparator network).
__device__ __forceinline__ void sort8(uint32_t (&k)[kFinRows], uint32_t (&g)[kFinRows]) {
#define NS_CX(i, j) cx(k[i], g[i], k[j], g[j])
  NS_CX(0, 2); NS_CX(1, 3); NS_CX(4, 6); NS_CX(5, 7);
  NS_CX(0, 4); NS_CX(1, 5); NS_CX(2, 6); NS_CX(3, 7);
  NS_CX(0, 1); NS_CX(2, 3); NS_CX(4, 5); NS_CX(6, 7);
  NS_CX(2, 4); NS_CX(3, 5);
  NS_CX(1, 4); NS_CX(3, 6);
  NS_CX(1, 2); NS_CX(3, 4); NS_CX(5, 6);
#undef NS_CX
}
// k rounds of a warp arg-max over the heads of per-lane sorted lists of L
// entries (key 0 = none): round r's winner goes to lane r, the winning lane
// shifts its list.  Returns this lane's entry of the warp's sorted top-k.
template <int L>
__device__ __forceinline__ uint2 warp_select(uint32_t (&k)[L], uint32_t (&g)[L], int kk) {
  const int lane = threadIdx.x & 31;
  uint2 mine = make_uint2(0u, 0xffffffffu);
  for (int r = 0; r < kk; ++r) {
    const uint32_t wk = __reduce_max_sync(0xffffffffu, k[0]);
    if (wk == 0u) break;  // fewer than kk entries: the rest stays padding
    const unsigned tied = __ballot_sync(0xffffffffu, k[0] == wk);
    // one holder of the maximum (the usual case): its id; a tie: the smallest id
    const uint32_t wg = (tied & (tied - 1u)) ? __reduce_min_sync(0xffffffffu, k[0] == wk ? g[0] : 0xffffffffu)
                                             : __shfl_sync(0xffffffffu, g[0], __ffs(tied) - 1);
    if (lane == r) mine = make_uint2(wk, wg);
    if (k[0] == wk && g[0] == wg) {
#pragma unroll
      for (int i = 0; i + 1 < L; ++i) { k[i] = k[i + 1]; g[i] = g[i + 1]; }
      k[L - 1] = 0u;
    }
  }
  return mine;
}

// Finisher of one (sequence, node): logits of the m active rows = sum of the S
// partials in split order; top-k by (value desc, id asc) mapped to global ids;
// lse over the active set.  Rows go in rounds of `rr` (a multiple of
// 128, <= kThreads * kFinRows): the round's S partial slices are staged in
// shared memory `sp` by 16-byte cp.async (one round trip, no registers held),
// then thread t sums rows t, t + kThreads, ...  `wl` holds kWarps lists of k
// entries, `wm` kWarps (max, sum exp) pairs.
__device__ void finish_node(const TcArgs& a, int seq, int node, float* sp, int rr, uint2* wl, float2* wm) {
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = a.k, S = a.S;
  const int m = clamp_nact(p, seq);
  const int32_t* ids = p.ids_base + (long long)seq * p.ids_stride;
  const long long pstride = (long long)p.n * kBM;  // floats between consecutive (tile, split) slots
  const float* pbase = a.part + (long long)seq * a.tps * S * pstride + (long long)node * kBM;
  float tm = -INFINITY, te = 0.f;  // this thread's lse partial
  uint2 run = make_uint2(0u, 0xffffffffu);  // this lane's entry of the warp's running top-k
  for (int r0 = 0; r0 < m; r0 += rr) {
    const int nrow = min(rr, m - r0);
    const int ntl = (nrow + kBM - 1) / kBM;  // tiles of this round
    const int nchunks = S * ntl * (kBM / 4);  // 16-B chunks: (split, tile, quarter-row group)
    for (int c = tid; c < nchunks; c += kThreads) {
      const int q = c & (kBM / 4 - 1), tl = (c / (kBM / 4)) % ntl, sidx = c / (kBM / 4 * ntl);
      const float* src = pbase + ((long long)(r0 / kBM + tl) * S + sidx) * pstride + q * 4;
      cp_async16(smem_u32(sp + (long long)sidx * rr + tl * kBM + q * 4), src, 16u);
    }
    cp_async_commit();
    uint32_t key[kFinRows], gid[kFinRows];
#pragma unroll
    for (int i = 0; i < kFinRows; ++i) {
      const int j = i * kThreads + tid;
      gid[i] = j < nrow ? (uint32_t)__ldcg(ids + r0 + j) : 0xffffffffu;
    }
    cp_async_wait<0>();
    for (int c = tid; c < nchunks; c += kThreads) {  // leave the scratch zeroed for poll-mode launches
      const int q = c & (kBM / 4 - 1), tl = (c / (kBM / 4)) % ntl, sidx = c / (kBM / 4 * ntl);
      float* src = const_cast<float*>(pbase) + ((long long)(r0 / kBM + tl) * S + sidx) * pstride + q * 4;
      *reinterpret_cast<uint4*>(src) = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    if (tid == 0 && r0 == 0 && (int)blockIdx.x == seq * p.n + node) trace_mark(p.trace, 10);  // partials staged
#pragma unroll
    for (int i = 0; i < kFinRows; ++i) {
      const int j = i * kThreads + tid;
      key[i] = 0u;
      if (j < nrow) {
        float z = 0.f;
        for (int s2 = 0; s2 < S; ++s2) z += sp[s2 * rr + j];
        key[i] = float_key(z);
        lse_fold(tm, te, z, 1.f);
        if (p.logits) p.logits[((long long)seq * p.n + node) * p.max_ids + r0 + j] = z;
      }
    }
    __syncthreads();  // sp free for the next round
    if (tid == 0 && r0 == 0 && (int)blockIdx.x == seq * p.n + node) trace_mark(p.trace, 11);  // summed
    sort8(key, gid);
    const uint2 c = warp_select<kFinRows>(key, gid, k);
    if (tid == 0 && r0 == 0 && (int)blockIdx.x == seq * p.n + node) trace_mark(p.trace, 12);  // warp top-k
    if (r0 == 0) {
      run = c;
    } else {  // merge the round's list into the running one (two sorted entries per lane)
      uint32_t mk[2] = {run.x, c.x}, mg[2] = {run.y, c.y};
      cx(mk[0], mg[0], mk[1], mg[1]);
      run = warp_select<2>(mk, mg, k);
    }
  }
  // lse: warp, then block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, tm, o), e2 = __shfl_xor_sync(0xffffffffu, te, o);
    lse_fold(tm, te, m2, e2);
  }
  if (lane < k) wl[warp * k + lane] = run;
  if (lane == 0) wm[warp] = make_float2(tm, te);
  __syncthreads();
  if (tid == 0 && (int)blockIdx.x == seq * p.n + node) trace_mark(p.trace, 13);  // lists in smem
  if (warp == 0) {
    // merge the kWarps sorted lists: lane t holds list t's head
    int hp = 0;
    uint32_t hk[1], hg[1];
    hk[0] = lane < kWarps ? wl[lane * k].x : 0u;
    hg[0] = lane < kWarps ? wl[lane * k].y : 0xffffffffu;
    uint2 mine = make_uint2(0u, 0xffffffffu);
    for (int r = 0; r < k; ++r) {
      const uint32_t wk = __reduce_max_sync(0xffffffffu, hk[0]);
      if (wk == 0u) break;
      const uint32_t wg = __reduce_min_sync(0xffffffffu, hk[0] == wk ? hg[0] : 0xffffffffu);
      if (lane == r) mine = make_uint2(wk, wg);
      if (hk[0] == wk && hg[0] == wg) {
        ++hp;
        const uint2 nx = hp < k ? wl[lane * k + hp] : make_uint2(0u, 0xffffffffu);
        hk[0] = nx.x; hg[0] = nx.y;
      }
    }
    float bm = -INFINITY, be = 0.f;
    if (lane < kWarps) { bm = wm[lane].x; be = wm[lane].y; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, bm, o), e2 = __shfl_xor_sync(0xffffffffu, be, o);
      lse_fold(bm, be, m2, e2);
    }
    const long long ob = ((long long)seq * p.n + node) * k;
    if (lane < k) {
      a.topk_logit[ob + lane] = mine.x ? key_value(mine.x) : -INFINITY;
      a.topk_id[ob + lane] = mine.x ? (int32_t)mine.y : -1;
    }
    if (a.lse && lane == 0) a.lse[(long long)seq * p.n + node] = bm == -INFINITY ? -INFINITY : bm + logf(be);
  }
  __syncthreads();  // wl / wm free for the next pair
}

// ranked by counting.  Returns this lane's entry of the sorted top-k.
__device__ __forceinline__ uint2 warp_topk_thr(const uint32_t (&key)[4], const uint32_t (&gid)[4], int k,
                                               uint2* scratch) {
  const int lane = threadIdx.x & 31;
  uint32_t lmk = 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i) lmk = key[i] > lmk ? key[i] : lmk;
  const uint32_t T = warp_kth_key(lmk, k);
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool c = key[i] != 0u && key[i] >= T;
    const unsigned bal = __ballot_sync(0xffffffffu, c);
    if (c) scratch[cnt + __popc(bal & ((1u << lane) - 1u))] = make_uint2(key[i], gid[i]);
    cnt += __popc(bal);
  }
  uint2* best = scratch + kBM;
  if (lane < k) best[lane] = make_uint2(0u, 0xffffffffu);
  __syncwarp();
  warp_rank_write(scratch, cnt, k, best);
  __syncwarp();
  const uint2 r = lane < k ? best[lane] : make_uint2(0u, 0xffffffffu);
  __syncwarp();
  return r;
}

// ---------------------------------------------------------------- poll mode
// Level 1 for one (tile, node), one warp: wait for the S encoded partials of
// the node's 128 rows (4 per lane), sum them in split order, zero them, then
// the tile's sorted top-k (sort 4 per lane, k rounds of a warp arg-max) and
// (max, sum exp); publishes k encoded (key, id) entries + the lse partial.
// Cluster mode: the partials are the S cluster CTAs' shared-memory tiles
// Pm[node][128] (read over DSMEM); the list is published with plain stores
// (the caller's release atomic orders them).
template <bool kPollMode>
__device__ void level1(const TcArgs& a, int tile, int node, const int32_t* ids_s, int rows, int row0,
                       const float* Pm, uint2* scratch, uint32_t stale4 = 0u) {
  const HeadProblem& p = a.p;
  const int lane = threadIdx.x & 31;
  const int S = a.S, k = a.k;
  const long long sstride = (long long)p.n * kBM;  // floats between splits
  float* src = a.part + ((long long)tile * S * p.n + node) * kBM + 4 * lane;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  if (!kPollMode) {
    const uint32_t la = smem_u32(Pm + node * kBM + 4 * lane);
    float4 x[kMaxCluster];  // all S partials in flight at once (one DSMEM round trip)
#pragma unroll
    for (int j = 0; j < kMaxCluster; ++j)  // K chunk j of this tile was computed by cluster rank (j - tile) mod S
      if (j < S) x[j] = ld_dsmem_v4(mapa_shared(la, (uint32_t)((j + S - tile % S) % S)));
#pragma unroll
    for (int j = 0; j < kMaxCluster; ++j)
      if (j < S) { v[0] += x[j].x; v[1] += x[j].y; v[2] += x[j].z; v[3] += x[j].w; }  // K-chunk order
  }
  for (int s0 = 0; kPollMode && s0 < S; s0 += 8) {
    uint4 x[8];
    long long spins = 0;
    while (true) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (s0 + j < S) {
          x[j] = ld_relaxed_v4(src + (s0 + j) * sstride);
          ok = ok && x[j].x && x[j].y && x[j].z && x[j].w;
        }
      if (__all_sync(0xffffffffu, ok)) break;
      if (++spins > kSpinLimit) __trap();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (s0 + j < S) {  // split order
        v[0] += __uint_as_float(x[j].x ^ kEncF);
        v[1] += __uint_as_float(x[j].y ^ kEncF);
        v[2] += __uint_as_float(x[j].z ^ kEncF);
        v[3] += __uint_as_float(x[j].w ^ kEncF);
        *reinterpret_cast<uint4*>(src + (s0 + j) * sstride) = make_uint4(0u, 0u, 0u, 0u);
      }
  }
  const int r0 = 4 * lane;
  uint32_t key[4], gid[4];
  if (!kPollMode) {
    // lse partial + threshold selection written straight to the tile's list
    uint32_t lmk = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = r0 + i < rows && !((stale4 >> i) & 1u);  // fused step: rows whose id left I
      key[i] = ok ? float_key(v[i]) : 0u;
      gid[i] = ok ? (uint32_t)ids_s[r0 + i] : 0xffffffffu;
      lmk = key[i] > lmk ? key[i] : lmk;
      if (ok && p.logits) p.logits[((long long)(tile / a.tps) * p.n + node) * p.max_ids + row0 + r0 + i] = v[i];
    }
    const float M = key_value(__reduce_max_sync(0xffffffffu, lmk));
    float es = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (key[i]) es += __expf(v[i] - M);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
    uint2* out = a.cand + ((long long)tile * p.n + node) * (k + 1);
    if (a.l2poll) {  // one encoded store per entry: a poller never sees a half-written list
      const uint2 mine = warp_topk_thr(key, gid, k, scratch);
      if (lane < k) st_relaxed_v2(out + lane, make_uint2(mine.x ^ kEncK, mine.y ^ kEncG));
      if (lane == 0) st_relaxed_v2(out + k, make_uint2(__float_as_uint(M) ^ kEncF, __float_as_uint(es) ^ kEncF));
      return;
    }
    const uint32_t T = warp_kth_key(lmk, k);
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool c = key[i] != 0u && key[i] >= T;
      const unsigned bal = __ballot_sync(0xffffffffu, c);
      if (c) scratch[cnt + __popc(bal & ((1u << lane) - 1u))] = make_uint2(key[i], gid[i]);
      cnt += __popc(bal);
    }
    if (lane < k) out[lane] = make_uint2(0u, 0xffffffffu);  // padding when rows < k
    if (lane == 0) out[k] = make_uint2(__float_as_uint(M), __float_as_uint(es));
    __syncwarp();
    warp_rank_write(scratch, cnt, k, out);
    return;
  }
  float mloc = -INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool ok = r0 + i < rows;
    key[i] = ok ? float_key(v[i]) : 0u;
    gid[i] = ok ? (uint32_t)ids_s[r0 + i] : 0xffffffffu;
    if (ok) mloc = fmaxf(mloc, v[i]);
    if (ok && p.logits) {
      const int seq = tile / a.tps;
      p.logits[((long long)seq * p.n + node) * p.max_ids + row0 + r0 + i] = v[i];
    }
  }
  // lse partial of the tile's valid rows
  float M = mloc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float es = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (key[i]) es += __expf(v[i] - M);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
  uint2 mine;
  if (kPollMode) {
    cx(key[0], gid[0], key[1], gid[1]);
    cx(key[2], gid[2], key[3], gid[3]);
    cx(key[0], gid[0], key[2], gid[2]);
    cx(key[1], gid[1], key[3], gid[3]);
    cx(key[1], gid[1], key[2], gid[2]);
    mine = warp_select<4>(key, gid, k);
  } else {
    mine = warp_topk_thr(key, gid, k, scratch);
  }
  uint2* out = a.cand + ((long long)tile * p.n + node) * (k + 1);
  if (kPollMode) {
    if (lane < k) st_relaxed_v2(out + lane, make_uint2(mine.x ^ kEncK, mine.y ^ kEncG));
    if (lane == 0) st_relaxed_v2(out + k, make_uint2(__float_as_uint(M) ^ kEncF, __float_as_uint(es) ^ kEncF));
  } else {
    if (lane < k) out[lane] = mine;
    if (lane == 0) out[k] = make_uint2(__float_as_uint(M), __float_as_uint(es));
  }
}

// Level 2 for one (sequence, node), one warp: wait for the ntiles encoded
// lists, stage them (decoded) in the warp's shared scratch, zero them, merge by
// k rounds of a warp arg-max over the list heads (lane t owns lists t, t+32,
// ...), combine the lse partials, write the outputs.
// Cluster mode: the lists are complete (acquired by the caller): plain loads.
template <int kPer, bool kPollMode>  // lists per lane (ntiles <= 32 * kPer)
__device__ void level2(const TcArgs& a, int seq, int node, int ntiles, uint2* scratch) {
  const HeadProblem& p = a.p;
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const int kl = k + 1;
  float bm = -INFINITY, be = 0.f;
  for (int t = lane; t < ntiles; t += 32) {
    uint2* src = a.cand + ((long long)(seq * a.tps + t) * p.n + node) * kl;
    uint2* dst = scratch + t * kl;
    for (int j0 = 0; !kPollMode && j0 < kl; j0 += 8) {
      uint2 e[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < kl) e[j] = __ldcg(src + j0 + j);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < kl) dst[j0 + j] = e[j];
    }
    for (int j0 = 0; kPollMode && j0 < kl; j0 += 8) {
      uint2 e[8];
      long long spins = 0;
      while (true) {
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < kl) {
            e[j] = ld_relaxed_v2(src + j0 + j);
            ok = ok && e[j].x && e[j].y;
          }
        if (ok) break;
        if (++spins > kSpinLimit) __trap();
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < kl) {
          dst[j0 + j] = j0 + j < k ? make_uint2(e[j].x ^ kEncK, e[j].y ^ kEncG) : make_uint2(e[j].x ^ kEncF, e[j].y ^ kEncF);
          src[j0 + j] = make_uint2(0u, 0u);
        }
    }
    const float2 st = make_float2(__uint_as_float(dst[k].x), __uint_as_float(dst[k].y));
    lse_fold(bm, be, st.x, st.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, bm, o), e2 = __shfl_xor_sync(0xffffffffu, be, o);
    lse_fold(bm, be, m2, e2);
  }
  __syncwarp();
  if (threadIdx.x == 0) trace_mark(p.trace, 12);  // warp 0: lists staged
  int hp[kPer];
  uint32_t hk[kPer], hg[kPer];
#pragma unroll
  for (int c = 0; c < kPer; ++c) {
    const int t = lane + 32 * c;
    hp[c] = 0;
    hk[c] = t < ntiles ? scratch[t * kl].x : 0u;
    hg[c] = t < ntiles ? scratch[t * kl].y : 0xffffffffu;
  }
  uint2 mine = make_uint2(0u, 0xffffffffu);
  for (int r = 0; r < k; ++r) {
    // this lane's best head
    uint32_t lk = 0u, lg = 0xffffffffu;
#pragma unroll
    for (int c = 0; c < kPer; ++c)
      if (key_before(hk[c], hg[c], lk, lg)) { lk = hk[c]; lg = hg[c]; }
    const uint32_t wk = __reduce_max_sync(0xffffffffu, lk);
    if (wk == 0u) break;
    const uint32_t wg = __reduce_min_sync(0xffffffffu, lk == wk ? lg : 0xffffffffu);
    if (lane == r) mine = make_uint2(wk, wg);
#pragma unroll
    for (int c = 0; c < kPer; ++c)
      if (hk[c] == wk && hg[c] == wg) {
        const int t = lane + 32 * c;
        ++hp[c];
        const uint2 nx = hp[c] < k ? scratch[t * kl + hp[c]] : make_uint2(0u, 0xffffffffu);
        hk[c] = nx.x; hg[c] = nx.y;
      }
  }
  const long long ob = ((long long)seq * p.n + node) * k;
  if (lane < k) {
    a.topk_logit[ob + lane] = mine.x ? key_value(mine.x) : -INFINITY;
    a.topk_id[ob + lane] = mine.x ? (int32_t)mine.y : -1;
  }
  if (a.lse && lane == 0) a.lse[(long long)seq * p.n + node] = bm == -INFINITY ? -INFINITY : bm + logf(be);
}

// Poll-mode tail of the CTA that owns unit (tile, split): level 1 for nodes
// split, split + S, ... (one warp each); the tile-0 CTAs then run level 2 for
// the same nodes.
__device__ void poll_tail(const TcArgs& a, int tile, int split, const int32_t* ids_s, int m, uint2* smem,
                          int smem_bytes) {
  const HeadProblem& p = a.p;
  const int warp = threadIdx.x >> 5;
  const int S = a.S;
  const int seq = tile / a.tps, tin = tile - seq * a.tps;
  const int row0 = tin * kBM;
  const int rows = min(kBM, m - row0);
  const int ntiles = (m + kBM - 1) / kBM;
  for (int c = split + S * warp; c < p.n; c += S * kWarps) level1<true>(a, tile, c, ids_s, rows, row0, nullptr, nullptr);
  if (threadIdx.x == 0) trace_mark(p.trace, 10);  // warp 0: level 1 published
  if (p.trace && (threadIdx.x & 31) == 0)  // last warp of the CTA to publish
    atomicMax(&p.trace[(long long)blockIdx.x * kTraceSlots + 13], globaltimer());
  if (tin != 0) return;
  uint2* scratch = smem + (long long)warp * (smem_bytes / 8 / kWarps);
  for (int c = split + S * warp; c < p.n; c += S * kWarps) {
    if (ntiles <= 32) level2<1, true>(a, seq, c, ntiles, scratch);
    else if (ntiles <= 64) level2<2, true>(a, seq, c, ntiles, scratch);
    else level2<kMaxL2Lists / 32, true>(a, seq, c, ntiles, scratch);
  }
  if (threadIdx.x == 0) trace_mark(p.trace, 11);  // warp 0: level 2 written
}

// Level 2 (cluster mode, lists complete) for ntiles <= 32, one global round
// trip: lane t copies list t (k entries + its lse partial) into the warp's
// scratch with 8-byte cp.async; T = k-th largest head (k lists each own an
// entry >= T, so every top-k entry is >= T); each lane's sorted prefix >= T is
// compacted (warp scan) and the candidates are ranked by counting.  Scratch:
// ntiles * (2k + 1) + k entries.  List t comes from tile t (t < nreg), else
// from tile treg + t - nreg (the fused step's patch tiles).
__device__ void level2_thr(const TcArgs& a, int seq, int node, int ntiles, uint2* scratch, int nreg = 1 << 30,
                           int treg = 0) {
  const HeadProblem& p = a.p;
  const int lane = threadIdx.x & 31;
  const int k = a.k, kl = k + 1;
  const int lt = lane < nreg ? lane : treg + lane - nreg;
  uint2* mine = scratch + lane * kl;
  if (lane < ntiles) {
    const uint2* lst = a.cand + ((long long)(seq * a.tps + lt) * p.n + node) * kl;
    for (int j = 0; j < kl; ++j) cp_async8(smem_u32(mine + j), lst + j);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  uint2 head = make_uint2(0u, 0xffffffffu), st = make_uint2(__float_as_uint(-INFINITY), 0u);
  if (lane < ntiles) { head = mine[0]; st = mine[k]; }
  float bm = __uint_as_float(st.x), be = __uint_as_float(st.y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, bm, o), e2 = __shfl_xor_sync(0xffffffffu, be, o);
    lse_fold(bm, be, m2, e2);
  }
  const uint32_t T = ntiles >= k ? warp_kth_key(head.x, k) : 0u;
  int c = 0;  // this lane's qualifying prefix
  if (lane < ntiles)
    while (c < k && mine[c].x != 0u && mine[c].x >= T) ++c;
  int pre = c;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += y;
  }
  const int cnt = __shfl_sync(0xffffffffu, pre, 31);
  uint2* cand = scratch + ntiles * kl;
  for (int j = 0; j < c; ++j) cand[pre - c + j] = mine[j];
  uint2* best = cand + ntiles * k;
  if (lane < k) best[lane] = make_uint2(0u, 0xffffffffu);
  __syncwarp();
  warp_rank_write(cand, cnt, k, best);
  __syncwarp();
  const long long ob = ((long long)seq * p.n + node) * k;
  if (lane < k) {
    const uint2 r = best[lane];
    a.topk_logit[ob + lane] = r.x ? key_value(r.x) : -INFINITY;
    a.topk_id[ob + lane] = r.x ? (int32_t)r.y : -1;
  }
  if (a.lse && lane == 0) a.lse[(long long)seq * p.n + node] = bm == -INFINITY ? -INFINITY : bm + logf(be);
}

// Cluster-mode tail of the CTA (tile, split): after a cluster barrier, level 1
// for nodes split, split + S, ... (one warp each, partials over DSMEM); the
// warp whose list completes a node (per-node arrival counter, release/acquire)
// runs level 2 for it -- the last arriver finishes the node, nobody waits.
__device__ void cluster_tail(const TcArgs& a, int tile, int split, const int32_t* ids_s, int m, const float* Pm,
                             uint2* smem, int smem_bytes) {
  const HeadProblem& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const int seq = tile / a.tps, tin = tile - seq * a.tps;
  const int row0 = tin * kBM;
  const int rows = min(kBM, m - row0);
  const int ntiles = (m + kBM - 1) / kBM;
  cluster_sync();  // every CTA of the cluster has its partial tile in shared memory
  if (threadIdx.x == 0) trace_mark(p.trace, 5);
  // level-2 scratch: the part of the stage area above the partial tile
  const int pbytes = (p.n * kBM * 4 + 1023) / 1024 * 1024;
  uint2* scratch = smem + pbytes / 8 + (long long)warp * ((smem_bytes - pbytes) / 8 / kWarps);
  if (a.l2poll) {
    // lists handed over through L2 without fences: the tile-0 CTAs poll them
    for (int c = split + S * warp; c < p.n; c += S * kWarps) level1<false>(a, tile, c, ids_s, rows, row0, Pm, scratch);
    if (threadIdx.x == 0) trace_mark(p.trace, 10);
    cluster_sync();  // peers are done reading this CTA's partial tile
    if (tin == 0)
      for (int c = split + S * warp; c < p.n; c += S * kWarps) level2<1, true>(a, seq, c, ntiles, scratch);
    return;
  }
  for (int c = split + S * warp; c < p.n; c += S * kWarps) {
    level1<false>(a, tile, c, ids_s, rows, row0, Pm, scratch);
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
      last = atom_add_acq_rel(&a.node_ctr[seq * p.n + c], 1u) == (unsigned)(ntiles - 1);
      if (last) a.node_ctr[seq * p.n + c] = 0u;  // every tile has arrived: reset for the next launch
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) level2_thr(a, seq, c, ntiles, scratch);  // cluster mode: <= 32 tiles per sequence
  }
  if (threadIdx.x == 0) trace_mark(p.trace, 10);
  cluster_sync();  // peers are done reading this CTA's partial tile
}

// ---------------------------------------------------------------- fused step
// The update's hand-off to the head, run by every thread of the updating CTA
// between the count update and the slot-table writes: the stale-slot bitmap
// (pre-update slots whose id left I) and the entering ids go to scratch; once
// every other CTA has read the pre-update ids / n_active (arrive counter) the
// generation is bumped (release) and update_fast goes on to rewrite ids[].
struct FusedPublish {
  const TcArgs* a;
  uint32_t* stale_s;  // shared, w_max / 32 words
  __device__ void operator()(const StateView& sv, UpdSmem& sm, int n_old, int nl, int ne) const {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int words = (sv.w_max + 31) >> 5;
    for (int w = tid; w < words; w += nt) stale_s[w] = 0u;
    __syncthreads();
    for (int q = tid; q < nl; q += nt) atomicOr(&stale_s[sm.hole[q] >> 5], 1u << (sm.hole[q] & 31));
    __syncthreads();
    for (int w = tid; w < words; w += nt) a->stale[w] = stale_s[w];
    const int32_t gmul = sv.n_shards <= 1 ? 1 : sv.n_shards, gadd = sv.n_shards <= 1 ? 0 : sv.rank;
    for (int t = tid; t < ne; t += nt) a->enter_ids[t] = sm.enter[t] * gmul + gadd;
    if (tid == 0) { a->enter_meta[0] = ne; a->enter_meta[1] = n_old - nl + ne; a->enter_meta[2] = n_old; }
    __syncthreads();
    if (tid == 0) {
      long long spins = 0;
      trace_mark(a->p.trace, 13);  // updater: counts done, waiting for the readers
      while (ld_acquire(a->arrive_ctr) != gridDim.x - 1u)
        if (++spins > kSpinLimit) __trap();
      *a->arrive_ctr = 0u;  // every arrival of this launch is in
      __threadfence();
      red_add_release(a->step_ctr, 1u);
    }
    __syncthreads();
  }
};

__device__ __forceinline__ void wait_published(const TcArgs& a, unsigned g0) {
  if (threadIdx.x == 0) {
    long long spins = 0;
    while (ld_acquire(a.step_ctr) == g0)
      if (++spins > kSpinLimit) __trap();
  }
  __syncthreads();
}

// Distinct valid ids of the update lists (draft, then verify), first
// occurrence, computed identically by every patch CTA; ids_s[t] = the
// (base + t)-th of them.  Returns their count.  `sm`: 2 * kHashSlots +
// kFastThreads + 64 ints of scratch shared memory.
__device__ int fused_unique_ids(const TcArgs& a, int32_t* sm, int base, int32_t* ids_s) {
  int32_t* hkey = sm;
  int32_t* hval = sm + kHashSlots;
  int32_t* uniq = sm + 2 * kHashSlots;
  int* scan = reinterpret_cast<int*>(uniq + kFastThreads);
  const int tid = threadIdx.x;
  const StateView& sv = a.upd.sv;
  const int la = (int)a.upd.a.len, lb = (int)a.upd.b.len, L = la + lb;
  for (int h = tid; h < kHashSlots; h += blockDim.x) { hkey[h] = -1; hval[h] = 0x7fffffff; }
  int32_t e = -1;
  if (tid < la) e = a.upd.a.ptr[tid];
  else if (tid < L) e = a.upd.b.ptr[tid - la];
  __syncthreads();
  const bool valid = tid < L && e >= 0 && e < sv.vocab && is_local(sv, e);
  int hs = -1;
  if (valid) {
    hs = hash_insert(hkey, e);
    atomicMin(&hval[hs], tid);
  }
  __syncthreads();
  const bool keep = valid && hval[hs] == tid;
  int nu;
  const int pos = block_exclusive_scan(keep ? 1 : 0, scan, &nu);
  if (keep) uniq[pos] = e;
  __syncthreads();
  if (tid < kBM) ids_s[tid] = base + tid < nu ? uniq[base + tid] : 0;
  __syncthreads();
  return nu;
}


// Tail of a fused-step CTA (cluster mode), after the update has published:
// regular tiles drop the rows whose id left I (stale slots), patch tiles keep
// only the rows of ids entering I (a shared-memory hash of the published
// entering ids); level 2 merges the lists of the nreg live regular tiles and
// all n_patch patch tiles.  The last 8 KB of the stage area hold the hash.
__device__ void fused_tail(const TcArgs& a, int tile, int split, const int32_t* ids_s, int nu, const float* Pm,
                           uint2* smem, int smem_bytes, const uint32_t* stale_tile) {
  const HeadProblem& p = a.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const bool patch = tile >= a.tps_reg;
  const int m_old = __ldcg(&a.enter_meta[2]);
  const int nreg = (m_old + kBM - 1) / kBM;
  const int ntiles = nreg + a.n_patch;
  const int row0 = patch ? (tile - a.tps_reg) * kBM : tile * kBM;
  const int rows = min(kBM, (patch ? nu : m_old) - row0);
  const int hash_bytes = kHashSlots * 4;  // reserved at the end of the stage area (launcher accounting)
  // this lane's rows (4 * lane + i) that do not count: stale slots (regular
  // tiles) or ids already active before the update (patch tiles); the mask
  // was built by loader warp 15 during the stream (empty patch tiles: none)
  const uint32_t drop4 = rows > 0 ? (stale_tile[lane >> 3] >> ((lane & 7) * 4)) & 0xfu : 0u;
  cluster_sync();  // every CTA of the cluster has its partial tile in shared memory
  if (threadIdx.x == 0) trace_mark(p.trace, 5);
  const int pbytes = (p.n * kBM * 4 + 1023) / 1024 * 1024;
  uint2* scratch = smem + pbytes / 8 + (long long)warp * ((smem_bytes - hash_bytes - pbytes) / 8 / kWarps);
  for (int c = split + S * warp; c < p.n; c += S * kWarps) {
    level1<false>(a, tile, c, ids_s, rows, row0, Pm, scratch, drop4);
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
      last = atom_add_acq_rel(&a.node_ctr[c], 1u) == (unsigned)(ntiles - 1);
      if (last) a.node_ctr[c] = 0u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) level2_thr(a, 0, c, ntiles, scratch, nreg, a.tps_reg);
  }
  if (threadIdx.x == 0) trace_mark(p.trace, 10);
  cluster_sync();
}

template <int NT, int MODE>  // one instantiation per mode: only its own tail is compiled in
__global__ void __launch_bounds__(kThreads, 1) head_tc_kernel(TcArgs a) {
  // the persistent finisher mode processes two row tiles per unit: two MMAs per
  // K step share the hidden-state operand, so H crosses L2 half as often
  constexpr int UT = MODE == kModeFinishWide ? 2 : 1;
  using C = Cfg<NT, UT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned view that keeps the shared address space visible to the compiler
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStageArea);
  // bars[0..S) full, [S..2S) empty, [2S] tmem_full, [2S+1] tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 2);
  __shared__ int32_t ids_s[kBM * UT];   // the unit's row ids
  __shared__ int sh_m;

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int KB = p.d / kBK;
  const int S = a.S;

  if (tid == 0) trace_mark(p.trace, 0);  // start
  if (tid == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 14] = clock64();
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&bars[s]), kLoadWarps);        // full: one arrival per loader warp
      mbar_init(smem_u32(&bars[C::kStages + s]), 1);    // empty: one tcgen05.commit
    }
    mbar_init(smem_u32(&bars[2 * C::kStages]), 1);              // tmem_full
    mbar_init(smem_u32(&bars[2 * C::kStages + 1]), kLoadWarps);  // tmem_empty: one arrival per loader warp
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
  // the next kernel on the stream may be launched now (the fused step is
  // launched without PDL; its trigger below is inert)
  if (MODE != kModeFused) asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) trace_mark(p.trace, 1);  // dependency resolved
  // fused: the publication generation each CTA waits past; read before the
  // CTA arrives (the update publishes only after every arrival)
  __shared__ unsigned sh_g0;
  __shared__ uint32_t sh_stale[kBM / 32];  // fused, regular tile: rows whose id left I
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = make_idesc(kBM, NT);
  // Loader pattern: thread t moves 16-B chunk (t & 7) of tile rows lr and
  // lr + 64 (lr = t >> 3) of every W stage, and of H rows lr + 64 i < NT.
  const int lr = tid >> 3;
  const uint32_t swz = (uint32_t)(((tid & 7) ^ (lr & 7)) << 4);

  const int tiles_g = p.batch * a.tps;
  const int split = S > 1 ? (int)blockIdx.x % S : 0;
  const int first = S > 1 ? (int)blockIdx.x / S : (int)blockIdx.x;
  const int step = S > 1 ? tiles_g : (int)gridDim.x;
  int it = 0;      // pipeline iteration counter across units
  int local = 0;   // units processed by this CTA
  bool patch_rows = false;
  if (MODE == kModeFused && first == a.tps_reg + a.n_patch) {
    // the update cluster: CTA 0 applies the state update (its dependent global
    // round trips overlap the streaming of every other cluster), the others
    // just check in; none of them streams
    if (split == 0) {
      FusedPublish pub{&a, reinterpret_cast<uint32_t*>(smem + (sizeof(UpdSmem) + 255) / 256 * 256)};
      update_fast(a.upd, a.upd.seq0, *reinterpret_cast<UpdSmem*>(smem), pub, nullptr);
      if (tid == 0) trace_mark(p.trace, 11);  // updater: state updated and published
    } else if (tid == 0) {
      red_add_release(a.arrive_ctr, 1u);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kLoadWarps) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
    }
    return;
  }
  const int tpu = (a.tps + UT - 1) / UT;  // units per sequence
  const int units_g = UT == 1 ? tiles_g : p.batch * tpu;
  for (int unit = first; unit < units_g; unit += step) {
    const int seq = unit / tpu, t0 = (unit - seq * tpu) * UT;  // first tile of the unit within its sequence
    const int tile = seq * a.tps + t0;
    const int tin = t0;
    int row0 = tin * kBM;
    int m;
    if (MODE == kModeFused && tile >= a.tps_reg) {
      // patch tile p: rows [128p, 128p + 128) of the distinct valid ids of the
      // update lists (draft, then verify; first occurrence) -- a superset of the
      // ids entering I, known without waiting for the update; the rows of ids
      // that were already active are dropped at level 1
      if (tid == kLoaders) {  // the MMA warp: its release fence would stall a loader thread
        sh_g0 = ld_relaxed_u32(a.step_ctr);  // compared against later; the wait acquires
        red_add_release(a.arrive_ctr, 1u);
      }
      const int nu = fused_unique_ids(a, reinterpret_cast<int32_t*>(smem), (tile - a.tps_reg) * kBM, ids_s);
      row0 = (tile - a.tps_reg) * kBM;
      m = nu;
      if (tid == 0) sh_m = nu;
      patch_rows = true;
    } else {
      // one round trip: the tile's ids (rows past n_active are never dereferenced)
      // and n_active
      if (tid < kBM * UT)
        ids_s[tid] = row0 + tid < p.max_ids ? __ldcg(p.ids_base + (long long)seq * p.ids_stride + row0 + tid) : 0;
      if (tid == kBM * UT) sh_m = clamp_nact(p, seq);
      if (MODE == kModeFused && tid == kBM + 1) sh_g0 = ld_relaxed_u32(a.step_ctr);  // same round trip
      __syncthreads();
      // pre-update ids / n_active read: arrive from the MMA warp (its release
      // fence would stall a loader thread and with it the first stage)
      if (MODE == kModeFused && tid == kLoaders) red_add_release(a.arrive_ctr, 1u);
      m = sh_m;
    }
    if (tid == 0 && local == 0) trace_mark(p.trace, 7);  // ids + n_active in shared memory
    const int rows = min(kBM * UT, m - row0);  // rows of the unit (UT tiles)
    if (rows <= 0) {  // past n_active: every CTA of the tile skips it
      __syncthreads();
      if (MODE == kModeFused && patch_rows) local = -1;  // fused: the empty patch tile still publishes padding
      continue;
    }
    // K chunk of this CTA: cluster modes rotate the chunk by the tile, so at any
    // moment the 24 tiles' CTAs read S different slices of H instead of all
    // hitting the same L2 lines (the reduction sums in chunk order, so equal
    // rows in different tiles still give bit-equal logits)
    const int chunk = (MODE == kModeCluster || MODE == kModeFused) ? (split + tile) % S : split;
    const int kb0 = chunk * KB / S, kb1 = (chunk + 1) * KB / S;
    const int nk = kb1 - kb0;

    if (warp < kLoadWarps) {
      // ---------------- producers: gather rows of W_head + H into SW128 stages
      const uint16_t* rp[2 * UT];  // rows lr + 64 i (i < 2) of each of the UT tiles
#pragma unroll
      for (int i = 0; i < 2 * UT; ++i) {
        const int ur = (i >> 1) * kBM + lr + 64 * (i & 1);
        const int32_t g = ids_s[ur];
        const long long row = p.n_shards > 1 ? g / p.n_shards : g;
        rp[i] = (ur < rows) ? p.w + row * p.ldw + (tid & 7) * 8 : nullptr;
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
          for (int i = 0; i < 2 * UT; ++i)
            cp_async16(sA + (i >> 1) * (kBM * 128) + (lr + 64 * (i & 1)) * 128 + swz,
                       rp[i] ? (const void*)(rp[i] + kcol) : (const void*)p.w, rp[i] ? 16u : 0u);
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
          // this thread's copies of stage q - (kStages - 1) have landed; made
          // visible to the tensor core's async proxy; one arrival per warp
          // (512 per-thread shared-memory arrivals per stage were measurable)
          cp_async_wait<C::kStages - 1>();
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bars[(it + q - (C::kStages - 1)) % C::kStages]));
        }
      }
      if (tid == 0 && local == 0) trace_mark(p.trace, 3);  // all loads issued and landed
      if (MODE == kModeFused && warp == kLoadWarps - 1) {
        // while the last MMAs run: wait for the update's publication (long
        // done by now) and build this tile's drop mask -- regular tiles: the
        // stale-slot words; patch tiles: rows whose id is not in the entering
        // list (a warp-wide membership scan by shuffles)
        if (lane == 0) {
          long long spins = 0;
          while (ld_acquire(a.step_ctr) == sh_g0)
            if (++spins > kSpinLimit) __trap();
        }
        __syncwarp();
        if (!patch_rows) {
          if (lane < kBM / 32) sh_stale[lane] = __ldcg(&a.stale[(row0 >> 5) + lane]);
        } else {
          const int ne = __ldcg(&a.enter_meta[0]);
          int32_t mid[4];
          bool found[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) { mid[i] = ids_s[4 * lane + i]; found[i] = false; }
          for (int base = 0; base < ne; base += 64) {  // up to 64 entering ids per round trip
            const int32_t e0 = base + lane < ne ? __ldcg(&a.enter_ids[base + lane]) : -1;
            const int32_t e1 = base + 32 + lane < ne ? __ldcg(&a.enter_ids[base + 32 + lane]) : -1;
            for (int j = 0; j < 32; ++j) {
              const int32_t x0 = __shfl_sync(0xffffffffu, e0, j), x1 = __shfl_sync(0xffffffffu, e1, j);
#pragma unroll
              for (int i = 0; i < 4; ++i) found[i] = found[i] || x0 == mid[i] || x1 == mid[i];
            }
          }
          uint32_t nib = 0u;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (4 * lane + i < rows && !found[i]) nib |= 1u << i;
          uint32_t w = nib << ((lane & 7) * 4);
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
          if ((lane & 7) == 0) sh_stale[lane >> 3] = w;
        }
      }
      // ---------------- epilogue: TMEM -> registers -> this unit's slot of P
      mbar_wait(smem_u32(&bars[2 * C::kStages]), local & 1);
      tc_fence_after();
      if (tid == 0 && local == 0) trace_mark(p.trace, 4);  // last MMA done
      const int lg = warp & 3, cgp = warp >> 2;   // TMEM lane group, column group
      const int r = lg * 32 + lane;               // TMEM lane == tile row
      const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
      // per column, the 32 lanes of a warp store 128 consecutive bytes
#pragma unroll 1
      for (int h = 0; h < UT; ++h) {
      if (h > 0 && (t0 + h >= a.tps || row0 + h * kBM >= m)) break;  // the unit's second tile is empty
      float* Pw = (MODE == kModeCluster || MODE == kModeFused) ? reinterpret_cast<float*>(smem) + r
                                         : a.part + (((long long)(tile + h) * S + split) * p.n) * kBM + r;
      if (cgp < C::kColGroups) {
#pragma unroll 1
        for (int c0 = cgp * 16; c0 < NT && c0 < p.n; c0 += 16 * C::kColGroups) {
          float v[16];
          tmem_ld16(taddr + h * NT + c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < p.n) {
              if (MODE == kModePoll)  // strong store: visible to the polling CTAs without a fence
                st_relaxed_f32(Pw + (c0 + c) * kBM, __uint_as_float(__float_as_uint(v[c] == 0.f ? 0.f : v[c]) ^ kEncF));
              else
                Pw[(c0 + c) * kBM] = v[c];
            }
        }
      }
      }  // tiles of the unit
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars[2 * C::kStages + 1]));
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
        if (MODE == kModeCluster && lane == 0 && local == 0 && p.trace) {  // debug trace: stage readiness
          if (q == 0) trace_mark(p.trace, 11);
          if (q == nk / 2) trace_mark(p.trace, 12);
          if (q == nk - 1) trace_mark(p.trace, 13);
        }
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sB = sA + C::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
#pragma unroll
            for (int h = 0; h < UT; ++h)  // tile h of the unit into TMEM columns [h NT, (h + 1) NT)
              umma_bf16(tmem + h * NT, sw128_desc(sA + h * (kBM * 128) + kk * 32), sw128_desc(sB + kk * 32), idesc,
                        (q | kk) ? 1u : 0u);
          umma_commit(smem_u32(&bars[C::kStages + stage]));
          if (q == nk - 1) umma_commit(smem_u32(&bars[2 * C::kStages]));
        }
        __syncwarp();
      }
      // the MMA warp waits until the epilogue has drained TMEM
      mbar_wait(smem_u32(&bars[2 * C::kStages + 1]), local & 1);
    }
    it += nk;
    __syncthreads();  // ids_s free for the next unit
    ++local;
  }

  tc_fence_before();
  __syncthreads();  // every partial of this CTA is stored; TMEM drained
  if (warp == kLoadWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
  if (tid == 0) trace_mark(p.trace, 9);  // drained
  if (MODE == kModeFused) asm volatile("griddepcontrol.launch_dependents;");  // late trigger
  if (MODE == kModeFused) {
    if (local <= 0) wait_published(a, sh_g0);  // streaming CTAs: loader warp 15 already did
    if (tid == 0) trace_mark(p.trace, 12);  // publication seen
    if (local != 0)
      fused_tail(a, first, split, ids_s, local < 0 ? 0 : sh_m, reinterpret_cast<const float*>(smem),
                 reinterpret_cast<uint2*>(smem), C::kStageArea, sh_stale);
    if (tid == 0) trace_mark(p.trace, 8);  // done
    return;
  }
  if (MODE == kModeCluster) {
    if (local > 0)
      cluster_tail(a, first, split, ids_s, sh_m, reinterpret_cast<const float*>(smem), reinterpret_cast<uint2*>(smem),
                   C::kStageArea);
    if (tid == 0) trace_mark(p.trace, 8);  // done
    return;
  }
  if (MODE == kModePoll) {
    if (local > 0) poll_tail(a, first, split, ids_s, sh_m, reinterpret_cast<uint2*>(smem), C::kStageArea);
    if (tid == 0) trace_mark(p.trace, 8);  // done
    if (tid == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 15] = clock64();
    return;
  }
  // ---------------- grid arrival; finishers wait for the generation to change
  const int npairs = p.batch * p.n;
  const bool finisher = (int)blockIdx.x < npairs;
  __shared__ unsigned sh_gen;
  if (tid == 0) {
    const unsigned old = atom_add_acq_rel(a.grid_word, 1u);
    const unsigned cmask = (1u << kCountBits) - 1u;
    if ((old & cmask) == gridDim.x - 1u) red_add_release(a.grid_word, (1u << kCountBits) - gridDim.x);
    else if (finisher)
      while ((ld_acquire(a.grid_word) >> kCountBits) == (old >> kCountBits)) {}
  }
  if (!finisher) {
    if (tid == 0) trace_mark(p.trace, 8);  // done
    return;
  }
  __syncthreads();
  if (tid == 0) trace_mark(p.trace, 5);  // all partials visible
  // stage area: [0, kSpBytes) partial slices of a round, then the per-warp lists
  constexpr int kListBytes = kWarps * kMaxK * 8 + kWarps * 8;
  constexpr int kSpBytes = (C::kStageArea - kListBytes) / 1024 * 1024;
  int rr = kSpBytes / (4 * S) / kBM * kBM;
  if (rr > kThreads * kFinRows / kBM * kBM) rr = kThreads * kFinRows / kBM * kBM;
  float* sp = reinterpret_cast<float*>(smem);
  uint2* wl = reinterpret_cast<uint2*>(smem + kSpBytes);                         // [kWarps][k]
  float2* wm = reinterpret_cast<float2*>(smem + kSpBytes + kWarps * kMaxK * 8);  // [kWarps]
  for (int pr = blockIdx.x; pr < npairs; pr += gridDim.x) finish_node(a, pr / p.n, pr % p.n, sp, rr, wl, wm);
  if (tid == 0) trace_mark(p.trace, 8);  // done
  (void)sh_gen;
}

int g_head_mode = -1;  // -1 auto; kModeFinish / kModePoll / kModeCluster forced where feasible
int g_cluster_cap = 0;  // debug: largest cluster (K-split) size tried, 0 = kMaxCluster
// The fused step is launched WITHOUT programmatic dependent launch: its CTAs
// wait on each other across clusters (arrivals, publication), which needs the
// whole grid resident; an early-launched dependent grid places its clusters on
// the SMs this grid frees and can fragment the GPCs so that some of its own
// clusters cannot be placed while its placed CTAs wait for them (measured:
// graph of 200 back-to-back steps faulted with PDL, passes without).  The
// head-only kernels have no cross-cluster waits and keep PDL.
int g_fused_pdl = 0;  // (PDL with the trigger moved after the stream also faulted: kept off)

struct ScratchLayout {
  size_t grid_word, node_ctr, part, cand, step_ctr, arrive_ctr, stale, enter_ids, enter_meta, pcand, total;
};
constexpr int kMaxPatchTiles = kFastThreads / kBM;  // fused step: entering ids <= kFastThreads

// S * tiles_g <= kMaxSMs whenever S > 1, and S = 1 otherwise: the partial
// buffer holds max(kMaxSMs, tiles) tiles of n x 128 floats.
inline ScratchLayout scratch_layout(int batch, int max_ids, int n) {
  const size_t tiles = (size_t)batch * ((max_ids + kBM - 1) / kBM);
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  ScratchLayout L;
  size_t off = 0;
  L.grid_word = off; off += al(sizeof(unsigned));
  L.node_ctr = off;  off += al(sizeof(unsigned) * (size_t)batch * n);
  L.part = off;      off += al((tiles > (size_t)kMaxSMs ? tiles : (size_t)kMaxSMs) * n * kBM * sizeof(float));
  const size_t ctiles = (tiles < (size_t)kMaxSMs ? tiles : (size_t)kMaxSMs) + kMaxPatchTiles;
  L.cand = off;      off += al(ctiles * n * (kMaxK + 1) * sizeof(uint2));
  L.step_ctr = off;  off += al(sizeof(unsigned));
  L.arrive_ctr = off; off += al(sizeof(unsigned));
  L.stale = off;     off += al(sizeof(uint32_t) * (size_t)((max_ids + 31) / 32));
  L.enter_ids = off; off += al(sizeof(int32_t) * kFastThreads);
  L.enter_meta = off; off += al(sizeof(int) * 4);
  L.pcand = off;     off += al(pair_cand_bytes(n));  // head_pair.cu level-1 lists
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
        cudaFuncSetAttribute(head_tc_kernel<NT, kModeFinish>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(head_tc_kernel<NT, kModeFinishWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Cfg<NT, 2>::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(head_tc_kernel<NT, kModePoll>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(head_tc_kernel<NT, kModeCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const ScratchLayout L = scratch_layout(p.batch, p.max_ids, p.n);
  if (L.total > scratch_bytes) return cudaErrorInvalidValue;
  char* sc = (char*)scratch;
  TcArgs a;
  a.p = p;
  a.grid_word = (unsigned*)(sc + L.grid_word);
  a.part = (float*)(sc + L.part);
  a.cand = (uint2*)(sc + L.cand);
  a.node_ctr = (unsigned*)(sc + L.node_ctr);
  a.step_ctr = (unsigned*)(sc + L.step_ctr);
  a.arrive_ctr = (unsigned*)(sc + L.arrive_ctr);
  a.stale = (uint32_t*)(sc + L.stale);
  a.enter_ids = (int32_t*)(sc + L.enter_ids);
  a.enter_meta = (int*)(sc + L.enter_meta);
  a.tps_reg = 0;
  a.n_patch = 0;
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.k = k;
  a.tps = (p.max_ids + kBM - 1) / kBM;
  const int G = num_sms < kMaxSMs ? num_sms : kMaxSMs;
  const int tiles_g = p.batch * a.tps;
  const int KB = p.d / kBK;
  // Mode.  One unit per CTA (tiles_g <= #SMs): prefer clusters of S K-splits
  // per tile (the largest S <= 8 whose tiles_g clusters are all co-resident,
  // so the DSMEM reduction never waits for a second wave); else S = #SMs /
  // tiles_g with the L2 hand-off (poll mode); else persistent finishers.
  static int max_clusters[kMaxCluster + 1] = {0};
  const int env_mode = g_head_mode;  // debug override (nanospec_debug_set_head_mode), -1 = auto
  int S = 1, mode = kModeFinish;
  const long long warp_bytes = (C::kStageArea - p.n * kBM * 4 - 1024) / kWarps;  // level-2 scratch per warp
  if (tiles_g <= G && a.tps <= kMaxL2Lists && (long long)a.tps * (k + 1) * 8 <= warp_bytes) {
    const int smax = g_cluster_cap >= 2 && g_cluster_cap < kMaxCluster ? g_cluster_cap : kMaxCluster;
    const bool cl_ok = a.tps <= 32 && ((long long)a.tps * (2 * k + 1) + k) * 8 <= warp_bytes;
    for (int s = smax; s >= 2 && cl_ok && env_mode != kModePoll && env_mode != kModeFinish; --s) {
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
        if (cudaOccupancyMaxActiveClusters(&nc, head_tc_kernel<NT, kModeCluster>, &q) != cudaSuccess || nc <= 0) {
          (void)cudaGetLastError();
          nc = -1;
        }
        max_clusters[s] = nc;
      }
      if (max_clusters[s] >= tiles_g) { S = s; mode = kModeCluster; break; }
    }
    if (mode != kModeCluster && env_mode != kModeFinish) {
      S = G / tiles_g;
      if (S > KB) S = KB;
      if (S > kMaxSplit) S = kMaxSplit;
      mode = kModePoll;
    }
  }
  a.S = S;
  a.mode = mode;
  a.l2poll = (mode == kModeCluster && g_head_mode == 4) ? 1 : 0;

  cudaLaunchConfig_t cfg = {};
  // finisher mode: two tiles per unit once the tile capacity is at least twice
  // the SM count (halves the hidden-state traffic without starving SMs; the
  // host cannot see n_active, so the rule is on capacity)
  const bool wide = mode == kModeFinish && tiles_g >= 2 * G;
  const int units2 = p.batch * ((a.tps + 1) / 2);
  cfg.gridDim = dim3(mode != kModeFinish ? tiles_g * S : wide ? (units2 < G ? units2 : G) : (tiles_g < G ? tiles_g : G));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = wide ? Cfg<NT, 2>::kSmemBytes : C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  if (mode == kModeCluster) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = S;
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  auto kern = mode == kModeCluster ? head_tc_kernel<NT, kModeCluster>
              : mode == kModePoll  ? head_tc_kernel<NT, kModePoll>
                     : wide              ? head_tc_kernel<NT, kModeFinishWide>
                                         : head_tc_kernel<NT, kModeFinish>;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    cfg.attrs = attrs + 1;  // without PDL
    cfg.numAttrs = na - 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  return e;
}

// Fused step: the state update of one sequence (fast path) and its head in
// one launch.  Clusters of S K-split CTAs over the tps_reg row tiles of the
// pre-update slots plus P patch tiles for the entering ids; CTA 0 of the first
// patch cluster runs the update.  cudaErrorNotSupported when the clusters do
// not all fit in one wave (the caller then launches update + head).
template <int NT>
cudaError_t launch_step_nt(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit, int32_t* topk_id,
                           float* lse, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream,
                           bool dry_run) {
  using C = Cfg<NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(head_tc_kernel<NT, kModeFused>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const ScratchLayout L = scratch_layout(1, p.max_ids, p.n);
  if (!dry_run && L.total > scratch_bytes) return cudaErrorInvalidValue;
  const int G = num_sms < kMaxSMs ? num_sms : kMaxSMs;
  const int KB = p.d / kBK;
  const int tps_reg = (p.max_ids + kBM - 1) / kBM;
  const long long nl = upd.a.len + upd.b.len;
  const int P = nl <= 0 ? 1 : (int)((nl + kBM - 1) / kBM);  // patch tiles
  const int tiles_g = tps_reg + P + 1;                         // + the update cluster
  if (P > kMaxPatchTiles || tps_reg + P > 32 || tiles_g * 2 > G) return cudaErrorNotSupported;
  if ((long long)((sizeof(UpdSmem) + 255) / 256 * 256) + (p.max_ids + 31) / 32 * 4 > C::kStageArea)
    return cudaErrorNotSupported;
  const long long warp_entries = (C::kStageArea - kHashSlots * 4 - (p.n * kBM * 4 + 1023) / 1024 * 1024) / 8 / kWarps;
  if ((long long)(tps_reg + P) * (2 * k + 1) + k > warp_entries || warp_entries < 2 * kBM) return cudaErrorNotSupported;
  static int max_clusters[kMaxCluster + 1] = {0};
  int S = 0;
  const int smax = g_cluster_cap >= 2 && g_cluster_cap < kMaxCluster ? g_cluster_cap : kMaxCluster;
  for (int s = smax; s >= 2; --s) {
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
      if (cudaOccupancyMaxActiveClusters(&nc, head_tc_kernel<NT, kModeFused>, &q) != cudaSuccess || nc <= 0) {
        (void)cudaGetLastError();
        nc = -1;
      }
      max_clusters[s] = nc;
    }
    if (max_clusters[s] >= tiles_g) { S = s; break; }
  }
  if (S < 2) return cudaErrorNotSupported;
  if (dry_run) return cudaSuccess;
  char* sc = (char*)scratch;
  TcArgs a;
  a.p = p;
  a.grid_word = (unsigned*)(sc + L.grid_word);
  a.part = (float*)(sc + L.part);
  a.cand = (uint2*)(sc + L.cand);
  a.node_ctr = (unsigned*)(sc + L.node_ctr);
  a.step_ctr = (unsigned*)(sc + L.step_ctr);
  a.arrive_ctr = (unsigned*)(sc + L.arrive_ctr);
  a.stale = (uint32_t*)(sc + L.stale);
  a.enter_ids = (int32_t*)(sc + L.enter_ids);
  a.enter_meta = (int*)(sc + L.enter_meta);
  a.upd = upd;
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.k = k;
  a.tps = tiles_g;
  a.tps_reg = tps_reg;
  a.n_patch = P;
  a.l2poll = 0;
  a.S = S;
  a.mode = kModeFused;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles_g * S);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = S;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if (g_fused_pdl == 0) { cfg.attrs = attrs + 1; cfg.numAttrs = 1; }
  cudaError_t e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT, kModeFused>, a);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    cfg.attrs = attrs + 1;  // without PDL
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, head_tc_kernel<NT, kModeFused>, a);
  }
  return e;
}

}  // namespace

// The split head's scratch follows the older kernels' (whose counters must stay zero between launches).
size_t head_tc_scratch_bytes(int batch, int max_ids, int n) {
  return scratch_layout(batch, max_ids, n).total + head_split_scratch_bytes(batch, max_ids, n);
}

void set_head_tc_mode(int mode) { g_head_mode = mode; }
void set_head_tc_cluster_cap(int s) { g_cluster_cap = s; }

PairScratch pair_scratch(void* scratch, const ScratchLayout& L) {
  char* sc = (char*)scratch;
  PairScratch s;
  s.cand = (uint2*)(sc + L.pcand);
  s.node_ctr = (unsigned*)(sc + L.node_ctr);
  s.grid_word = (unsigned*)(sc + L.grid_word);
  s.step_ctr = (unsigned*)(sc + L.step_ctr);
  s.arrive_ctr = (unsigned*)(sc + L.arrive_ctr);
  s.stale = (uint32_t*)(sc + L.stale);
  s.enter_ids = (int32_t*)(sc + L.enter_ids);
  s.enter_meta = (int*)(sc + L.enter_meta);
  return s;
}

cudaError_t launch_step_tc(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit, int32_t* topk_id,
                           float* lse, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream,
                           bool dry_run) {
  if (g_head_mode == -1 || g_head_mode == kModeSplit) {  // default: the two-kernel head (head_split.cu)
    const size_t off = scratch_layout(1, p.max_ids, p.n).total;
    const cudaError_t e = launch_step_split(p, upd, k, topk_logit, topk_id, lse, dry_run ? nullptr : (char*)scratch + off,
                                            dry_run ? 0 : scratch_bytes - off, num_sms, stream, dry_run);
    if (e != cudaErrorNotSupported || g_head_mode == kModeSplit) return e;
  }
  if (g_head_mode == kModePair) {  // opt-in: the pair-split kernel (head_pair.cu)
    const ScratchLayout L = scratch_layout(1, p.max_ids, p.n);
    if (dry_run || L.total <= scratch_bytes) {
      const cudaError_t e = launch_step_pair(p, upd, k, topk_logit, topk_id, lse,
                                             dry_run ? PairScratch{} : pair_scratch(scratch, L), num_sms, stream,
                                             dry_run);
      return e;
    }
  }
  if (p.batch != 1 || p.d % kBK != 0 || p.n < 1 || p.n > 256 || p.ldw % 8 != 0 || k < 1 || k > kMaxK)
    return cudaErrorNotSupported;
#define NS_STEP(NTV) \
  launch_step_nt<NTV>(p, upd, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream, dry_run)
  if (p.n <= 16) return NS_STEP(16);
  if (p.n <= 32) return NS_STEP(32);
  if (p.n <= 64) return NS_STEP(64);
  if (p.n <= 128) return NS_STEP(128);
  return NS_STEP(256);
#undef NS_STEP
}

cudaError_t launch_step_split_only(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit,
                                   int32_t* topk_id, float* lse, void* scratch, size_t scratch_bytes, int num_sms,
                                   cudaStream_t stream) {
  const size_t off = scratch_layout(1, p.max_ids, p.n).total;
  if (off > scratch_bytes) return cudaErrorInvalidValue;
  return launch_step_split(p, upd, k, topk_logit, topk_id, lse, (char*)scratch + off, scratch_bytes - off, num_sms,
                           stream, false);
}

cudaError_t launch_head_tc(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                           void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream) {
  if (g_head_mode == -1 || g_head_mode == kModeSplit) {  // default: the two-kernel head (head_split.cu)
    const size_t off = scratch_layout(p.batch, p.max_ids, p.n).total;
    if (off > scratch_bytes) return cudaErrorInvalidValue;
    const cudaError_t e = launch_head_split(p, k, topk_logit, topk_id, lse, (char*)scratch + off, scratch_bytes - off,
                                            num_sms, stream);
    if (e != cudaErrorNotSupported || g_head_mode == kModeSplit) return e;
  }
  if (g_head_mode == kModePair) {  // opt-in: the pair-split kernel (head_pair.cu)
    const ScratchLayout L = scratch_layout(p.batch, p.max_ids, p.n);
    if (L.total > scratch_bytes) return cudaErrorInvalidValue;
    return launch_head_pair(p, k, topk_logit, topk_id, lse, pair_scratch(scratch, L), num_sms, stream);
  }
  if (p.d % kBK != 0 || p.n < 1 || p.n > 256 || p.ldw % 8 != 0 || k < 1 || k > kMaxK) return cudaErrorNotSupported;
  if (p.n <= 16) return launch_nt<16>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 32) return launch_nt<32>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 64) return launch_nt<64>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  if (p.n <= 128) return launch_nt<128>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
  return launch_nt<256>(p, k, topk_logit, topk_id, lse, scratch, scratch_bytes, num_sms, stream);
}

}  // namespace nanospec
