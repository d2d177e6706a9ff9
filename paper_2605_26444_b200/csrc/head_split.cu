// a3+a4+a5 (and, for nanospec_step, a2) as TWO kernels chained by
// programmatic dependent launch -- no CTA ever waits for another CTA of the
// head path, so no launch needs the whole grid resident:
//
//   z'[b][i][j] = sum_c W[row(ids_b[j])][c] * H[b][i][c]     (Eq. 2 on I)
//   then per (b, i) the top-k of z' by (value desc, id asc) + lse
//
// Kernel A (head_stream_kernel, 544 threads, one CTA per SM): the active rows
// of a sequence are cut into 128-row tiles; every tile is split along K over
// S CTAs (S = #SMs / #tiles: 6 at the headline, 24 tiles x 6 = 144 CTAs; S = 1
// and a persistent loop over tiles when the tiles outnumber the SMs).  A CTA
// gathers its tile's rows of W_head (16-byte cp.async straight from the
// [V x d] weight into 128B-swizzled shared memory: no repack buffer, the
// paper's P:247-258 design is prior art) and the hidden states' K slice,
// one lane issues tcgen05.mma (M = 128 rows, N = NT >= n nodes, K = 16) into
// TMEM, and the 16 loader warps drain the fp32 partial tile to L2 (one
// 128-byte store per node per warp).  It then exits: nothing in A waits for
// another CTA.
//
// Kernel B (one CTA per (sequence, node)) waits for A (griddepcontrol.wait:
// A complete, its stores visible) and sums every row's S partials in K-chunk
// order (one order for every tile: equal rows give bit-equal logits); a row
// counts only if it is in I.  head_select_tiles_kernel (<= 32 tiles: every
// head of one sequence up to |I| = 4096): warp w reduces tile w to its top-k
// list + (max, sum exp) (warp_topk4: threshold = k-th largest lane maximum by
// a bitonic sort over lanes, the few keys above it ranked by counting), then
// warp 0 merges the lists the same way and warp 1 folds the lse.
// head_select_kernel (more tiles): rounds of 32 tiles with a two-pass radix
// threshold.  Global ids come from the row-id table A wrote, so B never reads
// the state.
//
// List mode (split-K 1, more tiles than SMs: dp64, the dense [0, V) head, a
// 32k window): A gets 8 more warps.  The TMEM accumulator is double-buffered;
// while the loaders stream unit j + 1, the epilogue warps stage unit j's
// columns into shared memory and reduce every (tile, node) to its top-k list
// + (max, sum exp) (warp_topk4); the CTA's last unit is reduced by all its
// warps together once the stream is done.  head_merge_kernel then merges the
// per-tile lists of each (sequence, node): a few hundred candidates instead of
// |I| logits.
//
// Fused step (nanospec_step, one sequence): A streams a SUPERSET of the
// post-update active set that is known without waiting for the update -- the
// pre-update slots ids[0, n_old) plus the raw update-list entries as "patch"
// rows -- while its last CTA runs the O(changes) state update (state_fast.cuh).
// The update writes a drop bitmap (pre-update slots whose id left I; patch
// rows that are a repeat, invalid, or whose id was already active) and waits,
// one way only, until every streaming CTA has read the pre-update slots
// before it rewrites ids[] / pos[] / meta (the streaming CTAs never wait, so
// this cannot deadlock whatever the residency).  B then drops those rows.
// Result == update, then head.
#include <cuda.h>
#include <math.h>
#include <stdlib.h>

#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "state_fast.cuh"
#include "tc_ptx.cuh"

namespace nanospec {

namespace {

constexpr int kBM = 128;           // rows per tile (UMMA M)
constexpr int kBK = 64;            // K per stage: one 128-byte swizzle atom
constexpr int kLW = 16;            // loader / drain warps
constexpr int kLoaders = kLW * 32;
constexpr int kAThreads = kLoaders + 32;  // + the MMA-issue warp
constexpr int kBudget = 192 * 1024;
constexpr int kMaxS = 32;          // K splits per tile
constexpr int kMaxK = 32;
constexpr long long kSpin = 1ll << 30;  // updater's arrival poll bound (a trap beats a hung GPU)

// List mode (persistent split-K 1): kEW epilogue warps reduce every finished
// tile, straight from TMEM, to per-node top-k lists + lse partials while the
// loaders stream the next unit (the TMEM accumulator is double-buffered).
constexpr int kEW = 8;  // two per TMEM lane group: each stages half of a chunk's columns
constexpr int kAThreadsL = kAThreads + kEW * 32;
constexpr int kZCols = 64;                               // nodes per epilogue chunk
constexpr int kListExtra = kZCols * kBM * 4 /*Z*/ + 2 * kBM * 4 /*row ids*/ + kEW * kBM * 8 /*candidates*/;
constexpr int kListCap = 26000;                          // merge kernel: candidates per (sequence, node)

template <int NT, int AG = 1, int UT = 1, bool LIST = false>  // AG: 64-column K atoms per stage; UT: 128-row tiles per unit
struct ACfg {
  static constexpr int kAtomA = UT * kBM * kBK * 2;  // UT x 16 KB of W rows per atom
  static constexpr int kAtomB = NT * kBK * 2;     // NT x 128 B of H per atom
  static constexpr int kABytes = AG * kAtomA;
  static constexpr int kBBytes = AG * kAtomB;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBud = LIST ? 224 * 1024 - kListExtra - 2048 : kBudget;
  static constexpr int kStages = (kBud / kStageBytes) > 8 ? 8 : (kBud / kStageBytes);
  static constexpr int kTmemCols = (LIST ? 2 : 1) * UT * NT < 32 ? 32 : (LIST ? 2 : 1) * UT * NT;
  static constexpr int kStageArea = kStages * kStageBytes;
  static constexpr int kExtra = LIST ? kListExtra : 0;     // after the barriers: Z, row ids, candidates
  static constexpr int kSmemBytes = kStageArea + 1024 /*align*/ + 256 /*barriers*/ + kExtra;
  static constexpr int kColGroups = NT / 16 < 4 ? NT / 16 : 4;  // drain column groups
  static_assert(kStages >= 2, "at least two pipeline stages");
};

struct SplitArgs {
  HeadProblem p;
  float* part;          // [units][n][128] fp32 partial tiles
  int32_t* rowgid;      // [batch * (tps + n_patch)][128] global id of every streamed row (-1: none)
  int tps;              // regular tiles per sequence = ceil(max_ids / 128)
  int n_patch;          // fused step: patch tiles (raw update-list entries, 128 per tile)
  int ntiles;           // batch * tps + n_patch; global tile t: regular (t / tps, t % tps), then patch tiles
  int S, extra;         // K splits: tiles t < extra take S + 1, the others S (every SM busy)
  int ut;               // 128-row tiles per unit: 2 in the persistent split-K-1 mode (two MMAs share H)
  int upt;              // units per sequence when ut == 2: ceil(tps / 2)
  int units;            // sum of the tiles' splits
  int heads;            // streaming CTAs (the fused grid has one more: the updater)
  // fused step (batch 1)
  AppendArgs upd;
  int L;                // raw update-list entries (patch rows)
  unsigned* arrive_ctr; // streaming CTAs that have read the pre-update slots (the updater re-zeroes it)
  int* mrows;           // [batch] rows of the regular tiles (|I| as A read it), written by A's (tile 0, split 0) CTA
  uint32_t* drop;       // [(tps + n_patch) * 4] rows that do not count, written by the updater
  // outputs (B)
  float* topk_logit;    // [batch][n][k]
  int32_t* topk_id;
  float* lse;           // [batch][n] or null
  int k;
  int plain;            // 1: the stream kernel waits for the previous grid at its start (experiment flag 16384)
  long long list_stats; // list mode: byte offset (in part) of the [tiles][n] (M, sum exp) lse partials
  long long dbg_ld;     // debug logits: floats between the rows of one (sequence, node)
  int trace_base;       // debug trace: B's CTA b writes trace row trace_base + b (after A's rows)
};

// The kernel parameters live in the constant bank; their first reads miss the
// constant cache (an L2 round trip each, and the index math chains several).
// Touch every 64-byte line of the parameter block before waiting on the
// previous grid, so those misses overlap the wait.
__device__ __forceinline__ void warm_params(const SplitArgs& a) {
  constexpr int kLines = (int)((sizeof(SplitArgs) + 63) / 64);
  const int t = threadIdx.x;
  if (t < kLines) {
    const int v = reinterpret_cast<const int*>(&a)[t * 16];
    asm volatile("" ::"r"(v));
  }
}

__device__ __forceinline__ void trace_b(const SplitArgs& a, int e) {
  if (a.p.trace) a.p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + e] = globaltimer();
}

// Unit u -> (sequence, tile within the sequence, split, splits of the tile, unit of split 0).
struct Unit {
  int seq, tile, split, S, base;
};
// Splits and first unit of global tile t.
__device__ __forceinline__ void tile_units(const SplitArgs& a, int t, int& S, int& base) {
  if (t < a.extra) { S = a.S + 1; base = t * S; }
  else { S = a.S; base = a.extra * (a.S + 1) + (t - a.extra) * a.S; }
}
__device__ __forceinline__ int global_tile(const SplitArgs& a, int seq, int tile) {
  return tile < a.tps ? seq * a.tps + tile : a.p.batch * a.tps + (tile - a.tps);
}
__device__ __forceinline__ Unit unit_of(const SplitArgs& a, int u) {
  Unit r;
  const int hi = a.extra * (a.S + 1);
  int t;
  if (u < hi) {
    r.S = a.S + 1;
    t = u / r.S;
    r.split = u - t * r.S;
    r.base = t * r.S;
  } else {
    r.S = a.S;
    const int j = (u - hi) / a.S;
    t = a.extra + j;
    r.split = (u - hi) - j * a.S;
    r.base = hi + j * a.S;
  }
  const int treg = a.p.batch * a.tps;
  if (t < treg) {
    r.seq = t / a.tps;
    r.tile = t - r.seq * a.tps;
  } else {
    r.seq = 0;
    r.tile = a.tps + (t - treg);
  }
  return r;
}

// A unit with its K range: chunk (split + tile) mod S of the tile's K atoms
// (rotated, so the tiles read different slices of H at any moment).
struct UnitPlan {
  int seq, tile, split, S, base, kb0, nk;
};
__device__ __forceinline__ UnitPlan plan_unit(const SplitArgs& a, int u) {
  if (a.ut == 2) {  // two consecutive tiles of one sequence, full K (split-K 1)
    UnitPlan r;
    r.seq = u / a.upt;
    r.tile = 2 * (u - r.seq * a.upt);
    r.split = 0;
    r.S = 1;
    r.base = r.seq * a.tps + r.tile;
    r.kb0 = 0;
    r.nk = a.p.d / kBK;
    return r;
  }
  const Unit un = unit_of(a, u);
  UnitPlan r;
  r.seq = un.seq; r.tile = un.tile; r.split = un.split; r.S = un.S; r.base = un.base;
  const int KB = a.p.d / kBK;
  const int chunk = (un.split + un.tile) % un.S;
  r.kb0 = chunk * KB / un.S;
  r.nk = (chunk + 1) * KB / un.S - r.kb0;
  return r;
}

__device__ __forceinline__ int32_t list_entry(const AppendArgs& u, int e) {
  return e < (int)u.a.len ? u.a.ptr[e] : u.b.ptr[e - (int)u.a.len];
}

// ------------------------------------------------------------------ fused step: the update's hand-off
struct SplitPublish {
  const SplitArgs* a;
  uint32_t* words;  // shared: (tps + n_patch) * 4 drop words
  __device__ void operator()(const StateView& sv, UpdSmem& sm, int n_old, int nl, int ne) const {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nw = (a->tps + a->n_patch) * 4;
    const int L = a->L;
    const int32_t* list = sm.raw;  // the raw update lists, staged by update_fast in its first round trip
    // the streaming CTAs' arrivals (long complete by now): the acquire load is
    // issued here and checked after the drop bitmap, so its round trip overlaps
    unsigned arrived = 0u;
    if (tid == 0) arrived = ld_acquire(a->arrive_ctr);
    for (int w = tid; w < nw; w += nt) words[w] = 0u;
    __syncthreads();
    // pre-update slots whose id left I (the slot of every leaving id, hole[q])
    for (int q = tid; q < nl; q += nt) atomicOr(&words[sm.hole[q] >> 5], 1u << (sm.hole[q] & 31));
    // a patch row counts iff it is the first entry of its id, valid, on this
    // shard, and its id enters I
    for (int t = tid; t < L; t += nt) {  // no early exits: the shared-memory loads pipeline
      const int32_t g = list[t];
      const bool valid = g >= 0 && g < sv.vocab && is_local(sv, g);
      const int32_t lg = valid ? local_of(sv, g) : -1;
      bool dup = false, in = false;
#pragma unroll 8
      for (int q = 0; q < t; ++q) dup |= list[q] == g;
#pragma unroll 8
      for (int q = 0; q < ne; ++q) in |= sm.enter[q] == lg;
      if (!(valid && !dup && in)) atomicOr(&words[a->tps * 4 + (t >> 5)], 1u << (t & 31));
    }
    __syncthreads();
    for (int w = tid; w < nw; w += nt) a->drop[w] = words[w];
    if (tid == 0) {
      // every streaming CTA has read the pre-update slots / n_active: only
      // then may ids[], pos[] and meta change (one-way wait: the streaming
      // CTAs never wait, so they always get to arrive)
      long long spins = 0;
      while (arrived != (unsigned)a->heads) {
        arrived = ld_acquire(a->arrive_ctr);
        if (++spins > kSpin) __trap();
      }
      *a->arrive_ctr = 0u;  // visible to the next launch at this grid's completion
    }
    __syncthreads();
  }
};

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One warp, one (tile, node): the 128 logits zc[0, 128) of the tile's rows
// (lane owns rows lane + 32 j, id gid[j], -1 = not in I) ->
//   out[0, k)  the tile's top-k (key, id) by (value desc, id asc), padded with (0, -1)
//   *stat      (M, sum exp(z - M)) over the rows in I (M = -inf: none)
// Threshold T = the k-th largest lane maximum: k lanes own a key >= T, so every
// top-k key is >= T; the few keys >= T are staged in cs (<= 128 entries) and
// ranked by counting.
__device__ __forceinline__ void warp_topk4(const uint32_t (&key)[4], const int32_t (&gid)[4], int k, uint2* cs,
                                           uint2* out, float2* stat) {
  const int lane = threadIdx.x & 31;
  uint32_t lm = 0u;
#pragma unroll
  for (int j = 0; j < 4; ++j) lm = key[j] > lm ? key[j] : lm;
  // bitonic sort (ascending over lanes) of the lane maxima: lane 32 - k holds the k-th largest
  uint32_t v = lm;
#pragma unroll
  for (int sz = 2; sz <= 32; sz <<= 1)
#pragma unroll
    for (int st = sz >> 1; st > 0; st >>= 1) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v, st);
      const bool keep_min = ((lane & st) == 0) == ((lane & sz) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  const uint32_t T = __shfl_sync(0xffffffffu, v, 32 - k);  // 0 when fewer than k lanes hold a row
  const uint32_t mx = __shfl_sync(0xffffffffu, v, 31);
  const float M = key_value(mx);
  float es = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (key[j]) es += __expf(key_value(key[j]) - M);
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool in = key[j] != 0u && key[j] >= T;
    const unsigned b = __ballot_sync(0xffffffffu, in);
    if (in) cs[cnt + __popc(b & ((1u << lane) - 1u))] = make_uint2(key[j], (uint32_t)gid[j]);
    cnt += __popc(b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
  __syncwarp();
  for (int q = lane; q < cnt; q += 32) {
    const uint2 me = cs[q];
    int rk = 0;
#pragma unroll 4
    for (int f = 0; f < cnt; ++f) {
      const uint2 o = cs[f];
      rk += key_before(o.x, o.y, me.x, me.y) ? 1 : 0;
    }
    if (rk < k) out[rk] = me;
  }
  for (int q = cnt + lane; q < k; q += 32) out[q] = make_uint2(0u, 0xffffffffu);
  if (lane == 0) *stat = make_float2(mx ? M : -INFINITY, es);
  __syncwarp();  // cs reused by the caller's next call
}

__device__ __forceinline__ void warp_tile_topk(const float* zc, const int32_t (&gid)[4], int k, uint2* cs, uint2* out,
                                               float2* stat, float* dbg) {
  const int lane = threadIdx.x & 31;
  uint32_t key[4];
  float zv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    zv[j] = zc[lane + 32 * j];
    key[j] = gid[j] >= 0 ? float_key(zv[j]) : 0u;
  }
  warp_topk4(key, gid, k, cs, out, stat);
  if (dbg) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (gid[j] >= 0) dbg[lane + 32 * j] = zv[j];
  }
}

__device__ __forceinline__ int unit_rows(const SplitArgs& a, const UnitPlan& un, int ut) {
  return min(kBM * ut, clamp_nact(a.p, un.seq) - un.tile * kBM);  // as the loaders compute it (non-fused)
}

// Per-CTA hand-off from the epilogue warps to the joint tail (list mode).
struct ListTail {
  int u, e;  // the CTA's last unit with rows and its index among those units (-1: none)
};

// ------------------------------------------------------------------ list-mode epilogue
// The kEW epilogue warps of a persistent split-K-1 stream kernel: for every
// unit this CTA streams (same order as the MMA warp) except its last one, wait
// for its TMEM buffer, stage each 64-node chunk of each 128-row tile into
// shared memory (node-major), release the buffer after its last read, and
// reduce every (tile, node) with warp_tile_topk into
//   list[seq][node][tile][0, k), stats[seq][node][tile] (a (sequence, node)
//   pair's lists are contiguous: the merge reads them coalesced, from HBM when
//   the weight stream has evicted them from L2).
// The CTA's last unit is left to the joint tail (every warp of the CTA, once
// the loaders and the MMA warp are done): its epilogue is the exposed part.
template <int NT, int UT>
__device__ __forceinline__ void list_epilogue(const SplitArgs& a, uint32_t tmem, uint64_t* tbars, float* Z,
                                              int32_t* gid_s, uint2* cand, ListTail* tail) {
  // tbars[2b] = tmem_full of buffer b, tbars[2b + 1] = its tmem_empty
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ew = warp - (kLW + 1), etid = tid - (kLW + 1) * 32;
  const int lg = warp & 3;  // TMEM lane group this warp may read
  const int k = a.k;
  uint2* cs = cand + ew * kBM;
  uint2* lists = reinterpret_cast<uint2*>(a.part);
  float2* stats = reinterpret_cast<float2*>(reinterpret_cast<char*>(a.part) + a.list_stats);
  int e = 0;
  int u = blockIdx.x;
  UnitPlan un = plan_unit(a, u < a.units ? u : 0);
  int rows = u < a.units ? unit_rows(a, un, UT) : 0;
  while (u < a.units && rows <= 0) {  // the first unit with rows
    u += a.heads;
    if (u < a.units) { un = plan_unit(a, u); rows = unit_rows(a, un, UT); }
  }
  while (u < a.units) {
    // the next unit with rows (none: this one is the CTA's last -> the joint tail)
    int u2 = u + a.heads, rows2 = 0;
    UnitPlan un2 = un;
    while (u2 < a.units) {
      un2 = plan_unit(a, u2);
      rows2 = unit_rows(a, un2, UT);
      if (rows2 > 0) break;
      u2 += a.heads;
    }
    if (u2 >= a.units) {
      if (etid == 0) { tail->u = u; tail->e = e; }
      return;
    }
    const int32_t* ids = p.ids_base + (long long)un.seq * p.ids_stride + un.tile * kBM;
    for (int r = etid; r < kBM * UT; r += kEW * 32) gid_s[r] = r < rows ? __ldcg(ids + r) : -1;
    const int tb = e & 1;
    mbar_wait(smem_u32(&tbars[2 * tb]), (e >> 1) & 1);
    tc_fence_after();
    const int nh = (rows + kBM - 1) / kBM;
    const int ncc = (p.n + kZCols - 1) / kZCols;
    for (int h = 0; h < nh; ++h) {
      const long long gt = (long long)un.seq * p.n * a.tps + un.tile + h;  // + node * tps: the (tile, node) slot
      for (int cc = 0; cc < ncc; ++cc) {
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + tb * UT * NT + h * NT + cc * kZCols;
        const int r = lg * 32 + lane;
#pragma unroll
        for (int c16 = 0; c16 < kZCols / 16; ++c16) {
          if (c16 % (kEW / 4) == ew / 4 && cc * kZCols + c16 * 16 < NT && cc * kZCols + c16 * 16 < p.n) {
            float v[16];
            tmem_ld16(taddr + c16 * 16, v);
#pragma unroll
            for (int c = 0; c < 16; ++c) Z[(c16 * 16 + c) * kBM + r] = v[c];
          }
        }
        if (h == nh - 1 && cc == ncc - 1) {  // the last read of this TMEM buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tbars[2 * tb + 1]));
        }
        named_sync(2, kEW * 32);  // Z (and, the first time, gid_s) complete
        int32_t gid[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) gid[j] = gid_s[h * kBM + lane + 32 * j];
        const int cn = min(kZCols, p.n - cc * kZCols);
        for (int c = ew; c < cn; c += kEW) {
          const int node = cc * kZCols + c;
          warp_tile_topk(Z + c * kBM, gid, k, cs, lists + (gt + (long long)node * a.tps) * k, stats + gt + (long long)node * a.tps,
                         p.logits ? p.logits + ((long long)un.seq * p.n + node) * a.dbg_ld + (un.tile + h) * kBM
                                  : nullptr);
        }
        named_sync(2, kEW * 32);  // Z free
      }
    }
    ++e;
    u = u2;
    un = un2;
    rows = rows2;
  }
  if (etid == 0) { tail->u = -1; tail->e = -1; }
}

// The joint tail (list mode): every warp of the CTA reduces the CTA's last
// unit -- the 16 loader warps stage each tile's TMEM columns into the (now
// idle) stage area, then all warps share its (tile, node) reductions.
template <int NT, int UT>
__device__ __forceinline__ void list_tail(const SplitArgs& a, uint32_t tmem, uint64_t* tbars, float* Zt,
                                          int32_t* gid_s, uint2* cand, const ListTail& tail) {
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kWarps = kAThreadsL / 32;
  const int k = a.k;
  uint2* lists = reinterpret_cast<uint2*>(a.part);
  float2* stats = reinterpret_cast<float2*>(reinterpret_cast<char*>(a.part) + a.list_stats);
  const UnitPlan un = plan_unit(a, tail.u);
  const int rows = unit_rows(a, un, UT);
  const int32_t* ids = p.ids_base + (long long)un.seq * p.ids_stride + un.tile * kBM;
  for (int r = tid; r < kBM * UT; r += kAThreadsL) gid_s[r] = r < rows ? __ldcg(ids + r) : -1;
  const int tb = tail.e & 1;
  mbar_wait(smem_u32(&tbars[2 * tb]), (tail.e >> 1) & 1);
  tc_fence_after();
  const int nh = (rows + kBM - 1) / kBM;
  for (int h = 0; h < nh; ++h) {
    const long long gt = (long long)un.seq * p.n * a.tps + un.tile + h;
    if (warp < kLW) {  // TMEM -> Zt[node][row]
      const int lg = warp & 3, cgp = warp >> 2;
      const int r = lg * 32 + lane;
      const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + tb * UT * NT + h * NT;
      for (int c0 = cgp * 16; c0 < NT && c0 < p.n; c0 += 64) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int c = 0; c < 16; ++c) Zt[(c0 + c) * kBM + r] = v[c];
      }
    }
    __syncthreads();
    int32_t gid[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) gid[j] = gid_s[h * kBM + lane + 32 * j];
    for (int node = warp; node < p.n; node += kWarps)
      warp_tile_topk(Zt + node * kBM, gid, k, cand + warp * kBM, lists + (gt + (long long)node * a.tps) * k,
                     stats + gt + (long long)node * a.tps,
                     p.logits ? p.logits + ((long long)un.seq * p.n + node) * a.dbg_ld + (un.tile + h) * kBM : nullptr);
    __syncthreads();
  }
}

// ------------------------------------------------------------------ kernel A
template <int NT, bool FUSED, int AG, int UT, bool LIST = false>
__global__ void __launch_bounds__(LIST ? kAThreadsL : kAThreads, 1) head_stream_kernel(const __grid_constant__ SplitArgs a) {
  using C = ACfg<NT, AG, UT, LIST>;
  constexpr int kRows = kBM * UT;  // rows per unit
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStageArea);
  // bars[0..St) full, [St..2St) empty, [2St] tmem_full, [2St+1] tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4);
  __shared__ int32_t ids_s[2][kBM * UT];  // the unit's row ids (double-buffered: the next unit's are prefetched)
  __shared__ int sh_m[2];
  __shared__ ListTail sh_tail;  // list mode: the CTA's last unit, left to the joint tail

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KB = p.d / kBK;
  if (tid == 0) trace_mark(p.trace, 0);
  if (tid == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 14] = clock64();
  if (tid == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&bars[s]), kLW);                // full: one arrival per loader warp
      mbar_init(smem_u32(&bars[C::kStages + s]), 1);     // empty: one tcgen05.commit
    }
    mbar_init(smem_u32(&bars[2 * C::kStages]), 1);       // tmem_full
    mbar_init(smem_u32(&bars[2 * C::kStages + 1]), LIST ? kEW : kLW); // tmem_empty: one arrival per drain warp
    if (LIST) {  // the second TMEM buffer's pair
      mbar_init(smem_u32(&bars[2 * C::kStages + 2]), 1);
      mbar_init(smem_u32(&bars[2 * C::kStages + 3]), kEW);
    }
    fence_proxy_async();
  }
  if (warp == kLW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  warm_params(a);
  // the first unit's plan (index math only) and a warm-up of the translation
  // and L2 line of its row ids (the first dependent round trip after the
  // wait); the state itself is read only after the wait
  UnitPlan cur = plan_unit(a, (int)blockIdx.x < a.units ? (int)blockIdx.x : 0);
  if ((int)blockIdx.x < a.units && tid < 4 && cur.tile < a.tps) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.ids_base + (long long)cur.seq * p.ids_stride + cur.tile * kBM + 32 * tid));
    if (tid == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.nact_base + (long long)cur.seq * p.nact_stride));
  }
  // The previous kernel on the stream is either not programmatic (this grid
  // then starts after it completed) or one of this library's select / merge
  // kernels, which trigger only after their own wait, i.e. once the stream
  // kernel before them -- the last writer of the state this grid reads -- has
  // completed (the state update kernel does not trigger early).  So the row
  // ids, the lists and the hidden states may be read right away; only the
  // scratch (row-id table, partial tiles, drop words), which that select
  // kernel may still be reading, waits for it: the streaming CTAs wait just
  // before their drain, the updater before it starts.  The stream of step
  // s + 1 overlaps the select kernel of step s.  (List mode keeps the plain
  // order: its epilogue writes from the first unit on.)
  if (LIST || a.plain) pdl_wait();
  // B (which waits for this grid to complete) may be scheduled now
  asm volatile("griddepcontrol.launch_dependents;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) trace_mark(p.trace, 1);

  if (LIST && warp > kLW) {
    // list mode: the epilogue warps (tmem_full / tmem_empty pairs: bars[2St], [2St+2] / [2St+1], [2St+3])
    uint8_t* ex = smem + C::kStageArea + 256;
    float* Z = reinterpret_cast<float*>(ex);
    int32_t* gid_s = reinterpret_cast<int32_t*>(ex + kZCols * kBM * 4);
    uint2* cand = reinterpret_cast<uint2*>(ex + kZCols * kBM * 4 + 2 * kBM * 4);
    list_epilogue<NT, UT>(a, tmem, bars + 2 * C::kStages, Z, gid_s, cand, &sh_tail);
  } else if (FUSED && (int)blockIdx.x == a.heads) {
    // the updater: a2 while every other CTA streams
    uint8_t* base = smem;
    UpdSmem& us = *reinterpret_cast<UpdSmem*>(base);
    uint32_t* words = reinterpret_cast<uint32_t*>(base + (sizeof(UpdSmem) + 255) / 256 * 256);
    SplitPublish pub{&a, words};
    pdl_wait();  // the previous select kernel has read the drop words; the state is then final
    update_fast(a.upd, a.upd.seq0, us, pub, p.trace);
    if (tid == 0) trace_mark(p.trace, 11);
  } else {
    constexpr uint32_t idesc = make_idesc(kBM, NT);
    const int lr = tid >> 3;  // loader: 16-B chunk (tid & 7) of rows lr and lr + 64
    const uint32_t swz = (uint32_t)(((tid & 7) ^ (lr & 7)) << 4);
    int it = 0, local = 0, nrun = 0;  // pipeline iterations, units visited, units streamed
    bool arrived = !FUSED;
    const int stride = a.heads;
    // ids of unit u into ids_s[buf]: one round trip (ids + n_active or the lists)
    auto fetch_ids = [&](const UnitPlan& un, int buf) {
      if (un.tile < a.tps) {
        const int row0 = un.tile * kBM;
        if (tid < kRows)
          ids_s[buf][tid] = row0 + tid < p.max_ids ? __ldcg(p.ids_base + (long long)un.seq * p.ids_stride + row0 + tid)
                                                   : -1;
        if (tid == kRows) sh_m[buf] = clamp_nact(p, un.seq) - row0;
      } else {  // patch rows: the raw update-list entries (invalid / foreign ids are not streamed)
        const int e = (un.tile - a.tps) * kBM + tid;
        if (tid < kBM) {
          int32_t g = e < a.L ? list_entry(a.upd, e) : -1;
          if (!(g >= 0 && g < a.upd.sv.vocab && is_local(a.upd.sv, g))) g = -1;
          ids_s[buf][tid] = g;
        }
        if (tid == kBM) sh_m[buf] = a.L - (un.tile - a.tps) * kBM;
      }
    };
    // loaders + MMA warp (the list-mode epilogue warps run their own loop)
    auto sync_lm = [] {
      if (LIST) named_sync(1, kAThreads);
      else __syncthreads();
    };
    if ((int)blockIdx.x < a.units) fetch_ids(cur, 0);
    sync_lm();
    if (tid == 0) trace_mark(p.trace, 7);
    if (tid == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 12] = clock64();
    for (int u = blockIdx.x; u < a.units; u += stride, ++local) {
      const int buf = local & 1;
      const UnitPlan un = cur;
      const int rows = min(kRows, sh_m[buf]);  // rows of this unit in the row list (<= 0: none)
      if (FUSED && !arrived && tid == kLoaders) {  // pre-update slots read (the MMA warp: no loader stalls)
        red_add_release(a.arrive_ctr, 1u);
        arrived = true;
      }
      const int un_next = u + stride;
      int32_t nx_id = -1;
      int nx_m = 0;
      bool nx = un_next < a.units;
      if (nx) {  // prefetch the next unit's ids into registers (lands during the stream)
        const UnitPlan n2 = plan_unit(a, un_next);
        cur = n2;
        if (n2.tile < a.tps) {
          const int row0 = n2.tile * kBM;
          if (tid < kRows && row0 + tid < p.max_ids) nx_id = __ldcg(p.ids_base + (long long)n2.seq * p.ids_stride + row0 + tid);
          if (tid == kRows) nx_m = clamp_nact(p, n2.seq) - row0;
        }
      }
      if (rows <= 0) {
        if (!LIST) {  // no rows: the row-id table still says so (after the previous select kernel)
          pdl_wait();
          if (un.split == 0 && un.tile == 0 && tid == kRows) a.mrows[un.seq] = sh_m[buf];
          if (un.split == 0 && tid < kRows && (un.tile >= a.tps || un.tile * kBM + tid < a.tps * kBM))
            a.rowgid[((long long)un.seq * (a.tps + a.n_patch) + un.tile) * kBM + tid] = -1;
        }
        if (nx) {
          if (tid < kRows) ids_s[buf ^ 1][tid] = nx_id;
          if (tid == kRows) sh_m[buf ^ 1] = nx_m;
        }
        sync_lm();
        continue;
      }
      const int kb0 = un.kb0, nk = un.nk;
      const int nst = (nk + AG - 1) / AG;  // pipeline stages of this unit
      if (warp < kLW) {
        // ---------------- loaders: rows of W_head + H into SW128 stages
        const uint16_t* rp[2 * UT];
#pragma unroll
        for (int i = 0; i < 2 * UT; ++i) {
          const int r = lr + 64 * i;
          const int32_t g = r < rows ? ids_s[buf][r] : -1;
          const long long row = p.n_shards > 1 ? g / p.n_shards : g;
          const uint16_t* base = p.packed ? p.packed + ((long long)un.seq * p.max_ids + un.tile * kBM + r) * p.ldp
                                          : p.w + row * p.ldw;  // repacked rows: contiguous slots
          rp[i] = g >= 0 ? base + (tid & 7) * 8 : nullptr;
        }
        const uint16_t* hp = p.h + (long long)un.seq * p.n * p.d + (tid & 7) * 8;
        if (tid == 0 && local == 0) trace_mark(p.trace, 2);
        if (tid == 0 && local == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 13] = clock64();
        for (int q = 0; q < nst + C::kStages - 1; ++q) {
          if (q < nst) {
            const int g_it = it + q;
            const int stage = g_it % C::kStages;
            if (g_it >= C::kStages) mbar_wait(smem_u32(&bars[C::kStages + stage]), ((g_it / C::kStages) - 1) & 1);
            const uint32_t sA = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t sB = sA + C::kABytes;
            // a row's AG atoms back to back: AG * 128 contiguous bytes per row per stage
#pragma unroll
            for (int i = 0; i < 2 * UT; ++i)
#pragma unroll
              for (int at = 0; at < AG; ++at) {
                const bool in = q * AG + at < nk;
                const int kcol = (kb0 + q * AG + at) * kBK;
                if (in)
                  cp_async16(sA + at * C::kAtomA + (lr + 64 * i) * 128 + swz,
                             rp[i] ? (const void*)(rp[i] + kcol) : (const void*)p.w, rp[i] ? 16u : 0u);
              }
#pragma unroll
            for (int at = 0; at < AG; ++at) {
              const int kcol = (kb0 + q * AG + at) * kBK;
              if (q * AG + at < nk) {
#pragma unroll
                for (int i = 0; i < (NT * 8 + kLoaders - 1) / kLoaders; ++i) {
                  const int hr = lr + 64 * i;
                  if (hr < NT)
                    cp_async16(sB + at * C::kAtomB + hr * 128 + swz,
                               hr < p.n ? (const void*)(hp + (long long)hr * p.d + kcol) : (const void*)p.h,
                               hr < p.n ? 16u : 0u);
                }
              }
            }
          }
          cp_async_commit();
          if (q >= C::kStages - 1) {
            cp_async_wait<C::kStages - 1>();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[(it + q - (C::kStages - 1)) % C::kStages]));
          }
        }
        if (tid == 0 && local == 0) trace_mark(p.trace, 3);
        if (LIST) {
          // the tile's row ids (split 0 only; rows past the list: -1) -- list mode waited at the start
          if (un.split == 0 && un.tile == 0 && tid == kRows) a.mrows[un.seq] = sh_m[buf];
          if (un.split == 0 && tid < kRows && (un.tile >= a.tps || un.tile * kBM + tid < a.tps * kBM))
            a.rowgid[((long long)un.seq * (a.tps + a.n_patch) + un.tile) * kBM + tid] = tid < rows ? ids_s[buf][tid] : -1;
        } else {
        // ---------------- the scratch: the previous select kernel has completed
        if (nrun == 0) pdl_wait();
        // the tile's row ids for B (split 0 only); rows past the list: -1
        if (un.split == 0 && un.tile == 0 && tid == kRows) a.mrows[un.seq] = sh_m[buf];
        if (un.split == 0 && tid < kRows && (un.tile >= a.tps || un.tile * kBM + tid < a.tps * kBM))
          a.rowgid[((long long)un.seq * (a.tps + a.n_patch) + un.tile) * kBM + tid] = tid < rows ? ids_s[buf][tid] : -1;
        if (tid == 0 && nrun == 0) trace_mark(p.trace, 1);
        // ---------------- drain: TMEM -> the unit's partial tile in L2
        mbar_wait(smem_u32(&bars[2 * C::kStages]), nrun & 1);
        tc_fence_after();
        if (tid == 0 && nrun == 0) trace_mark(p.trace, 4);
        const int lg = warp & 3, cgp = warp >> 2;
        const int r = lg * 32 + lane;  // TMEM lane == tile row
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
#pragma unroll
        for (int h = 0; h < UT; ++h) {  // tile h of the unit: TMEM columns [h NT, (h + 1) NT)
          if (UT > 1 && un.tile + h >= a.tps) break;
          float* Pw = a.part + ((long long)(un.base + un.split + h) * p.n) * kBM + r;
          if (cgp < C::kColGroups) {
#pragma unroll 1
            for (int c0 = cgp * 16; c0 < NT && c0 < p.n; c0 += 16 * C::kColGroups) {
              float v[16];
              tmem_ld16(taddr + h * NT + c0, v);
#pragma unroll
              for (int c = 0; c < 16; ++c)
                if (c0 + c < p.n) Pw[(c0 + c) * kBM] = v[c];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars[2 * C::kStages + 1]));
        }
      } else {
        // ---------------- MMA issue (warp 16, one lane)
        const int tb = LIST ? (nrun & 1) : 0;  // TMEM buffer (list mode: double-buffered)
        if (LIST) {
          if (nrun >= 2) {  // the epilogue has read this buffer's previous unit
            mbar_wait(smem_u32(&bars[2 * C::kStages + 2 * tb + 1]), ((nrun >> 1) - 1) & 1);
            tc_fence_after();
          }
        } else if (nrun > 0) {  // the previous unit's partial has left TMEM
          mbar_wait(smem_u32(&bars[2 * C::kStages + 1]), (nrun - 1) & 1);
          tc_fence_after();
        }
        for (int q = 0; q < nst; ++q) {
          const int g_it = it + q;
          const int stage = g_it % C::kStages;
          mbar_wait(smem_u32(&bars[stage]), (g_it / C::kStages) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sA = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t sB = sA + C::kABytes;
#pragma unroll
            for (int at = 0; at < AG; ++at)
              if (q * AG + at < nk) {
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
#pragma unroll
                  for (int h = 0; h < UT; ++h)  // the UT tiles share the H operand
                    umma_bf16(tmem + (tb * UT + h) * NT, sw128_desc(sA + at * C::kAtomA + h * (kBM * 128) + kk * 32),
                              sw128_desc(sB + at * C::kAtomB + kk * 32), idesc, (q | at | kk) ? 1u : 0u);
              }
            umma_commit(smem_u32(&bars[C::kStages + stage]));
            if (q == nst - 1) {
              umma_commit(smem_u32(&bars[2 * C::kStages + 2 * tb]));
              if (LIST) trace_mark(p.trace, 4);  // list mode: the last unit's last MMA issued
            }
          }
          __syncwarp();
        }
      }
      it += nst;
      ++nrun;
      if (nx) {
        if (tid < kRows) ids_s[buf ^ 1][tid] = nx_id;
        if (tid == kRows) sh_m[buf ^ 1] = nx_m;
      }
      sync_lm();  // ids_s[buf] free; the next unit's ids in ids_s[buf ^ 1]
    }
    if (FUSED && !arrived && tid == kLoaders) red_add_release(a.arrive_ctr, 1u);
  }
  if (LIST) {  // the joint tail: every warp reduces the CTA's last unit
    __syncthreads();
    const ListTail t = sh_tail;
    if (t.u >= 0) {
      uint8_t* ex = smem + C::kStageArea + 256;
      if (tid == 0) trace_mark(p.trace, 5);
      list_tail<NT, UT>(a, tmem, bars + 2 * C::kStages, reinterpret_cast<float*>(smem),
                        reinterpret_cast<int32_t*>(ex + kZCols * kBM * 4), reinterpret_cast<uint2*>(ex), t);
      if (tid == 0) trace_mark(p.trace, 6);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kLW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
  }
  if (tid == 0) trace_mark(p.trace, 9);
  if (tid == 0 && p.trace) p.trace[(long long)blockIdx.x * kTraceSlots + 15] = clock64();
}

// ------------------------------------------------------------------ kernel B
// One CTA (32 warps) per (sequence, node), in rounds of 32 tiles, one per warp
// (the headline is one round).  Tiles are visited in the order [regular tiles
// 0, tps) ++ [patch tiles]; a row counts iff its row id (written by A: -1 past
// the row list) is >= 0 and its drop bit is clear, so no state is read: every
// lane's loads -- the S partials of its 4 rows in K-chunk order, the row ids,
// the drop bits -- are in flight at once (one round trip).  Per round: logits
// and order keys; the threshold T = max(k-th key of the running top-k, the
// 16-bit prefix of the round's k-th largest key) by a two-pass radix select
// over shared-memory histograms (8 bits each: every thread adds its keys, one
// warp finds the bin) -- at least k round keys are >= T, so no round key below
// T is in the top-k; the few keys >= T (k plus the ties of a 16-bit prefix)
// are appended behind the running top-k and every candidate is ranked by
// counting by its own thread; lse = M + log sum exp(z - M) with M the block
// maximum (one exp per row), folded across rounds.  No sequential merge of
// lists anywhere.
constexpr int kBThreads = 1024;
constexpr int kBWarps = kBThreads / 32;
constexpr int kSmallBin = 96;                     // candidates a one-pass threshold may leave

// One warp, a 256-bin histogram: the largest bin b whose suffix count
// (bins >= b) reaches `need`, and how many keys are still needed inside it:
// (b, need - count(bins > b)); (0xffffffff, need) when the total is below need.
__device__ __forceinline__ uint2 radix_bin(const uint32_t* hist, uint32_t need) {
  const int lane = threadIdx.x & 31;
  uint32_t h[8], sum = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) { h[j] = hist[8 * lane + j]; sum += h[j]; }
  uint32_t suf = sum;  // inclusive suffix over lanes >= this one
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, suf, o);
    if (lane + o < 32) suf += y;
  }
  const unsigned ok = __ballot_sync(0xffffffffu, suf >= need && need > 0u);
  if (ok == 0u) return make_uint2(0xffffffffu, need);
  const int L = 31 - __clz(ok);  // the highest lane whose suffix reaches need
  const uint32_t above = __shfl_sync(0xffffffffu, suf - sum, L);  // keys in lanes > L
  uint32_t bin = 0u, rem = 0u;
  if (lane == L) {
    uint32_t acc = above;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      if (acc + h[j] >= need) { bin = 8u * lane + j; rem = need - acc; break; }
      acc += h[j];
    }
  }
  bin = __shfl_sync(0xffffffffu, bin, L);
  rem = __shfl_sync(0xffffffffu, rem, L);
  return make_uint2(bin, rem);
}

// NP (sequence, node) pairs per CTA, WP = 32 / NP warps each, TPW tiles per
// warp per round: <1, 1> for few pairs (the headline: 60 CTAs of one pair,
// 32 tiles a round), <4, 3> for many pairs whose tiles fit one round (dp64:
// 24 tiles per sequence, 3840 pairs -> 960 CTAs).  The pairs of a CTA run in
// lock step (the CTA's barriers); each pair has its own shared-memory slice.
template <int NP, int TPW>
struct BCfg {
  static constexpr int WP = kBWarps / NP;               // warps per pair
  static constexpr int kRound = WP * TPW;               // tiles per round
  static constexpr int kCandN = kMaxK + kRound * kBM;   // worst case: every row of a round ties at T
  static constexpr size_t kSmem = (size_t)NP * kCandN * 8;  // dynamic: the candidate arrays
};

template <int NP, int TPW, bool MR>  // MR: several rounds (the later ones may skip the radix passes)
__global__ void __launch_bounds__(kBThreads, 1) head_select_kernel(const __grid_constant__ SplitArgs a) {
  using C = BCfg<NP, TPW>;
  constexpr int WP = C::WP;
  extern __shared__ __align__(16) uint8_t bsm[];
  __shared__ uint2 res_all[NP][kMaxK];
  __shared__ uint32_t hist1_all[NP][256], hist2_all[NP][256];
  __shared__ uint32_t sh_wm_all[NP][WP];
  __shared__ float sh_es_all[NP][WP];
  __shared__ uint32_t sh_b1_all[NP], sh_need_all[NP], sh_T_all[NP];
  __shared__ int sh_cnt_all[NP];
  __shared__ float sh_M_all[NP], sh_E_all[NP];  // running lse: maximum and sum exp(z - maximum)
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pi = warp / WP, wq = warp - pi * WP, ptid = tid - pi * WP * 32;  // pair of the CTA, warp / thread in it
  uint2* cand = reinterpret_cast<uint2*>(bsm) + (size_t)pi * C::kCandN;  // [0, k): running top-k; then candidates
  uint2* res = res_all[pi];
  uint32_t* hist1 = hist1_all[pi];
  uint32_t* hist2 = hist2_all[pi];
  uint32_t* sh_wm = sh_wm_all[pi];
  float* sh_es = sh_es_all[pi];
  const int k = a.k;
  const int pair = blockIdx.x * NP + pi;
  const bool live_pair = pair < p.batch * p.n;
  const int seq = live_pair ? pair / p.n : 0, node = live_pair ? pair - seq * p.n : 0;
  const int ntp = a.tps + a.n_patch;
  const long long pst = (long long)p.n * kBM;
  const int r0 = 4 * lane;
  warm_params(a);
  if (ptid < kMaxK) cand[ptid] = make_uint2(0u, 0xffffffffu);
  if (ptid < 256) { hist1[ptid] = 0u; hist2[ptid] = 0u; }
  if (ptid == 0) { sh_cnt_all[pi] = 0; sh_M_all[pi] = -INFINITY; sh_E_all[pi] = 0.f; }
  if (tid == 0) trace_b(a, 0);
  // round 0's addresses (index math only) before the wait
  int S[TPW], base[TPW];
  bool on[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int tile = wq * TPW + j;
    on[j] = live_pair && tile < ntp;
    S[j] = 0;
    base[j] = 0;
    if (on[j]) tile_units(a, global_tile(a, seq, tile), S[j], base[j]);
    if (on[j] && lane == 0) {  // warm the translations / L2 lines while A still runs
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rowgid + ((long long)seq * ntp + tile) * kBM));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.part + (long long)base[j] * pst + (long long)node * kBM));
    }
  }
  pdl_wait();  // A complete: partials, row ids (and the fused step's drop bitmap) visible
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) trace_b(a, 1);
  if (tid == 0 && p.trace) {
    p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + 14] = clock64();
    p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + 12] = 0xB;  // a B row
  }
  int treg = a.tps;  // regular tiles holding rows (known after round 0; NP == 1 only: one round otherwise)
  for (int v0 = 0; v0 < ntp; v0 += C::kRound) {
    if (v0 > 0 && v0 >= treg && v0 + C::kRound <= a.tps) continue;  // a chunk of tiles past n_active
    uint32_t key[4 * TPW], gid[4 * TPW];  // the logit is key_value(key): no float copy kept
    uint32_t lm = 0u;
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int tile = v0 + wq * TPW + j;  // regular tiles [0, tps), then patch tiles
      if (v0 > 0) {
        on[j] = live_pair && tile < ntp && !(tile >= treg && tile < a.tps);
        S[j] = 0;
        base[j] = 0;
        if (on[j]) tile_units(a, global_tile(a, seq, tile), S[j], base[j]);
      }
      const int4 g4 = on[j] ? __ldcg(reinterpret_cast<const int4*>(a.rowgid + ((long long)seq * ntp + tile) * kBM) + lane)
                            : make_int4(-1, -1, -1, -1);
      const uint32_t dw = (on[j] && a.drop) ? __ldcg(&a.drop[tile * 4 + (lane >> 3)]) >> ((lane & 7) * 4) : 0u;
      float zz[4] = {0.f, 0.f, 0.f, 0.f};
      if (TPW > 1) {  // the many-pair layout runs with split-K 1: one partial per tile
        if (on[j] && S[j] == 1) {
          const float4 x = __ldcg(reinterpret_cast<const float4*>(a.part + (long long)base[j] * pst +
                                                                   (long long)node * kBM + r0));
          zz[0] = x.x; zz[1] = x.y; zz[2] = x.z; zz[3] = x.w;
        }
      } else {
        const float* src = a.part + (long long)base[j] * pst + (long long)node * kBM + r0;
        const int Sj = S[j], rot = Sj ? tile % Sj : 0;
        for (int c0 = 0; c0 < Sj; c0 += 8) {  // K chunk c was computed by split (c - tile) mod S
          float4 x[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < Sj) {
              int sp = c0 + q - rot;
              if (sp < 0) sp += Sj;
              x[q] = __ldcg(reinterpret_cast<const float4*>(src + (long long)sp * pst));
            }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < Sj) { zz[0] += x[q].x; zz[1] += x[q].y; zz[2] += x[q].z; zz[3] += x[q].w; }
        }
      }
      const int32_t g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool ok = g[i] >= 0 && !((dw >> i) & 1u);
        key[4 * j + i] = ok ? float_key(zz[i]) : 0u;
        gid[4 * j + i] = ok ? (uint32_t)g[i] : 0xffffffffu;
        lm = key[4 * j + i] > lm ? key[4 * j + i] : lm;
        if (g[i] >= 0 && p.logits) {
          const long long col = tile < a.tps ? (long long)tile * kBM + r0 + i
                                             : (long long)p.max_ids + (tile - a.tps) * kBM + r0 + i;
          p.logits[((long long)seq * p.n + node) * a.dbg_ld + col] = zz[i];
        }
      }
    }
    if (tid == 0 && v0 == 0) trace_b(a, 5);
    const uint32_t wm = __reduce_max_sync(0xffffffffu, lm);
    if (lane == 0) sh_wm[wq] = wm;
    if (MR && NP == 1 && v0 > 0) {
      // ---- a later round: when the top-k so far already prunes all but a few
      // keys (<= 4 keys on each of <= 32 threads), its k-th key is the
      // threshold and the radix passes are skipped
      const uint32_t Tk = res[k - 1].x;  // the top-k so far (stable since the previous round's last barrier)
      int q = 0;
#pragma unroll
      for (int i = 0; i < 4 * TPW; ++i) q |= (key[i] != 0u && key[i] >= Tk) ? 1 : 0;
      if (__syncthreads_count(q) <= 32) {  // also publishes the warp maxima
        const uint32_t Mk = __reduce_max_sync(0xffffffffu, lane < WP ? sh_wm[lane] : 0u);
        const float M = key_value(Mk);
        float es = 0.f;
#pragma unroll
        for (int i = 0; i < 4 * TPW; ++i)
          if (key[i]) es += __expf(key_value(key[i]) - M);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
        if (lane == 0) sh_es[wq] = es;
        if (ptid < k) res[ptid] = make_uint2(0u, 0xffffffffu);
        int c = 0;
#pragma unroll
        for (int i = 0; i < 4 * TPW; ++i) c += (key[i] != 0u && key[i] >= Tk) ? 1 : 0;
        if (__ballot_sync(0xffffffffu, c > 0)) {
          int pre = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
          }
          int wbase = 0;
          if (lane == 31) wbase = atomicAdd(&sh_cnt_all[pi], pre);
          wbase = __shfl_sync(0xffffffffu, wbase, 31);
          int o2 = k + wbase + pre - c;
#pragma unroll
          for (int i = 0; i < 4 * TPW; ++i)
            if (key[i] != 0u && key[i] >= Tk) cand[o2++] = make_uint2(key[i], gid[i]);
        }
        __syncthreads();  // candidates, lse partials
        if (wq == WP - 1) {
          float x = lane < WP ? sh_es[lane] : 0.f;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          if (lane == 0 && Mk != 0u) lse_fold(sh_M_all[pi], sh_E_all[pi], M, x);
        }
        const int tot = k + sh_cnt_all[pi];
        for (int e = ptid; e < tot; e += WP * 32) {
          const uint2 me = cand[e];
          if (me.x == 0u) continue;
          int rk = 0;
          for (int f = 0; f < tot; ++f) {
            const uint2 o = cand[f];
            rk += (o.x != 0u && key_before(o.x, o.y, me.x, me.y)) ? 1 : 0;
          }
          if (rk < k) res[rk] = me;
        }
        __syncthreads();  // the round's top-k in res
        if (ptid < k) cand[ptid] = res[ptid];
        if (ptid == 0) sh_cnt_all[pi] = 0;
        continue;
      }
    }
    // ---- pass 1 of the radix select: histogram of the keys' top 8 bits
#pragma unroll
    for (int i = 0; i < 4 * TPW; ++i)
      if (key[i]) atomicAdd(&hist1[key[i] >> 24], 1u);
    if (tid == 0 && v0 == 0) trace_b(a, 6);
    __syncthreads();  // S1: histogram 1, warp maxima; the running top-k of the previous round
    if (tid == 0 && v0 == 0) trace_b(a, 2);
    if (NP == 1 && v0 == 0) treg = (__ldcg(a.mrows + seq) + kBM - 1) / kBM;
    const uint32_t Mk = __reduce_max_sync(0xffffffffu, lane < WP ? sh_wm[lane] : 0u);  // the round's maximum key
    const float M = key_value(Mk);
    {  // lse partial of the round (one exp per row against the round maximum)
      float es = 0.f;
#pragma unroll
      for (int i = 0; i < 4 * TPW; ++i)
        if (key[i]) es += __expf(key_value(key[i]) - M);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
      if (lane == 0) sh_es[wq] = es;
    }
    if (wq == 0) {
      // bin of the round's k-th largest key (top 8 bits) and the keys still
      // needed inside it; when that bin and the ones above hold few keys the
      // threshold is its lower edge and the second pass is skipped
      const uint2 r = radix_bin(hist1, k);
      const uint32_t Tk = cand[k - 1].x;
      if (lane == 0) {
        sh_b1_all[pi] = r.x;
        sh_need_all[pi] = r.y;
        uint32_t T = 0xffffffffu;  // "second pass needed"
        if (r.x == 0xffffffffu) T = 0u;  // fewer than k keys: all of them are candidates
        else if ((uint32_t)k - r.y + hist1[r.x] <= (uint32_t)kSmallBin) T = r.x << 24;
        sh_T_all[pi] = T == 0xffffffffu ? T : (T > Tk ? T : Tk);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) hist1[8 * lane + j] = 0u;  // ready for the next round (read above)
    }
    if (ptid < k) res[ptid] = make_uint2(0u, 0xffffffffu);  // fewer than k candidates: padding
    __syncthreads();  // S2: threshold or pass-2 bin; every warp's lse partial
    if (wq == WP - 1) {  // fold the round's lse into the running one
      float x = lane < WP ? sh_es[lane] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0 && Mk != 0u) lse_fold(sh_M_all[pi], sh_E_all[pi], M, x);
    }
    bool need2 = false;  // pass 2 for any pair of the CTA: its barriers are the CTA's
#pragma unroll
    for (int q = 0; q < NP; ++q) need2 = need2 || sh_T_all[q] == 0xffffffffu;
    if (need2) {  // pass 2: the next 8 bits of the keys inside bin b1
      const uint32_t b1 = sh_b1_all[pi];
      const bool mine2 = sh_T_all[pi] == 0xffffffffu;
      if (mine2) {
#pragma unroll
        for (int i = 0; i < 4 * TPW; ++i)
          if (key[i] && (key[i] >> 24) == b1) atomicAdd(&hist2[(key[i] >> 16) & 0xffu], 1u);
      }
      __syncthreads();  // S3: histogram 2
      if (wq == 0 && mine2) {
        // T = the 16-bit prefix of the round's k-th largest key: at least k round
        // keys are >= T, so no round key below max(T, running k-th key) is in
        // the top-k of (running list U round)
        const uint2 r = radix_bin(hist2, sh_need_all[pi]);
        const uint32_t T = r.x == 0xffffffffu ? (b1 << 24) : (b1 << 24) | (r.x << 16);
        const uint32_t Tk = cand[k - 1].x;
#pragma unroll
        for (int j = 0; j < 8; ++j) hist2[8 * lane + j] = 0u;  // ready for the next round (read above)
        __syncwarp();
        if (lane == 0) sh_T_all[pi] = T > Tk ? T : Tk;
      }
      __syncthreads();  // S4: threshold
    }
    const uint32_t T = sh_T_all[pi];
    // ---- the keys >= T go behind the running top-k
    int c = 0;
#pragma unroll
    for (int i = 0; i < 4 * TPW; ++i) c += (key[i] != 0u && key[i] >= T) ? 1 : 0;
    if (__ballot_sync(0xffffffffu, c > 0)) {
      int pre = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += y;
      }
      int wbase = 0;
      if (lane == 31) wbase = atomicAdd(&sh_cnt_all[pi], pre);
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      int o2 = k + wbase + pre - c;
#pragma unroll
      for (int i = 0; i < 4 * TPW; ++i)
        if (key[i] != 0u && key[i] >= T) cand[o2++] = make_uint2(key[i], gid[i]);
    }
    __syncthreads();  // S5: candidates in place
    if (tid == 0 && v0 == 0) trace_b(a, 7);
    const int tot = k + sh_cnt_all[pi];
    for (int e = ptid; e < tot; e += WP * 32) {  // every candidate ranked by its own thread
      const uint2 me = cand[e];
      if (me.x == 0u) continue;
      int rk = 0;
#pragma unroll 4
      for (int f = 0; f < tot; ++f) {
        const uint2 o = cand[f];
        rk += (o.x != 0u && key_before(o.x, o.y, me.x, me.y)) ? 1 : 0;
      }
      if (rk < k) res[rk] = me;
    }
    __syncthreads();  // S6: the round's top-k in res
    if (tid == 0 && v0 == 0) trace_b(a, 9);
    if (ptid < k) cand[ptid] = res[ptid];  // the new running top-k
    if (ptid == 0) sh_cnt_all[pi] = 0;
  }
  if (wq != 0 || !live_pair) return;
  const long long ob = ((long long)seq * p.n + node) * k;
  if (lane < k) {
    const uint2 r = res[lane];
    a.topk_logit[ob + lane] = r.x ? key_value(r.x) : -INFINITY;
    a.topk_id[ob + lane] = r.x ? (int32_t)r.y : -1;
  }
  if (a.lse && lane == 0)
    a.lse[(long long)seq * p.n + node] = sh_M_all[pi] == -INFINITY ? -INFINITY : sh_M_all[pi] + logf(sh_E_all[pi]);
  if (tid == 0) trace_b(a, 4);
  if (tid == 0 && p.trace) p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + 15] = clock64();
}

// ------------------------------------------------------------------ kernel B, one round of <= 32 tiles
// One CTA (32 warps) per (sequence, node), warp w on tile w (regular tiles
// [0, tps), then patch tiles): the S partials of its lane's 4 rows summed in
// K-chunk order (as head_select_kernel), then warp_topk4 -> the tile's top-k
// list + (M, sum exp) in shared memory; warp 0 merges the <= 32 lists (the
// k-th largest list head bounds every top-k key from below; the entries above
// it are ranked by counting) and folds the lse.
__global__ void __launch_bounds__(kBThreads, 1) head_select_tiles_kernel(const __grid_constant__ SplitArgs a) {
  __shared__ uint2 lst[kBWarps][kMaxK + 1];  // +1: lane t reading list t hits distinct banks
  __shared__ float2 sst[kBWarps];
  __shared__ uint2 csw[kBWarps][kBM];  // per-warp candidate scratch, then the merge's candidates
  uint2* cm = &csw[0][0];              // (free once every warp has its list)
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = a.k;
  const int pair = blockIdx.x;
  const int seq = pair / p.n, node = pair - seq * p.n;
  const int ntp = a.tps + a.n_patch;
  const long long pst = (long long)p.n * kBM;
  const int r0 = 4 * lane;
  const int tile = warp;
  const bool on = tile < ntp;
  int S = 0, base = 0;
  warm_params(a);
  if (on) {
    tile_units(a, global_tile(a, seq, tile), S, base);
    if (lane == 0) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rowgid + ((long long)seq * ntp + tile) * kBM));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.part + (long long)base * pst + (long long)node * kBM));
    }
  }
  if (tid == 0) trace_b(a, 0);
  pdl_wait();  // A complete: partials, row ids (and the fused step's drop bitmap) visible
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) {
    trace_b(a, 1);
    if (p.trace) p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + 12] = 0xB;  // a B row
  }
  if (on) {
    const int4 g4 = __ldcg(reinterpret_cast<const int4*>(a.rowgid + ((long long)seq * ntp + tile) * kBM) + lane);
    const uint32_t dw = a.drop ? __ldcg(&a.drop[tile * 4 + (lane >> 3)]) >> ((lane & 7) * 4) : 0u;
    float zz[4] = {0.f, 0.f, 0.f, 0.f};
    const float* src = a.part + (long long)base * pst + (long long)node * kBM + r0;
    const int rot = tile % S;
    for (int c0 = 0; c0 < S; c0 += 8) {  // K chunk c was computed by split (c - tile) mod S
      float4 x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q < S) {
          int sp = c0 + q - rot;
          if (sp < 0) sp += S;
          x[q] = __ldcg(reinterpret_cast<const float4*>(src + (long long)sp * pst));
        }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q < S) { zz[0] += x[q].x; zz[1] += x[q].y; zz[2] += x[q].z; zz[3] += x[q].w; }
    }
    const int32_t g[4] = {g4.x, g4.y, g4.z, g4.w};
    uint32_t key[4];
    int32_t gid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool ok = g[i] >= 0 && !((dw >> i) & 1u);
      key[i] = ok ? float_key(zz[i]) : 0u;
      gid[i] = ok ? g[i] : -1;
      if (g[i] >= 0 && p.logits) {
        const long long col = tile < a.tps ? (long long)tile * kBM + r0 + i
                                           : (long long)p.max_ids + (tile - a.tps) * kBM + r0 + i;
        p.logits[((long long)seq * p.n + node) * a.dbg_ld + col] = zz[i];
      }
    }
    if (tid == 0) trace_b(a, 5);
    warp_topk4(key, gid, k, csw[warp], lst[warp], &sst[warp]);
  }
  __syncthreads();
  if (tid == 0) trace_b(a, 7);
  const bool has = lane < ntp;
  if (warp == 1) {  // lse: fold the tiles' (M, sum exp)
    float M = has ? sst[lane].x : -INFINITY, E = has ? sst[lane].y : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, M, o);
      const float e2 = __shfl_xor_sync(0xffffffffu, E, o);
      lse_fold(M, E, m2, e2);
    }
    if (a.lse && lane == 0) a.lse[(long long)seq * p.n + node] = M == -INFINITY ? -INFINITY : M + logf(E);
  }
  if (warp != 0) return;
  // ---- merge the tiles' lists (lane t: tile t)
  const long long ck0 = clock64();
  unsigned long long* tr = p.trace ? p.trace + (long long)(a.trace_base + blockIdx.x) * kTraceSlots : nullptr;
  const uint32_t head = has ? lst[lane][0].x : 0u;
  uint32_t v = head;
#pragma unroll
  for (int sz = 2; sz <= 32; sz <<= 1)
#pragma unroll
    for (int st = sz >> 1; st > 0; st >>= 1) {
      const uint32_t o = __shfl_xor_sync(0xffffffffu, v, st);
      const bool keep_min = ((lane & st) == 0) == ((lane & sz) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  const uint32_t T = __shfl_sync(0xffffffffu, v, 32 - k);  // k distinct heads reach it (0: fewer than k tiles)
  if (tr && lane == 0) tr[8] = clock64() - ck0;
  int c = 0;  // the list is sorted: the entries >= T are a prefix
  if (has) {
#pragma unroll 8
    for (int q = 0; q < k; ++q) {
      const uint32_t x = lst[lane][q].x;
      c += (x != 0u && x >= T) ? 1 : 0;
    }
  }
  int pre = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += y;
  }
  const int cnt = __shfl_sync(0xffffffffu, pre, 31);
  for (int q = 0; q < c; ++q) cm[pre - c + q] = lst[lane][q];
  __syncwarp();
  if (tr && lane == 0) { tr[10] = clock64() - ck0; tr[11] = cnt; }
  const long long ob = ((long long)seq * p.n + node) * k;
  for (int q = lane; q < cnt; q += 32) {
    const uint2 me = cm[q];
    int rk = 0;
#pragma unroll 4
    for (int f = 0; f < cnt; ++f) {
      const uint2 o = cm[f];
      rk += key_before(o.x, o.y, me.x, me.y) ? 1 : 0;
    }
    if (rk < k) {
      a.topk_logit[ob + rk] = key_value(me.x);
      a.topk_id[ob + rk] = (int32_t)me.y;
    }
  }
  for (int q = cnt + lane; q < k; q += 32) {
    a.topk_logit[ob + q] = -INFINITY;
    a.topk_id[ob + q] = -1;
  }
  if (tr && lane == 0) tr[13] = clock64() - ck0;
  if (tid == 0) trace_b(a, 4);
}

// ------------------------------------------------------------------ list-mode merge
// One (sequence, node) pair per WPP warps (8 / WPP pairs per 256-thread CTA):
// the exact top-k of the union of the pair's live tiles' top-k lists (a
// global top-k entry is in its tile's list: fewer than k entries of that tile
// precede it) and lse = fold of the tiles' (M, sum exp).  Threshold: the k-th
// largest of the threads' maximum list heads -- k distinct heads reach it, so
// every top-k entry does; the entries >= it (a few per pair) are ranked by
// counting.
constexpr int kMThreads = 256;
template <int WPP>
__global__ void __launch_bounds__(kMThreads) head_merge_kernel(const __grid_constant__ SplitArgs a) {
  constexpr int PP = kMThreads / 32 / WPP;  // pairs per CTA
  constexpr int PT = 32 * WPP;              // threads per pair
  extern __shared__ __align__(16) uint2 mbuf[];
  __shared__ int cnt_s[PP];
  __shared__ uint32_t thr_s[kMThreads / 32];
  __shared__ float2 lse_s[kMThreads / 32];
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pi = warp / WPP, pt = tid - pi * PT;
  const int k = a.k;
  const int cap = a.tps * k;
  uint2* cs = mbuf + (size_t)pi * cap;
  const int pair = blockIdx.x * PP + pi;
  const bool live = pair < p.batch * p.n;
  const int seq = live ? pair / p.n : 0, node = live ? pair - seq * p.n : 0;
  if (pt == 0) cnt_s[pi] = 0;
  warm_params(a);
  if (tid == 0) trace_b(a, 0);
  pdl_wait();  // the stream kernel complete: its lists visible
  asm volatile("griddepcontrol.launch_dependents;");
  if (tid == 0) {
    trace_b(a, 1);
    if (a.p.trace) a.p.trace[(long long)(a.trace_base + blockIdx.x) * kTraceSlots + 12] = 0xB;  // a B row
  }
  const int T = live ? (clamp_nact(p, seq) + kBM - 1) / kBM : 0;  // live tiles
  const uint2* lists = reinterpret_cast<const uint2*>(a.part);
  const float2* stats = reinterpret_cast<const float2*>(reinterpret_cast<const char*>(a.part) + a.list_stats);
  const long long t0 = ((long long)seq * p.n + node) * a.tps;  // the pair's tiles are contiguous
  float M = -INFINITY, E = 0.f;
  uint32_t hm = 0u;
#pragma unroll 4
  for (int j = pt; j < T; j += PT) {
    const long long ti = t0 + j;
    const uint2 h0 = __ldcg(lists + ti * k);
    const float2 st = __ldcg(stats + ti);
    lse_fold(M, E, st.x, st.y);
    hm = h0.x > hm ? h0.x : hm;
  }
  if (tid == 0) trace_b(a, 5);
  uint32_t thr = warp_kth_key(hm, k);
  if (WPP > 1) {
    if (lane == 0) thr_s[warp] = thr;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < WPP; ++w) thr = thr_s[pi * WPP + w] > thr ? thr_s[pi * WPP + w] : thr;
  } else {
    __syncwarp();
  }
  // every list entry >= thr (lists are sorted: stop at the first below)
  for (int j = pt; j < T; j += PT) {
    const uint2* L = lists + (t0 + j) * k;
    for (int e0 = 0; e0 < k; e0 += 8) {
      uint2 c[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = e0 + q < k ? __ldcg(L + e0 + q) : make_uint2(0u, 0u);
      bool more = true;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (more && c[q].x != 0u && c[q].x >= thr) {
          const int o = atomicAdd(&cnt_s[pi], 1);
          cs[o] = c[q];
        } else {
          more = false;
        }
      }
      if (!more) break;
    }
  }
  if (WPP > 1) __syncthreads();
  else __syncwarp();
  const int cnt = cnt_s[pi];
  if (tid == 0) trace_b(a, 7);
  const long long ob = ((long long)seq * p.n + node) * k;
  if (live) {
    for (int q = pt; q < cnt; q += PT) {
      const uint2 me = cs[q];
      int rk = 0;
      for (int f = 0; f < cnt; ++f) {
        const uint2 o = cs[f];
        rk += key_before(o.x, o.y, me.x, me.y) ? 1 : 0;
      }
      if (rk < k) {
        a.topk_logit[ob + rk] = key_value(me.x);
        a.topk_id[ob + rk] = (int32_t)me.y;
      }
    }
    for (int q = cnt + pt; q < k; q += PT) {
      a.topk_logit[ob + q] = -INFINITY;
      a.topk_id[ob + q] = -1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, M, o);
    const float e2 = __shfl_xor_sync(0xffffffffu, E, o);
    lse_fold(M, E, m2, e2);
  }
  if (WPP > 1) {
    if (lane == 0) lse_s[warp] = make_float2(M, E);
    __syncthreads();
    if (pt == 0)
      for (int w = 1; w < WPP; ++w) lse_fold(M, E, lse_s[pi * WPP + w].x, lse_s[pi * WPP + w].y);
  }
  if (live && pt == 0 && a.lse) a.lse[(long long)seq * p.n + node] = M == -INFINITY ? -INFINITY : M + logf(E);
  if (tid == 0) trace_b(a, 4);
}

// ------------------------------------------------------------------ host side
struct SplitLayout {
  size_t part, rowgid, arrive, mrows, drop, total;
};
constexpr int kMaxPatch = kFastThreads / kBM;  // patch tiles (update lists <= kFastThreads entries)

SplitLayout split_layout(int batch, int max_ids, int n, int num_sms) {
  const size_t tps = (size_t)(max_ids + kBM - 1) / kBM;
  const size_t tiles = (size_t)batch * tps + kMaxPatch;
  const size_t units = tiles > (size_t)num_sms ? tiles : (size_t)num_sms;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  SplitLayout L;
  size_t off = 0;
  L.part = off;   off += al(units * (size_t)n * kBM * sizeof(float));
  L.rowgid = off; off += al(tiles * kBM * sizeof(int32_t));
  L.arrive = off; off += al(sizeof(unsigned));
  L.mrows = off;  off += al((size_t)batch * sizeof(int));
  L.drop = off;   off += al((tps + kMaxPatch) * 4 * sizeof(uint32_t));
  L.total = off;
  return L;
}

int g_split_pdl = 1;
int g_num_sms = 148;  // set by the launchers (the select kernel's layout choice)
int num_sms_cached() { return g_num_sms; }
int g_stream_only = 0;  // debug mode 1: kernel A alone (measurement; no outputs are written)
// experiments (NANOSPEC_SPLIT_FLAGS): 1 = skip kernel B, 2 = no PDL, 16 = kernel B alone,
// 32 = one K atom per pipeline stage, 64 = no 256-row units in the persistent mode,
// 128 = one K atom per stage with 256-row units, 256 = no list mode (split-K 1: partial tiles + select kernel),
// 512 = the radix select kernel for one-round heads (instead of per-tile warp lists),
// 8192 = list mode of one sequence with 2 K atoms per stage (and tile pairs when tiles >= 2 x SMs),
// 16384 = the stream kernel waits for the previous grid at its start (no overlap with the previous select)
int g_split_flags = -1;
int split_flags() {
  if (g_split_flags < 0) {
    const char* e = getenv("NANOSPEC_SPLIT_FLAGS");
    g_split_flags = e ? atoi(e) : 0;
  }
  return g_split_flags;
}

template <class K>
cudaError_t launch_ex(K kern, dim3 grid, int threads, size_t smem, cudaStream_t stream, const SplitArgs& a,
                      int cluster = 1) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  const int base = na;
  if (g_split_pdl && !(split_flags() & 2)) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess && na > base) {  // without programmatic dependent launch
    (void)cudaGetLastError();
    cfg.numAttrs = base;
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  return e;
}

template <int NT, bool FUSED, int AG, int UT, bool LIST = false>
cudaError_t set_attr_once() {
  static bool done[64] = {false};  // per device: the attribute is per (function, device)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(head_stream_kernel<NT, FUSED, AG, UT, LIST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       ACfg<NT, AG, UT, LIST>::kSmemBytes);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

template <int NP, int TPW, bool MR>
cudaError_t launch_select_cfg(const SplitArgs& b, cudaStream_t stream) {
  using C = BCfg<NP, TPW>;
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!done[dev]) {
    const cudaError_t e = cudaFuncSetAttribute(head_select_kernel<NP, TPW, MR>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    if (e != cudaSuccess) return e;
    done[dev] = true;
  }
  const int pairs = b.p.batch * b.p.n;
  return launch_ex(head_select_kernel<NP, TPW, MR>, dim3((pairs + NP - 1) / NP), kBThreads, C::kSmem, stream, b);
}

// Many (sequence, node) pairs whose tiles fit one round of the 4-pair layout
// (dp64: 24 tiles, 3840 pairs): four pairs per CTA; else one pair per CTA.
cudaError_t launch_select(const SplitArgs& b, int num_sms, cudaStream_t stream) {
  const int pairs = b.p.batch * b.p.n;
  const int ntp = b.tps + b.n_patch;
  if (ntp <= kBWarps && !(split_flags() & 512))  // one round: per-tile warp lists, then a warp merge
    return launch_ex(head_select_tiles_kernel, dim3(pairs), kBThreads, 0, stream, b);
  if (pairs >= 4 * num_sms && ntp <= BCfg<4, 3>::kRound && b.S == 1 && b.extra == 0)
    return launch_select_cfg<4, 3, false>(b, stream);
  if (ntp > BCfg<1, 1>::kRound) return launch_select_cfg<1, 1, true>(b, stream);
  return launch_select_cfg<1, 1, false>(b, stream);
}

template <int NT, bool FUSED, int AG, int UT>
cudaError_t launch_pair_of_kernels(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  cudaError_t e = set_attr_once<NT, FUSED, AG, UT>();
  if (e != cudaSuccess) return e;
  SplitArgs b = a;
  b.trace_base = grid_a;
  if (!(split_flags() & 16)) {  // experiment 16: kernel B alone (on the previous call's partials)
    e = launch_ex(head_stream_kernel<NT, FUSED, AG, UT>, dim3(grid_a), kAThreads, ACfg<NT, AG, UT>::kSmemBytes,
                  stream, a);
    if (e != cudaSuccess || (split_flags() & 1) || g_stream_only) return e;
  }
  return launch_select(b, num_sms_cached(), stream);
}

template <bool FUSED, int AG>
cudaError_t launch_nt_ag(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  const int n = a.p.n;
  if (n <= 16) return launch_pair_of_kernels<16, FUSED, AG, 1>(a, grid_a, stream);
  if (n <= 32) return launch_pair_of_kernels<32, FUSED, AG, 1>(a, grid_a, stream);
  if (n <= 64) return launch_pair_of_kernels<64, FUSED, AG, 1>(a, grid_a, stream);
  if (n <= 128) return launch_pair_of_kernels<128, FUSED, AG, 1>(a, grid_a, stream);
  return launch_pair_of_kernels<256, FUSED, 1, 1>(a, grid_a, stream);  // 48 KB per atom: one atom per stage
}

// Persistent split-K-1 mode with 256-row units (two tiles share every H stage):
// one atom per stage (40 KB at n <= 64: four stages).
template <int AG>
cudaError_t launch_nt_ut2_ag(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  const int n = a.p.n;
  if (n <= 16) return launch_pair_of_kernels<16, false, AG, 2>(a, grid_a, stream);
  if (n <= 32) return launch_pair_of_kernels<32, false, AG, 2>(a, grid_a, stream);
  if (n <= 64) return launch_pair_of_kernels<64, false, AG, 2>(a, grid_a, stream);
  return launch_pair_of_kernels<128, false, 1, 2>(a, grid_a, stream);
}
cudaError_t launch_nt_ut2(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  if (split_flags() & 128) return launch_nt_ut2_ag<1>(a, grid_a, stream);  // experiment: 1 atom per stage
  return launch_nt_ut2_ag<2>(a, grid_a, stream);  // 2 atoms x 2 tiles per stage, two stages in flight
}

// List mode: the stream kernel with epilogue warps, then the merge kernel.
template <int WPP>
cudaError_t launch_merge_cfg(const SplitArgs& b, cudaStream_t stream) {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  constexpr int PP = kMThreads / 32 / WPP;
  if (!done[dev]) {
    const cudaError_t e = cudaFuncSetAttribute(head_merge_kernel<WPP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               WPP == 1 ? PP * 32 * kMaxK * 8 : kListCap * 8);
    if (e != cudaSuccess) return e;
    done[dev] = true;
  }
  const int pairs = b.p.batch * b.p.n;
  const size_t smem = (size_t)PP * b.tps * b.k * 8;
  return launch_ex(head_merge_kernel<WPP>, dim3((pairs + PP - 1) / PP), kMThreads, smem, stream, b);
}

template <int NT, int AG, int UT>
cudaError_t launch_list_pair(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  cudaError_t e = set_attr_once<NT, false, AG, UT, true>();
  if (e != cudaSuccess) return e;
  e = launch_ex(head_stream_kernel<NT, false, AG, UT, true>, dim3(grid_a), kAThreadsL,
                ACfg<NT, AG, UT, true>::kSmemBytes, stream, a);
  if (e != cudaSuccess || (split_flags() & 1) || g_stream_only) return e;
  SplitArgs b = a;
  b.trace_base = grid_a;
  return a.tps <= 32 ? launch_merge_cfg<1>(b, stream) : launch_merge_cfg<8>(b, stream);
}

cudaError_t launch_list(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  const int n = a.p.n;
  if (a.ut == 1 && a.p.batch == 1 && !(split_flags() & 8192)) {  // one sequence: 512 / 384 contiguous bytes of a row per stage
    if (n <= 16) return launch_list_pair<16, 4, 1>(a, grid_a, stream);
    if (n <= 32) return launch_list_pair<32, 4, 1>(a, grid_a, stream);
    if (n <= 64) return launch_list_pair<64, 3, 1>(a, grid_a, stream);
  }
  if (a.ut == 2) {
    if (n <= 16) return launch_list_pair<16, 2, 2>(a, grid_a, stream);
    if (n <= 32) return launch_list_pair<32, 2, 2>(a, grid_a, stream);
    if (n <= 64) return launch_list_pair<64, 2, 2>(a, grid_a, stream);
    return launch_list_pair<128, 1, 2>(a, grid_a, stream);
  }
  if (n <= 16) return launch_list_pair<16, 2, 1>(a, grid_a, stream);
  if (n <= 32) return launch_list_pair<32, 2, 1>(a, grid_a, stream);
  if (n <= 64) return launch_list_pair<64, 2, 1>(a, grid_a, stream);
  if (n <= 128) return launch_list_pair<128, 2, 1>(a, grid_a, stream);
  return launch_list_pair<256, 1, 1>(a, grid_a, stream);
}

// atoms per stage: 2 (256 contiguous bytes of a row per stage) unless the
// experiment flag 32 asks for 1
template <bool FUSED>
cudaError_t launch_nt(const SplitArgs& a, int grid_a, cudaStream_t stream) {
  if (!FUSED && a.ut == 2) return launch_nt_ut2(a, grid_a, stream);
  if (split_flags() & 32) return launch_nt_ag<FUSED, 1>(a, grid_a, stream);
  return launch_nt_ag<FUSED, 2>(a, grid_a, stream);
}

SplitArgs base_args(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse, void* scratch,
                    const SplitLayout& L) {
  SplitArgs a = {};
  char* sc = (char*)scratch;
  a.p = p;
  a.part = (float*)(sc + L.part);
  a.rowgid = (int32_t*)(sc + L.rowgid);
  a.arrive_ctr = (unsigned*)(sc + L.arrive);
  a.mrows = (int*)(sc + L.mrows);
  a.drop = nullptr;
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.k = k;
  a.tps = (p.max_ids + kBM - 1) / kBM;
  a.dbg_ld = p.max_ids;
  a.plain = (split_flags() & 16384) ? 1 : 0;
  return a;
}

bool shape_ok(const HeadProblem& p, int k) {
  return p.d % kBK == 0 && p.n >= 1 && p.n <= 256 && p.ldw % 8 == 0 && k >= 1 && k <= kMaxK && p.d / kBK >= 1;
}

std::mutex g_upd_mu;
std::vector<std::pair<int, cudaStream_t>> g_upd_streams;  // (device, stream) whose last launch was an update

}  // namespace

void note_update_launch(cudaStream_t stream) {
  int dev = 0;
  (void)cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_upd_mu);
  for (auto& e : g_upd_streams)
    if (e.first == dev && e.second == stream) return;
  g_upd_streams.emplace_back(dev, stream);
}

bool take_update_launch(cudaStream_t stream) {
  int dev = 0;
  (void)cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_upd_mu);
  for (size_t i = 0; i < g_upd_streams.size(); ++i)
    if (g_upd_streams[i].first == dev && g_upd_streams[i].second == stream) {
      g_upd_streams.erase(g_upd_streams.begin() + (long)i);
      return true;
    }
  return false;
}

size_t head_tc_scratch_bytes(int batch, int max_ids, int n) { return split_layout(batch, max_ids, n, 256).total; }

void set_head_tc_mode(int mode) {
  g_split_pdl = mode == 0 ? 0 : 1;
  g_stream_only = mode == 1 ? 1 : 0;
}

// Splits: U units on the SMs; every tile takes S = U / tiles K splits and the
// first U % tiles tiles one more (S = 1 and a persistent loop when the tiles
// outnumber the SMs).  A split holds at least one 64-column K atom.
void plan_splits(SplitArgs& a, int U, int KB) {
  const int nt = a.ntiles;
  int S = nt <= U ? U / nt : 1;
  int extra = nt <= U ? U - S * nt : 0;
  if (S >= KB) { S = KB; extra = 0; }
  if (S >= kMaxS) { S = kMaxS; extra = 0; }
  a.S = S;
  a.extra = extra;
  a.units = nt * S + extra;
}

cudaError_t launch_head_tc(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                           void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream) {
  if (!shape_ok(p, k)) return cudaErrorNotSupported;
  g_num_sms = num_sms;
  const int G = num_sms < 256 ? num_sms : 256;
  const SplitLayout L = split_layout(p.batch, p.max_ids, p.n, 256);
  if (L.total > scratch_bytes) return cudaErrorInvalidValue;
  SplitArgs a = base_args(p, k, topk_logit, topk_id, lse, scratch, L);
  if (take_update_launch(stream)) a.plain = 1;  // right after an update kernel: wait before reading the state
  a.n_patch = 0;
  a.ntiles = p.batch * a.tps;
  plan_splits(a, G, p.d / kBK);
  a.ut = 1;
  if (a.S == 1 && a.ntiles > G && (p.batch > 1 || a.ntiles >= 2 * G) && p.n <= 128 && !(split_flags() & 64)) {
    // more tiles than SMs: 256-row units, two MMAs per K step sharing the hidden-state stage.
    // Not for one sequence of capacity < 2 x SMs tiles: its live tiles may be far
    // fewer (the host cannot see n_active), and halving the units would idle SMs.
    a.ut = 2;
    a.upt = (a.tps + 1) / 2;
    a.units = p.batch * a.upt;
  }
  if (a.ut == 2 && p.batch == 1 && p.n <= 64 && !(split_flags() & 8192)) {
    // one sequence (the dense [0, V) head, verify top-k): single-tile units with
    // 3-4 K atoms per stage stream better than tile pairs with 2 (measured:
    // verify top-3 x 6 positions 208 -> 202 us); batched heads keep the pairs
    a.ut = 1;
    a.units = a.ntiles;
  }
  a.heads = a.units < G ? a.units : G;
  // more tiles than SMs (split-K 1, persistent): the tiles are reduced to
  // top-k lists inside the stream kernel and merged by a small kernel
  if (a.S == 1 && a.extra == 0 && a.ntiles > G && (long long)a.tps * k <= kListCap && !(split_flags() & 256)) {
    a.list_stats = ((long long)a.ntiles * p.n * k * 8 + 255) / 256 * 256;
    return launch_list(a, a.heads, stream);
  }
  return launch_nt<false>(a, a.heads, stream);
}

cudaError_t launch_step_tc(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit,
                              int32_t* topk_id, float* lse, void* scratch, size_t scratch_bytes, int num_sms,
                              cudaStream_t stream, bool dry_run) {
  if (!shape_ok(p, k) || p.batch != 1) return cudaErrorNotSupported;
  const long long Lr = upd.a.len + upd.b.len;
  const int G = num_sms < 256 ? num_sms : 256;
  const int tps = (p.max_ids + kBM - 1) / kBM;
  const int n_patch = Lr <= 0 ? 0 : (int)((Lr + kBM - 1) / kBM);
  // one wave: every streaming CTA plus the updater resident at once is not
  // required (nobody waits for a streaming CTA), but each tile needs a CTA
  if (n_patch > kMaxPatch || tps + n_patch + 1 > G) return cudaErrorNotSupported;
  // the updater's shared memory: UpdSmem + drop words + the raw lists
  if ((sizeof(UpdSmem) + 255) / 256 * 256 + (size_t)(tps + n_patch) * 16 + (size_t)Lr * 4 > (size_t)kBudget)
    return cudaErrorNotSupported;
  if (dry_run) return cudaSuccess;
  const SplitLayout L = split_layout(1, p.max_ids, p.n, 256);
  if (L.total > scratch_bytes) return cudaErrorInvalidValue;
  SplitArgs a = base_args(p, k, topk_logit, topk_id, lse, scratch, L);
  if (take_update_launch(stream)) a.plain = 1;
  a.n_patch = n_patch;
  a.ntiles = tps + n_patch;
  plan_splits(a, G - 1, p.d / kBK);
  a.heads = a.units;
  a.upd = upd;
  a.L = (int)Lr;
  a.drop = (uint32_t*)((char*)scratch + L.drop);
  a.dbg_ld = (long long)p.max_ids + Lr;
  return launch_nt<true>(a, a.heads + 1, stream);
}

}  // namespace nanospec
