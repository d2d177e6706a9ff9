// a3+a4+a5 (and, for nanospec_step, a2) in ONE launch for the one-wave regime
// -- every row tile of the call resident at once, the headline shape:
//
//   z'[b][i][j] = sum_c W[row(ids_b[j])][c] * H[b][i][c]     (Eq. 2 on I)
//   then per (b, i) the top-k of z' by (value desc, id asc) + lse
//
// Work split (round 2).  The active rows of a sequence are cut into P tiles of
// R = ceil(capacity / P) rows; each tile is one thread-block CLUSTER of two
// CTAs (a CTA pair, 74 pairs fill the 148 SMs) that split K = d in halves.
// Swap-AB UMMA: A = the hidden states H (M = 64 or 128 nodes, K-major SW128),
// B = the tile's gathered W rows (N = rows, <= 256 per MMA, K-major SW128), D
// (nodes x rows, fp32) in TMEM.  Why pairs: every CTA must see the whole H
// slice of its K range (the L2->SM cost grows as 1/S), while the partial sums
// that cross SMs grow with S; at S = 2 the exchange is one 32-node half of a
// (nodes x R) tile over DSMEM (5.4 KB at the headline) and H costs 256 KB of
// L2 reads per SM, which the measured stream absorbs
// (scripts/micro/ksplit.cu: R 48 / S 2 streams as fast as R 128 / S 5).
//
// Loads.  16 loader warps issue 16-byte cp.async straight from W_head into
// the SW128 ring (no repack buffer, P:247-258 is prior art): a warp
// instruction covers one row x 512 contiguous bytes (G = 4 K-atoms per ring
// group; G = 2 or 1 when the tile is tall), H rows ride in the same stages.
// Group completion is tracked by cp.async.mbarrier.arrive.noinc, slot reuse by
// tcgen05.commit; one lane of warp 16 issues the MMAs.
//
// Tail (after the last MMA; no CTA ever waits for another cluster):
//   drain  TMEM -> shared memory, node-major;
//   pair   one cluster barrier, then CTA s owns the nodes i = s (mod 2) and
//          reads the peer's partial over DSMEM: z = P_split0 + P_split1
//          (fixed order, so equal rows give bit-equal logits);
//   level1 one warp per (tile, node): lse partial (max, sum exp) and the
//          tile's top-k (threshold = k-th largest lane maximum, compaction,
//          rank by counting), published to L2;
//   level2 a per-(sequence, node) arrival counter (acq_rel); the warp that
//          completes it merges the P lists (threshold = k-th largest head,
//          rank by counting) and writes the outputs.
//
// Fused step (nanospec_step).  One extra pair: its CTA 0 runs the fast state
// update (state_fast.cuh) while the head pairs stream the rows
// [raw update-list entries (draft, verify)] ++ [pre-update slots ids[0, n_old)]
// -- a superset of the post-update active set known without waiting for the
// update.  The update publishes the stale-slot bitmap (slots whose id left I)
// and the entering ids, waits until every head CTA has read the pre-update
// slots, bumps a generation word and only then rewrites ids[] / pos[] / meta.
// Before level 1 a head CTA drops stale slots and every update-list entry that
// is invalid, repeated, or not entering I.  Result == update, then head.  The
// head pairs wait for the update CTA, so this launch is cooperative (every CTA
// co-resident or the launch fails and the caller takes update + head).
#include <cuda.h>
#include <math.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "state_fast.cuh"
#include "tc_ptx.cuh"

namespace nanospec {

namespace {

constexpr int kPW = 16;                     // loader / drain / top-k warps
constexpr int kPThreads = kPW * 32 + 32;    // + the MMA-issue warp
constexpr int kPMaxRows = 128;              // rows per tile (UMMA N; level 1 holds 8 per lane)
constexpr int kPBudget = 200 * 1024;        // dynamic shared memory (ring; the tail reuses it)
constexpr int kPMaxGroups = 12;
constexpr int kPTmemCols = 512;
constexpr int kPMaxList = 512;              // fused: raw update-list entries staged in shared memory
constexpr long long kPSpin = 1ll << 26;     // polls before giving up (a trap beats a hung GPU)

struct alignas(64) PairArgs {
  CUtensorMap hmap;  // H as a [batch * n, d] bf16 tensor: 64-column x NT-row SW128 boxes (TMA)
  HeadProblem p;
  int k;
  int P;             // head pairs (tiles) per sequence
  int R;             // rows per tile
  int G, NG;         // ring: NG groups of G K-atoms
  int stage_bytes;   // NT * 128 (H) + RP * 128 (W), RP = R rounded up to 16
  int ps;            // floats between nodes of the drained partial (RP + 4)
  int pown_bytes;    // drained partial area (1024-aligned)
  int warp_scratch;  // bytes of tail scratch per warp
  int kle;           // list stride in entries: k + 1 (lse pair), rounded up to even
  int dbg_stride;    // floats between the debug-logit rows of one node (row-list capacity)
  int flags;         // experiments: 1 = no L2 prefetch of the W rows
  uint32_t* zkey;    // [batch][n][P * R] order keys of every row's logit (0: row does not count)
  uint32_t* zgid;    // [batch][P * R] global id of every row
  uint32_t* tmax;    // [batch][n][P] each tile's largest key
  float2* tlse;      // [batch][n][P] each tile's lse partial (max, sum exp)
  unsigned* bar;     // grid barrier: phase + 2 x kBarWords arrival words (fixed scratch offset)
  float* topk_logit;
  int32_t* topk_id;
  float* lse;
  // fused step (batch 1)
  AppendArgs upd;
  int L;             // raw update-list entries streamed as rows (la + lb)
  unsigned* step_ctr;    // publication generation
  unsigned* arrive_ctr;  // head CTAs that have read the pre-update slots
  uint32_t* stale;       // [capacity / 32] pre-update slots whose id left I
  int32_t* enter_ids;    // [kFastThreads] global ids entering I
  int* enter_meta;       // {ne, n_new, n_old}
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_dyn(int n) {  // n <= kPMaxGroups - 1
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    case 7: cp_async_wait<7>(); break;
    case 8: cp_async_wait<8>(); break;
    case 9: cp_async_wait<9>(); break;
    case 10: cp_async_wait<10>(); break;
    default: cp_async_wait<11>(); break;
  }
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t caddr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// mbarrier wait with a suspend-time hint (the waiting warp sleeps in the
// barrier unit instead of re-issuing try_wait)
__device__ __forceinline__ void mbar_sleep_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}
// Whole-warp MMA issue: every lane computes the same (warp-uniform) operands,
// one elected lane issues -- the operands stay in uniform registers, so an
// MMA costs a handful of instructions (a lone-lane branch made the compiler
// broadcast them per MMA).
__device__ __forceinline__ void umma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
// SW128 K-major descriptor without its start-address field (see sw128_desc)
constexpr uint64_t kDescHi = ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) | ((uint64_t)1u << 46) |
                             ((uint64_t)2u << 61);

// Row entry e of the raw update lists (draft first, then verify).
__device__ __forceinline__ int32_t list_entry(const AppendArgs& u, int e) {
  return e < (int)u.a.len ? u.a.ptr[e] : u.b.ptr[e - (int)u.a.len];
}

// One round of the warp's arg-max over one candidate per lane (key 0 = none),
// ordered by (value desc, id asc); a repeated (key, id) pair is taken once
// per round (lowest lane).  Returns false when no candidate is left.
__device__ __forceinline__ bool warp_argmax(uint32_t lk, uint32_t lg, uint32_t& wk, uint32_t& wg, int& wl) {
  wk = __reduce_max_sync(0xffffffffu, lk);
  if (wk == 0u) return false;
  const unsigned tied = __ballot_sync(0xffffffffu, lk == wk);
  wg = (tied & (tied - 1u)) ? __reduce_min_sync(0xffffffffu, lk == wk ? lg : 0xffffffffu)
                            : __shfl_sync(0xffffffffu, lg, __ffs(tied) - 1);
  wl = __ffs(__ballot_sync(0xffffffffu, lk == wk && lg == wg)) - 1;
  return true;
}

// The update's hand-off, run by every thread of the updating CTA between the
// count update and the slot-table writes (see the file comment).
struct PairPublish {
  const PairArgs* a;
  uint32_t* stale_s;  // shared, capacity / 32 words
  unsigned n_heads;   // head CTAs that must have read the pre-update slots
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
      while (ld_acquire(a->arrive_ctr) != n_heads)
        if (++spins > kPSpin) __trap();
      *a->arrive_ctr = 0u;  // every arrival of this launch is in
      __threadfence();
      red_add_release(a->step_ctr, 1u);
    }
    __syncthreads();
  }
};

// Packed sort key: (value desc, id asc) <=> larger packed value; 0 = none.
__device__ __forceinline__ uint64_t pack_key(uint32_t key, uint32_t gid) {
  return key ? ((uint64_t)key << 32) | (uint64_t)(0xffffffffu - gid) : 0ull;
}
__device__ __forceinline__ uint2 unpack_key(uint64_t v) {
  return make_uint2((uint32_t)(v >> 32), 0xffffffffu - (uint32_t)v);
}
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
// Bitonic sort, descending, of W*E packed keys held by groups of W lanes
// (lane l of a group holds elements l*E .. l*E+E-1); groups sort independently.
template <int W, int E>
__device__ __forceinline__ void bitonic_desc(uint64_t (&v)[E]) {
  const int gl = threadIdx.x & (W - 1);
#pragma unroll
  for (int size = 2; size <= W * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= E) {  // partner in another lane
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = gl * E + e;
          const uint64_t o = shfl_xor64(v[e], stride / E);
          const bool keep_max = ((i & size) == 0) == ((i & stride) == 0);
          v[e] = keep_max ? (o > v[e] ? o : v[e]) : (o < v[e] ? o : v[e]);
        }
      } else {  // partner in this lane
#pragma unroll
        for (int e = 0; e < E; ++e)
          if ((e & stride) == 0) {
            const int e2 = e | stride;
            const bool desc = ((gl * E + e) & size) == 0;
            const uint64_t x = v[e], y = v[e2];
            const bool sw = desc ? (y > x) : (x > y);
            v[e] = sw ? y : x;
            v[e2] = sw ? x : y;
          }
      }
    }
  }
}

// Level 1 of two (tile, node)s per warp, one per half-warp (16 lanes x E
// rows): z = P_split0 + P_split1 (split 0's partial first: one summation
// order for every tile, so equal rows give bit-equal logits); publishes every
// row's order key (0 = the row does not count), the tile's largest key and
// its lse partial.  No selection here: the grid-wide threshold of level 2
// discards almost every row.  node >= n: the half idles.
template <int E>
__device__ __forceinline__ void pair_level1(const PairArgs& a, int b, int t, int node, int rows_v, int split,
                                            const float* pown, uint32_t peer_pown, const int32_t* ids_s,
                                            const unsigned char* drop_s, int row0) {
  const HeadProblem& p = a.p;
  const int hl = threadIdx.x & 15;
  const bool on = node < p.n;
  const int nd = on ? node : 0;
  const float* own = pown + nd * a.ps + hl * E;
  const uint32_t peer = peer_pown + (uint32_t)(nd * a.ps + hl * E) * 4u;
  float z[E];
  uint32_t key[E];
  uint32_t lmax = 0u;
#pragma unroll
  for (int c = 0; c < E / 4; ++c) {
    const float4 x = *reinterpret_cast<const float4*>(own + 4 * c);
    const float4 y = ld_dsmem_v4(peer + 16u * c);
    z[4 * c + 0] = split == 0 ? x.x + y.x : y.x + x.x;
    z[4 * c + 1] = split == 0 ? x.y + y.y : y.y + x.y;
    z[4 * c + 2] = split == 0 ? x.z + y.z : y.z + x.z;
    z[4 * c + 3] = split == 0 ? x.w + y.w : y.w + x.w;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int r = hl * E + e;
    key[e] = 0u;
    if (on && r < rows_v) {
      const int32_t g = ids_s[r];
      if (g >= 0 && p.logits) p.logits[((long long)b * p.n + node) * a.dbg_stride + row0 + r] = z[e];
      if (g >= 0 && !drop_s[r]) key[e] = float_key(z[e]);
    }
    lmax = key[e] > lmax ? key[e] : lmax;
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmax = y > lmax ? y : lmax;
  }
  const float M = key_value(lmax);
  float es = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (key[e]) es += __expf(z[e] - M);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
  if (!on) return;
  const long long rows_all = (long long)a.P * a.R;
  uint32_t* zk = a.zkey + ((long long)b * p.n + node) * rows_all + row0 + hl * E;
  if (hl * E < a.R) {  // the tile's slots [row0, row0 + R) (rows past rows_v publish key 0)
#pragma unroll
    for (int c = 0; c < E / 4; ++c)
      if (hl * E + 4 * c < a.R) *reinterpret_cast<uint4*>(zk + 4 * c) = make_uint4(key[4 * c], key[4 * c + 1], key[4 * c + 2], key[4 * c + 3]);
  }
  if (hl == 0) {
    const long long ti = ((long long)b * p.n + node) * a.P + t;
    a.tmax[ti] = lmax;
    a.tlse[ti] = make_float2(lmax ? M : -INFINITY, es);
  }
}

// Grid barrier of a cooperative launch over the head CTAs.  bar[0] = phase
// p, bar[1 + 16 p + w] = arrivals on word w (CTA c arrives on word c % 16, so
// no word serialises more than ~10 atomics); 16 lanes of warp 0 poll the 16
// words of set p.  Afterwards CTA 0 zeroes set 1 - p (unused in this launch)
// and flips the phase for the next launch: every launch leaves the barrier
// clean for any grid size (the scratch starts zeroed).
constexpr int kBarWords = 16;
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned phase, int nctas) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned* set = bar + 1 + kBarWords * phase;
    if (lane == 0) red_add_release(&set[blockIdx.x % kBarWords], 1u);
    const unsigned cnt_l = (unsigned)(nctas / kBarWords + (lane < nctas % kBarWords ? 1 : 0));
    long long spins = 0;
    bool done = lane >= kBarWords || cnt_l == 0u;
    while (!__all_sync(0xffffffffu, done)) {
      if (!done) done = ld_acquire(&set[lane]) >= cnt_l;
      if (++spins > kPSpin) __trap();
    }
    if (blockIdx.x == 0 && lane < kBarWords) {
      bar[1 + kBarWords * (phase ^ 1u) + lane] = 0u;
      __syncwarp(0xffffu);
      if (lane == 0) bar[0] = phase ^ 1u;
    }
  }
  __syncthreads();
}

// Level 2 of one (sequence, node) by one CTA after the grid barrier, one
// global round trip: every thread loads its rows' keys and ids, warp 0 also
// the P tile maxima and lse partials; T = the k-th largest tile maximum (k
// tiles own an entry >= T, so the top-k is >= T); the rows with key >= T
// (normally a few more than k) go to shared memory and warp 0 ranks them by
// counting.  Rows per CTA: rows_all <= kL2Per * 512.
constexpr int kL2Per = 20;  // keys per thread (P * R <= 74 * 128 < 20 * 512)
__device__ void pair_level2(const PairArgs& a, int b, int node, uint64_t* surv, int* nsurv, uint64_t* tsh) {
  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = a.k, P = a.P;
  const int rows_all = P * a.R;
  const long long tb = ((long long)b * p.n + node) * P;
  const uint32_t* zk = a.zkey + ((long long)b * p.n + node) * rows_all;
  const uint32_t* zg = a.zgid + (long long)b * rows_all;
  uint32_t x[kL2Per], g[kL2Per];
  if (warp < kPW) {
#pragma unroll
    for (int c = 0; c < kL2Per; ++c) {
      const int r = tid + c * kPW * 32;
      x[c] = r < rows_all ? __ldcg(zk + r) : 0u;
      g[c] = r < rows_all ? __ldcg(zg + r) : 0u;
    }
  }
  float m = -INFINITY, e = 0.f;
  if (warp == 0) {
    uint32_t tm[3];
    float2 st[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int t2 = lane + 32 * c;
      tm[c] = t2 < P ? __ldcg(a.tmax + tb + t2) : 0u;
      st[c] = t2 < P ? __ldcg(a.tlse + tb + t2) : make_float2(-INFINITY, 0.f);
    }
    uint32_t hm = 0u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      hm = tm[c] > hm ? tm[c] : hm;
      lse_fold(m, e, st[c].x, st[c].y);
    }
    const uint32_t T = warp_kth_key(hm, k);  // 0 when fewer than k tiles have live rows: every live row survives
    if (lane == 0) { *tsh = T; *nsurv = 0; }
  }
  __syncthreads();
  const uint32_t T = (uint32_t)*tsh;
  if (warp < kPW) {
#pragma unroll
    for (int c = 0; c < kL2Per; ++c)
      if (x[c] != 0u && x[c] >= T) {
        const int q = atomicAdd(nsurv, 1);
        if (q < kPW * 64) surv[q] = pack_key(x[c], g[c]);
      }
  }
  __syncthreads();
  if (warp != 0) return;
  const int cnt = *nsurv;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), e2 = __shfl_xor_sync(0xffffffffu, e, o);
    lse_fold(m, e, m2, e2);
  }
  // rank every survivor by counting (broadcast shared-memory reads, independent)
  const int c2 = cnt < kPW * 64 ? cnt : kPW * 64;  // more only if every row ties
  for (int i = lane; i < c2; i += 32) {
    const uint64_t me = surv[i];
    int rk = 0;
    for (int j = 0; j < c2; ++j) {
      const uint64_t o = surv[j];
      rk += (o > me || (o == me && j < i)) ? 1 : 0;
    }
    if (rk < k) tsh[1 + rk] = me;
  }
  __syncwarp();
  const uint2 res = lane < k && lane < c2 ? unpack_key(tsh[1 + lane]) : make_uint2(0u, 0xffffffffu);
  const long long ob = ((long long)b * p.n + node) * k;
  if (lane < k) {
    a.topk_logit[ob + lane] = res.x ? key_value(res.x) : -INFINITY;
    a.topk_id[ob + lane] = res.x ? (int32_t)res.y : -1;
  }
  if (a.lse && lane == 0) a.lse[(long long)b * p.n + node] = m == -INFINITY ? -INFINITY : m + logf(e);
}

template <int NT, bool FUSED>  // NT = UMMA M: 64 (n <= 64) or 128 nodes
__global__ void __launch_bounds__(kPThreads, 1) head_pair_kernel(const __grid_constant__ PairArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  __shared__ __align__(8) uint64_t bar_full[kPMaxGroups];
  __shared__ __align__(8) uint64_t bar_empty[kPMaxGroups];
  __shared__ __align__(8) uint64_t bar_acc;
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t ids_s[kPMaxRows];          // global id of each tile row (-1: not loaded)
  __shared__ unsigned char drop_s[kPMaxRows];   // fused: rows that do not count
  __shared__ int32_t list_s[FUSED ? kPMaxList : 1];   // fused: the raw update lists
  __shared__ int32_t enter_s[FUSED ? kPMaxList : 1];  // fused: the ids entering I (published by the update)
  __shared__ unsigned sh_g0;
  __shared__ unsigned sh_phase;

  const HeadProblem& p = a.p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pair = blockIdx.x >> 1, split = blockIdx.x & 1;  // cluster (2,1,1): rank == split
  const int nhead = FUSED ? (int)(gridDim.x >> 1) - 1 : (int)(gridDim.x >> 1);
  if (tid == 0) trace_mark(p.trace, 0);

  if (FUSED && pair == nhead) {  // the update pair: CTA 0 updates, CTA 1 has nothing to do
    if (split == 0) {
      UpdSmem& us = *reinterpret_cast<UpdSmem*>(smem);
      uint32_t* stale_s = reinterpret_cast<uint32_t*>(smem + (sizeof(UpdSmem) + 255) / 256 * 256);
      PairPublish pub{&a, stale_s, (unsigned)(2 * nhead)};
      update_fast(a.upd, a.upd.seq0, us, pub, nullptr);
    }
    return;
  }

  const int b = pair / a.P, t = pair % a.P;
  const int KA = (p.d + 63) / 64;  // K atoms of 64
  const int ka0 = split == 0 ? 0 : KA / 2, ka1 = split == 0 ? KA / 2 : KA;
  const int nA = ka1 - ka0;
  const int G = a.G, NG = a.NG, ngroups = (nA + G - 1) / G;
  const int row0 = t * a.R;

  if (tid == 0) {
    sh_phase = *(volatile unsigned*)a.bar;  // grid-barrier phase of this launch
    for (int g = 0; g < NG; ++g) {
      mbar_init(smem_u32(&bar_full[g]), kPW * 32 + 1);  // an async arrival per loader thread + the TMA expect_tx
      mbar_init(smem_u32(&bar_empty[g]), 1);        // one tcgen05.commit
    }
    mbar_init(smem_u32(&bar_acc), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 32) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.hmap) : "memory");
  if (warp == kPW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "n"(kPTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }

  // ---- rows of this tile: every input load in one round trip
  int m_rows;  // rows of this sequence's row list
  {
    const int32_t* idsb = p.ids_base + (long long)b * p.ids_stride;
    const int m0 = clamp_nact(p, b);
    const int rg = row0 + tid;
    int32_t gid = -1;
    if (FUSED) {
      // rows: [0, L) raw update-list entries, then the pre-update slots [0, n_old)
      const int L = a.L;
      if (tid < L) list_s[tid] = list_entry(a.upd, tid);
      if (tid < a.R) {
        if (rg < L) {
          const int32_t g = list_entry(a.upd, rg);
          gid = (g >= 0 && g < a.upd.sv.vocab && is_local(a.upd.sv, g)) ? g : -1;
        } else if (rg - L < p.max_ids) {
          gid = idsb[rg - L];
        }
      }
      m_rows = L + m0;
      if (tid == 0) sh_g0 = ld_acquire(a.step_ctr);  // read before arriving: the update publishes after
    } else {
      if (tid < a.R && rg < p.max_ids) gid = idsb[rg];
      m_rows = m0;
    }
    if (tid < kPMaxRows) {
      ids_s[tid] = (tid < a.R && rg < m_rows) ? gid : -1;
      drop_s[tid] = 0;
    }
  }
  const int rows_v = max(0, min(a.R, m_rows - row0));  // rows of this tile in the row list
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (FUSED && tid == 0) red_add_release(a.arrive_ctr, 1u);  // pre-update slots read
  if (tid == 0) trace_mark(p.trace, 1);
  const bool work = rows_v > 0 && nA > 0;
  const uint32_t ring = smem_u32(smem);
  if (warp < kPW) {
    // ---------------- loaders: group gi = atoms [gi*G, gi*G + G) of this CTA's K range;
    // a warp instruction covers 4/G rows x G*128 contiguous bytes of each row
    if (work) {
      const int rpi = 4 / G;
      const int ch = lane & 7, sub = lane >> 3;
      const int ao = sub % G, ro = sub / G;
      for (int gi = 0; gi < ngroups; ++gi) {
        const int slot_g = gi % NG;
        if (gi >= NG) mbar_sleep_wait(smem_u32(&bar_empty[slot_g]), ((gi / NG) - 1) & 1);
        const int j = gi * G + ao;  // this lane's atom
        if (j < nA) {
          const uint32_t st = ring + (uint32_t)((slot_g * G + ao) * a.stage_bytes);
          const int col = (ka0 + j) * 64 + ch * 8;
          const bool colok = col < p.d;
          const uint32_t swz = (uint32_t)(ch << 4);
          const uint32_t stw = st + NT * 128;
          for (int r = warp * rpi + ro; r < rows_v; r += kPW * rpi) {
            const int32_t g = ids_s[r];
            if (g < 0) continue;
            const long long row = p.n_shards > 1 ? g / p.n_shards : g;
            cp_async16(stw + (uint32_t)(r * 128) + (swz ^ (uint32_t)((r & 7) << 4)),
                       p.w + row * p.ldw + (colok ? col : 0), colok ? 16u : 0u);
          }
        }
        if (tid == 0) {  // H of the group's atoms: one TMA box each (rows >= n: the next sequence or zeros)
          const int na = min(G, nA - gi * G);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_full[slot_g])),
                       "r"((uint32_t)(na * NT * 128))
                       : "memory");
          for (int q = 0; q < na; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    ring + (uint32_t)((slot_g * G + q) * a.stage_bytes)),
                "l"(&a.hmap), "r"((ka0 + gi * G + q) * 64), "r"(b * p.n), "r"(smem_u32(&bar_full[slot_g]))
                : "memory");
        }
        cp_async_mbar_arrive_noinc(smem_u32(&bar_full[slot_g]));
      }
    }
    if (tid == 0) trace_mark(p.trace, 2);
    // ---------------- fused: drop masks (warp 15) while the last loads land and the MMAs run
    if (FUSED && warp == kPW - 1) {
      if (lane == 0) {
        long long spins = 0;
        while (ld_acquire(a.step_ctr) == sh_g0)
          if (++spins > kPSpin) __trap();
      }
      __syncwarp();
      const int ne = min(__ldcg(&a.enter_meta[0]), kPMaxList);
      for (int q = lane; q < ne; q += 32) enter_s[q] = __ldcg(&a.enter_ids[q]);  // independent loads, one round trip
      __syncwarp();
      for (int r = lane; r < rows_v; r += 32) {
        const int rg = row0 + r;
        unsigned char drop = 0;
        if (rg < a.L) {  // an update-list entry counts iff it is the first of its id and enters I
          const int32_t g = ids_s[r];
          if (g >= 0) {
            for (int e2 = 0; e2 < rg && !drop; ++e2) drop = list_s[e2] == g;
            if (!drop) {
              bool in = false;
              for (int q = 0; q < ne && !in; ++q) in = enter_s[q] == g;
              drop = !in;
            }
          }
        } else {  // a pre-update slot counts iff its id is still active
          const int s2 = rg - a.L;
          drop = (__ldcg(&a.stale[s2 >> 5]) >> (s2 & 31)) & 1u;
        }
        drop_s[r] = drop;
      }
    }
    if (work) {
      mbar_sleep_wait(smem_u32(&bar_acc), 0);
      tc_fence_after();
    }
    if (tid == 0) trace_mark(p.trace, 3);
    // ---------------- drain TMEM -> pown[node][row] (nodes < n)
    float* pown = reinterpret_cast<float*>(smem);
    const int q = warp & 3, cg = warp >> 2;
    const int node = NT == 64 ? (lane < 16 ? 16 * q + lane : -1) : 32 * q + lane;
    const int nch16 = (rows_v + 15) >> 4;
    for (int cc = cg; cc < nch16; cc += 4) {
      float v[16];
      if (nA > 0) {
        tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(cc * 16), v);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      if (node >= 0 && node < p.n) {
        float4* dst = reinterpret_cast<float4*>(pown + node * a.ps + cc * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
  } else if (work) {
    // ---------------- MMA issue (warp 16; warp-uniform operands, one elected lane issues)
    const int nc0 = rows_v >= 256 ? 256 : (NT == 64 ? (rows_v + 7) & ~7 : (rows_v + 15) & ~15);
    const int nrem1 = rows_v - 256;
    const int nc1 = nrem1 <= 0 ? 0 : (NT == 64 ? (nrem1 + 7) & ~7 : (nrem1 + 15) & ~15);
    const uint32_t id0 = make_idesc(NT, nc0), id1 = make_idesc(NT, nc1 > 0 ? nc1 : 16);
    int gslot = 0, gphase = 0, ja = 0;  // ring group, its phase, atom within the group
    uint32_t st = ring;
    for (int j = 0; j < nA; ++j) {
      if (ja == 0) {
        mbar_sleep_wait(smem_u32(&bar_full[gslot]), (uint32_t)gphase);
        tc_fence_after();

      }
      const uint32_t a_lo = (st >> 4) & 0x3FFFu, b_lo = ((st + NT * 128) >> 4) & 0x3FFFu;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (j | kk) != 0;
        if (!(a.flags & 4)) umma_elect(tmem, kDescHi | (a_lo + 2 * kk), kDescHi | (b_lo + 2 * kk), id0, acc);
        if (nc1 > 0) umma_elect(tmem + 256, kDescHi | (a_lo + 2 * kk), kDescHi | (b_lo + 2048 + 2 * kk), id1, acc);
      }
      st += a.stage_bytes;
      if (++ja == G || j == nA - 1) {
        commit_elect(smem_u32(&bar_empty[gslot]));
        ja = 0;
        if (++gslot == NG) { gslot = 0; gphase ^= 1; st = ring; }
      }
    }
    commit_elect(smem_u32(&bar_acc));
  }
  tc_fence_before();
  __syncwarp();
  // ---------------- pair exchange: both partials drained
  cluster_arrive();
  cluster_wait();
  if (warp == kPW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kPTmemCols));
  }
  if (tid == 0) trace_mark(p.trace, 4);
  // ---------------- level 1 (nodes i = split mod 2), arrivals; level 2 by the last arriver
  const float* pown = reinterpret_cast<const float*>(smem);
  const uint32_t peer_pown = mapa_shared(ring, (uint32_t)(split ^ 1));
  uint2* scr = reinterpret_cast<uint2*>(smem + a.pown_bytes + warp * a.warp_scratch);
  if (warp < kPW) {
    // round rd: this warp's half-warps take local nodes 2 (warp + 16 rd) + half,
    // i.e. nodes split + 2 * local (this CTA owns the nodes i = split mod 2)
    const int half = lane >> 4;
    const int nown = (p.n - split + 1) / 2;
    for (int rd = 0; 2 * (warp + kPW * rd) < nown; ++rd) {
      const int local = 2 * (warp + kPW * rd) + half;
      const int node = local < nown ? split + 2 * local : p.n;
      if (a.R <= 64) pair_level1<4>(a, b, t, node, rows_v, split, pown, peer_pown, ids_s, drop_s, row0);
      else pair_level1<8>(a, b, t, node, rows_v, split, pown, peer_pown, ids_s, drop_s, row0);
    }
  }
  if (split == 0)  // the tile's global ids (padding slots: -1)
    for (int r = tid; r < a.R; r += blockDim.x) a.zgid[(long long)b * a.P * a.R + row0 + r] = (uint32_t)ids_s[r];
  if (tid == 0) trace_mark(p.trace, 5);
  __syncwarp();
  cluster_arrive();  // this CTA no longer reads the peer's partial
  grid_barrier(a.bar, sh_phase, 2 * nhead);
  if (tid == 0) trace_mark(p.trace, 6);
  // ---------------- level 2: one (sequence, node) per CTA
  uint64_t* surv = reinterpret_cast<uint64_t*>(smem + a.pown_bytes);
  __shared__ int sh_nsurv;
  __shared__ uint64_t sh_t[33];
  for (int j = blockIdx.x; j < p.batch * p.n; j += 2 * nhead) pair_level2(a, j / p.n, j % p.n, surv, &sh_nsurv, sh_t);
  if (tid == 0) trace_mark(p.trace, 7);
  __syncwarp();
  cluster_wait();  // the peer no longer reads this CTA's partial
}

int g_pair_enabled = 1;

struct PairPlan {
  int NT, P, R, RP, G, NG, stage_bytes, ps, pown_bytes, warp_scratch, kle, grid;
};

// Host-side plan: one wave of pairs, or false when the shape does not fit.
bool pair_plan(const HeadProblem& p, int k, int L, int num_sms, bool fused, PairPlan* out) {
  if (p.n < 1 || p.n > 128 || k < 1 || k > 32 || p.d % 8 != 0 || p.ldw % 8 != 0) return false;
  PairPlan q;
  q.NT = p.n <= 64 ? 64 : 128;
  const int pairs = (num_sms < kMaxPairSMs ? num_sms : kMaxPairSMs) / 2 - (fused ? 1 : 0);
  q.P = pairs / p.batch;
  if (q.P < 1 || q.P > 96) return false;  // level 2: <= 3 lists per lane
  const long long cap = (long long)p.max_ids + L;
  q.R = (int)((cap + q.P - 1) / q.P + 3) & ~3;  // level 1 publishes 4 rows per store
  if (q.R > kPMaxRows) return false;
  q.RP = (q.R + 15) & ~15;
  q.ps = q.RP + 4;
  q.pown_bytes = (p.n * q.ps * 4 + 1023) / 1024 * 1024;
  q.kle = (k + 2) & ~1;
  q.warp_scratch = (kPBudget - q.pown_bytes) / kPW / 16 * 16;
  if (kPBudget - q.pown_bytes < kPW * 64 * 8) return false;  // level 2: survivor slots
  q.stage_bytes = q.NT * 128 + q.RP * 128;
  q.G = 0;
  for (int g = 4; g >= 1; g >>= 1) {
    const int ng = kPBudget / (g * q.stage_bytes);
    if (ng >= 3 || (g == 1 && ng >= 2)) { q.G = g; q.NG = ng < kPMaxGroups ? ng : kPMaxGroups; break; }
  }
  if (q.G == 0) return false;
  if (const char* e = getenv("NANOSPEC_PAIR_G")) {  // experiments: force the ring grouping
    const int g = atoi(e);
    if (g == 1 || g == 2 || g == 4) {
      q.G = g;
      q.NG = kPBudget / (g * q.stage_bytes);
      if (q.NG > kPMaxGroups) q.NG = kPMaxGroups;
      if (q.NG < 2) return false;
    }
  }
  if (fused && ((long long)((sizeof(UpdSmem) + 255) / 256 * 256) + (p.max_ids + 31) / 32 * 4 > kPBudget ||
                L > kPMaxList))
    return false;
  q.grid = 2 * (q.P * p.batch + (fused ? 1 : 0));
  *out = q;
  return true;
}

template <int NT, bool FUSED>
cudaError_t launch_pair_nt(const PairPlan& q, const PairArgs& a, cudaStream_t stream) {
  static bool attr[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(head_pair_kernel<NT, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kPBudget + 1024);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(q.grid);
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = kPBudget + 1024;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // its CTAs wait for each other across clusters (grid barrier; fused: the
  // update hand-off): cooperative, so every CTA is co-resident or the launch fails
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, head_pair_kernel<NT, FUSED>, a);
}

// H as a [batch * n, d] bf16 tensor map with 64-column x NT-row SW128 boxes
// (cuTensorMapEncodeTiled through the runtime's driver entry point, no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool encode_hmap(CUtensorMap* m, const HeadProblem& p, int NT) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qr;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  if (!fn || ((uintptr_t)p.h & 15u)) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)p.d, (cuuint64_t)p.batch * (cuuint64_t)p.n};
  const cuuint64_t gstr[1] = {(cuuint64_t)p.d * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)NT};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(p.h), gdim, gstr, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

PairArgs make_args(const HeadProblem& p, const PairPlan& q, int k, float* topk_logit, int32_t* topk_id, float* lse,
                   const PairScratch& s) {
  PairArgs a = {};
  a.p = p;
  a.k = k;
  a.P = q.P;
  a.R = q.R;
  a.G = q.G;
  a.NG = q.NG;
  a.stage_bytes = q.stage_bytes;
  a.ps = q.ps;
  a.pown_bytes = q.pown_bytes;
  a.warp_scratch = q.warp_scratch;
  a.kle = q.kle;
  a.dbg_stride = p.max_ids;
  if (const char* e = getenv("NANOSPEC_PAIR_FLAGS")) a.flags = atoi(e);
  {
    const size_t rows = (size_t)(kMaxPairSMs / 2) * kPMaxRows;  // >= batch * P * R
    char* c = reinterpret_cast<char*>(s.cand);
    a.zkey = reinterpret_cast<uint32_t*>(c);
    a.zgid = reinterpret_cast<uint32_t*>(c + rows * p.n * 4);
    a.tmax = reinterpret_cast<uint32_t*>(c + rows * (p.n + 1) * 4);
    a.tlse = reinterpret_cast<float2*>(c + rows * (p.n + 1) * 4 + (size_t)(kMaxPairSMs / 2) * p.n * 4);
  }
  a.bar = s.grid_word + 16;  // 64 bytes into the scratch's first 256-byte block (head_tc.cu grid_word is word 0)
  a.topk_logit = topk_logit;
  a.topk_id = topk_id;
  a.lse = lse;
  a.step_ctr = s.step_ctr;
  a.arrive_ctr = s.arrive_ctr;
  a.stale = s.stale;
  a.enter_ids = s.enter_ids;
  a.enter_meta = s.enter_meta;
  return a;
}

}  // namespace

size_t pair_cand_bytes(int n) {
  const size_t tiles = kMaxPairSMs / 2, rows = tiles * kPMaxRows;
  return rows * (size_t)(n + 1) * 4 + tiles * (size_t)n * 12;
}

void set_head_pair_enabled(int on) { g_pair_enabled = on; }

cudaError_t launch_head_pair(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                             const PairScratch& s, int num_sms, cudaStream_t stream) {
  if (!g_pair_enabled) return cudaErrorNotSupported;
  PairPlan q;
  if (!pair_plan(p, k, 0, num_sms, false, &q)) return cudaErrorNotSupported;
  PairArgs a = make_args(p, q, k, topk_logit, topk_id, lse, s);
  if (!encode_hmap(&a.hmap, p, q.NT)) return cudaErrorNotSupported;
  const cudaError_t e = q.NT == 64 ? launch_pair_nt<64, false>(q, a, stream) : launch_pair_nt<128, false>(q, a, stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return cudaErrorNotSupported;  // e.g. not every CTA can be resident: the caller takes the other kernel
  }
  return e;
}

cudaError_t launch_step_pair(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit, int32_t* topk_id,
                             float* lse, const PairScratch& s, int num_sms, cudaStream_t stream, bool dry_run) {
  if (!g_pair_enabled || p.batch != 1) return cudaErrorNotSupported;
  const long long L = upd.a.len + upd.b.len;
  if (L > kFastThreads) return cudaErrorNotSupported;
  PairPlan q;
  if (!pair_plan(p, k, (int)L, num_sms, true, &q)) return cudaErrorNotSupported;
  if (dry_run) return cudaSuccess;
  PairArgs a = make_args(p, q, k, topk_logit, topk_id, lse, s);
  if (!encode_hmap(&a.hmap, p, q.NT)) return cudaErrorNotSupported;
  a.upd = upd;
  a.L = (int)L;
  a.dbg_stride = p.max_ids + (int)L;
  cudaError_t e = q.NT == 64 ? launch_pair_nt<64, true>(q, a, stream) : launch_pair_nt<128, true>(q, a, stream);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return cudaErrorNotSupported;  // e.g. cooperative + cluster refused: the caller takes update + head
  }
  return e;
}

}  // namespace nanospec
