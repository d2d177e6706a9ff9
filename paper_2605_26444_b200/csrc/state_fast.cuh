// The per-step fast path of a2 (state update), shared by the standalone
// update kernel (state.cu) and the fused update + head kernel (head_tc.cu).
#pragma once
#include "common.cuh"

namespace nanospec {

struct ListArg {
  const int32_t* ptr;   // base for sequence 0
  long long len;        // elements per sequence
  long long seq_stride; // elements between sequences (0 = same list for all)
  int dedup;            // tuple(.) semantics
};

struct AppendArgs {
  StateView sv;
  int seq0;
  int reset;
  ListArg a, b;
};

__device__ __forceinline__ bool is_local(const StateView& sv, int32_t g) {
  return sv.n_shards <= 1 || (g % sv.n_shards) == sv.rank;
}
__device__ __forceinline__ int32_t local_of(const StateView& sv, int32_t g) {
  return sv.n_shards <= 1 ? g : g / sv.n_shards;
}

// Per-step fast path of a2 (rule R1, no reset, both lists together <= 512 ids
// and <= W_max): one CTA per sequence, O(changes) work, three dependent global
// round trips (the single writer of a sequence needs no global atomics):
//   RT1  meta (total, n_active) + the two lists;
//        tuple(.) dedup in a shared-memory hash, block scan -> ring slots;
//   RT2  evicted ring slots, cnt[] of the appended ids, the last L ids[] slots
//        (candidates to move when I shrinks);
//   RT3  cnt[] and pos[] of the evicted ids;
// then every touched id's window count is updated by its net change
// (appends - evictions): count 0 -> >0 enters I, >0 -> 0 leaves it.  Slot
// table (pos[g] = slot of g in ids[]): entering ids take the slots of leaving
// ids, extra entries are appended, surplus holes are refilled from the tail,
// so ids[0, n_active) stays dense and every other id keeps its slot.
constexpr int kFastThreads = 512;
constexpr int kHashSlots = 2048;

__device__ __forceinline__ int hash_slot(int32_t key) {
  return (int)(((uint32_t)key * 2654435761u) >> 21) & (kHashSlots - 1);
}

// Insert `key` (>= 0) into an open-addressing table; returns its slot.
__device__ __forceinline__ int hash_insert(int32_t* keys, int32_t key) {
  int h = hash_slot(key);
  while (true) {
    const int32_t old = atomicCAS(&keys[h], -1, key);
    if (old == -1 || old == key) return h;
    h = (h + 1) & (kHashSlots - 1);
  }
}

// Shared memory of one update (45 KB): the standalone kernel declares it
// statically, the fused step kernel carves it out of its stage area.
struct UpdSmem {
  int32_t hkey[kHashSlots];   // dedup table, then the touched-id table
  int32_t hval[kHashSlots];   // first position, then net count change
  int32_t hcnt[kHashSlots];   // window count before this update
  int32_t hpos[kHashSlots];   // slot before this update (evicted ids)
  int32_t raw[kFastThreads];    // the update lists as given (draft, then verify), for the publish hook
  int32_t leave[kFastThreads];  // local ids leaving I
  int32_t enter[kFastThreads];  // local ids entering I
  int32_t hole[kFastThreads];   // their former slots
  int32_t tail[kFastThreads];   // tail[j] = ids[n_old - 1 - j]
  int32_t mover_slot[kFastThreads];
  int32_t low_hole[kFastThreads];
  unsigned char tail_hole[kFastThreads];
  int sh_scan[40];
  long long sh_total;
  int sh_nact, sh_err, sh_nl, sh_ne, sh_nm, sh_nh;
};

// Standalone update: nothing to publish.
struct NoPublish {
  __device__ void operator()(const StateView&, UpdSmem&, int /*n_old*/, int /*nl*/, int /*ne*/) const {}
};

// The fast update of sequence `seq` by the whole CTA (blockDim >= kFastThreads
// threads; threads past kFastThreads only join the barriers).  `publish(sv,
// sm, n_old, nl, ne)` runs once the leaving (sm.leave / sm.hole) and entering
// (sm.enter) ids are known and before ids[], pos[] and meta are written; all
// threads call it (it may synchronise the CTA).
template <class Publish>
__device__ void update_fast(const AppendArgs& args, int seq, UpdSmem& sm, Publish& publish,
                            unsigned long long* trace) {
  int32_t* hkey = sm.hkey; int32_t* hval = sm.hval; int32_t* hcnt = sm.hcnt; int32_t* hpos = sm.hpos;
  int32_t* leave = sm.leave; int32_t* enter = sm.enter; int32_t* hole = sm.hole; int32_t* tail = sm.tail;
  int32_t* mover_slot = sm.mover_slot; int32_t* low_hole = sm.low_hole; unsigned char* tail_hole = sm.tail_hole;
  int* sh_scan = sm.sh_scan;
  long long& sh_total = sm.sh_total;
  int& sh_nact = sm.sh_nact; int& sh_err = sm.sh_err; int& sh_nl = sm.sh_nl; int& sh_ne = sm.sh_ne;
  int& sh_nm = sm.sh_nm; int& sh_nh = sm.sh_nh;
  const StateView& sv = args.sv;
  const int tid = threadIdx.x;
  const int W = sv.w_max;
  const int la = (int)args.a.len, lb = (int)args.b.len;
  const int L = la + lb;
  uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
  int32_t* ring = sv.ring + (long long)seq * W;
  int32_t* cnt = sv.cnt + (long long)seq * sv.v_local;
  int32_t* pos = sv.pos + (long long)seq * sv.v_local;
  int32_t* ids = sv.ids + (long long)seq * W;
  // ---- RT1: meta + lists
  if (tid == 0) {
    sh_total = sv.meta[seq].total;
    sh_nact = sv.meta[seq].n_active;
    sh_err = 0; sh_nl = 0; sh_ne = 0; sh_nm = 0; sh_nh = 0;
  }
  int32_t e = -1;
  if (tid < la) e = args.a.ptr[(long long)(seq - args.seq0) * args.a.seq_stride + tid];
  else if (tid < L) e = args.b.ptr[(long long)(seq - args.seq0) * args.b.seq_stride + (tid - la)];
  for (int h = tid; h < kHashSlots; h += blockDim.x) { hkey[h] = -1; hval[h] = 0x7fffffff; }
  if (tid < L) sm.raw[tid] = e;
  __syncthreads();
  if (tid == 0) trace_mark(trace, 10);  // state: lists staged
  // ---- tuple(.): keep the first occurrence of every id within its own list
  const bool valid = tid < L && e >= 0 && e < sv.vocab;
  if (tid < L && !valid) sh_err = 1;
  int hs = -1;
  if (valid) {
    hs = hash_insert(hkey, e * 2 + (tid < la ? 0 : 1));
    atomicMin(&hval[hs], tid);
  }
  __syncthreads();
  const bool keep = valid && hval[hs] == tid;
  int nk;
  const int sp = block_exclusive_scan(keep ? 1 : 0, sh_scan, &nk);
  const long long total = sh_total;
  const int n_old = sh_nact;
  // ---- RT2: evicted slots, counts of the appended ids, tail of the slot table
  int slot = (int)(total % W) + sp;  // sp < W: one wrap at most
  if (slot >= W) slot -= W;
  const bool e_loc = keep && is_local(sv, e);
  const int32_t le = e_loc ? local_of(sv, e) : -1;
  int32_t old = -1, ce = 0, tl = -1;
  if (keep && total + sp >= W) old = ring[slot];
  if (e_loc) ce = cnt[le];
  if (tid < L && n_old - 1 - tid >= 0) tl = ids[n_old - 1 - tid];
  const bool o_loc = old >= 0 && is_local(sv, old);
  const int32_t lo = o_loc ? local_of(sv, old) : -1;
  // ---- RT3 (issued right away; independent of the shared-memory work below)
  int32_t co = 0, po = 0;
  if (o_loc) { co = cnt[lo]; po = pos[lo]; }
  if (keep) ring[slot] = e;
  if (tid < L) tail[tid] = tl;
  for (int h = tid; h < kHashSlots; h += blockDim.x) { hkey[h] = -1; hval[h] = 0; }
  __syncthreads();
  if (tid == 0) trace_mark(trace, 11);  // state: ring slots read
  // ---- net window-count change per touched local id, with its prior count / slot
  if (e_loc) {
    const int h = hash_insert(hkey, le);
    atomicAdd(&hval[h], 1);
    hcnt[h] = ce;
  }
  if (o_loc) {
    const int h = hash_insert(hkey, lo);
    atomicSub(&hval[h], 1);
    hcnt[h] = co;  // every writer of a slot stores the same pre-update value
    hpos[h] = po;
  }
  __syncthreads();
  for (int h = tid; h < kHashSlots; h += blockDim.x) {
    const int32_t l = hkey[h], dlt = hval[h];
    if (l < 0 || dlt == 0) continue;
    const int32_t before = hcnt[h];
    const int32_t after = before + dlt;
    cnt[l] = after;
    if (before > 0 && after == 0) {
      atomicAnd(&bm[l >> 5], ~(1u << (l & 31)));
      const int q = atomicAdd(&sh_nl, 1);
      leave[q] = l;
      hole[q] = hpos[h];  // a leaving id was evicted, so its slot was read in RT3
    } else if (before == 0 && after > 0) {
      atomicOr(&bm[l >> 5], 1u << (l & 31));
      enter[atomicAdd(&sh_ne, 1)] = l;
    }
  }
  __syncthreads();
  if (tid == 0) trace_mark(trace, 12);  // state: counts updated
  // ---- slot table
  const int nl = sh_nl, ne = sh_ne;
  const int n_new = n_old - nl + ne;
  publish(sv, sm, n_old, nl, ne);
  if (tid < n_old - n_new) tail_hole[tid] = 0;
  __syncthreads();
  const int32_t gmul = sv.n_shards <= 1 ? 1 : sv.n_shards, gadd = sv.n_shards <= 1 ? 0 : sv.rank;
  if (tid < ne) {  // entering ids: a freed slot, or a new slot at the end
    const int s2 = tid < nl ? hole[tid] : n_old + (tid - nl);
    const int32_t g = enter[tid] * gmul + gadd;
    ids[s2] = g;
    pos[enter[tid]] = s2;
    // a hole in the tail [n_new, n_old) refilled here is then moved down as a
    // live entry: keep the prefetched tail current
    const int j = n_old - 1 - s2;
    if (j >= 0 && j < L) tail[j] = g;
  }
  if (nl > ne) {
    // I shrinks by d = nl - ne: holes hole[ne..nl) below n_new are refilled
    // with the live entries of the tail [n_new, n_old)
    const int d = nl - ne;
    if (tid >= ne && tid < nl) {
      const int h = hole[tid];
      if (h >= n_new) tail_hole[h - n_new] = 1;
      else low_hole[atomicAdd(&sh_nh, 1)] = h;
    }
    __syncthreads();
    if (tid < d && !tail_hole[tid]) mover_slot[atomicAdd(&sh_nm, 1)] = n_new + tid;
    __syncthreads();
    if (tid < sh_nm) {  // sh_nm == sh_nh; any pairing works
      const int32_t g = tail[n_old - 1 - mover_slot[tid]];  // d <= L: inside the prefetched tail
      const int dst = low_hole[tid];
      ids[dst] = g;
      pos[local_of(sv, g)] = dst;
    }
  }
  if (tid == 0) {
    sv.meta[seq].total = total + nk;
    sv.meta[seq].n_active = n_new;
    if (sh_err) sv.meta[seq].err |= 1;
    trace_mark(trace, 14);  // state: done
  }
}


}  // namespace nanospec
