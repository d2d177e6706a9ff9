// a1/a2 of the hot path: GPU-resident candidate-stream state.
//
// One CTA per sequence.  A call appends up to two id lists to the stream
// (init: prompt verbatim, then tuple(prefill union) -- Eq. 3; update:
// tuple(C_draft) then tuple(C_ver) -- Eq. 4), maintaining
//   ring[W]  the last W stream slots (slot = position % W),
//   cnt[V]   how often each id occurs in the window,
//   bitmap   bit g set  <=>  cnt[g] > 0        (I = Unique(Suffix(S, W)), Eq. 5)
// and finally recompacts I into ids[] in ascending id by a block prefix sum
// over the bitmap.  Everything stays on the device; no host sync.
//
// tuple(.) deduplication (first occurrence within one list) uses first[V]:
// atomicMin of the list position per id, then "keep iff first[e] == i".
#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

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

// Rule R1 (Eq. 5 literally).  Appends `list` (already offset for this sequence).
__device__ void append_window(const StateView& sv, int seq, const int32_t* list, long long len, int dedup,
                              long long& total, int* sh_scan, int* sh_err) {
  const int tid = threadIdx.x, bs = blockDim.x;
  const int W = sv.w_max;
  int32_t* ring = sv.ring + (long long)seq * W;
  int32_t* cnt = sv.cnt + (long long)seq * sv.v_local;
  uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
  int32_t* first = sv.first + (long long)seq * sv.vocab;

  if (dedup) {
    for (long long i = tid; i < len; i += bs) {
      int32_t e = list[i];
      if (e >= 0 && e < sv.vocab) atomicMin(&first[e], (int32_t)i);
    }
    __syncthreads();
  }
  const int CH = bs < W ? bs : W;  // <= W kept per chunk: distinct ring slots
  for (long long base = 0; base < len; base += CH) {
    const long long i = base + tid;
    int32_t e = -1;
    bool keep = false;
    if (tid < CH && i < len) {
      e = list[i];
      bool valid = e >= 0 && e < sv.vocab;
      if (!valid) *sh_err = 1;
      keep = valid && (!dedup || first[e] == (int32_t)i);
    }
    int nk;
    int pos = block_exclusive_scan(keep ? 1 : 0, sh_scan, &nk);
    long long p = total + pos;
    int slot = (int)(p % W);
    int32_t old = -1;
    if (keep) {
      if (p >= W) {
        old = ring[slot];
        if (old >= 0 && is_local(sv, old)) atomicSub(&cnt[local_of(sv, old)], 1);
      }
      ring[slot] = e;
      if (is_local(sv, e)) atomicAdd(&cnt[local_of(sv, e)], 1);
    }
    __syncthreads();
    if (keep) {
      if (old >= 0 && is_local(sv, old)) {
        int32_t l = local_of(sv, old);
        if (cnt[l] == 0) atomicAnd(&bm[l >> 5], ~(1u << (l & 31)));
      }
      if (is_local(sv, e)) {
        int32_t l = local_of(sv, e);
        atomicOr(&bm[l >> 5], 1u << (l & 31));
      }
    }
    total += nk;
    __syncthreads();
  }
  if (dedup) {
    for (long long i = tid; i < len; i += bs) {
      int32_t e = list[i];
      if (e >= 0 && e < sv.vocab) first[e] = kFirstSentinel;
    }
    __syncthreads();
  }
}

// Rule R2 (unique-FIFO).  Sequential over the (deduplicated) list; only used
// unsharded.  ring holds the last W pushes, `total` counts pushes.
__device__ void append_fifo(const StateView& sv, int seq, const int32_t* list, long long len, int dedup,
                            long long& total, int* sh_err) {
  const int tid = threadIdx.x, bs = blockDim.x;
  const int W = sv.w_max;
  int32_t* ring = sv.ring + (long long)seq * W;
  uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
  int32_t* first = sv.first + (long long)seq * sv.vocab;
  if (dedup) {
    for (long long i = tid; i < len; i += bs) {
      int32_t e = list[i];
      if (e >= 0 && e < sv.vocab) atomicMin(&first[e], (int32_t)i);
    }
    __syncthreads();
  }
  if (tid == 0) {
    long long t = total;
    for (long long i = 0; i < len; ++i) {
      int32_t e = list[i];
      if (e < 0 || e >= sv.vocab) { *sh_err = 1; continue; }
      if (dedup && first[e] != (int32_t)i) continue;
      if ((bm[e >> 5] >> (e & 31)) & 1u) continue;  // already queued: not pushed
      int slot = (int)(t % W);
      if (t >= W) {
        int32_t old = ring[slot];
        bm[old >> 5] &= ~(1u << (old & 31));
      }
      ring[slot] = e;
      bm[e >> 5] |= 1u << (e & 31);
      ++t;
    }
    total = t;
  }
  __syncthreads();
  // every thread needs the new total
  __shared__ long long sh_total;
  if (tid == 0) sh_total = total;
  __syncthreads();
  total = sh_total;
  if (dedup) {
    for (long long i = tid; i < len; i += bs) {
      int32_t e = list[i];
      if (e >= 0 && e < sv.vocab) first[e] = kFirstSentinel;
    }
    __syncthreads();
  }
}

// Ascending compaction of the bitmap into ids[] (Q4).
__device__ void compact(const StateView& sv, int seq, int* sh_scan) {
  const int tid = threadIdx.x, bs = blockDim.x;
  const uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
  int32_t* ids = sv.ids + (long long)seq * sv.w_max;
  const int per = (sv.words + bs - 1) / bs;
  const int w0 = tid * per;
  const int w1 = min(sv.words, w0 + per);
  int c = 0;
#pragma unroll 8
  for (int w = w0; w < w1; ++w) c += __popc(__ldcg(bm + w));
  int n;
  int off = block_exclusive_scan(c, sh_scan, &n);
  for (int w = w0; w < w1; ++w) {
    uint32_t b = __ldcg(bm + w);
    while (b) {
      int bit = __ffs(b) - 1;
      b &= b - 1;
      int32_t l = (w << 5) + bit;
      if (off < sv.w_max) ids[off] = sv.n_shards <= 1 ? l : l * sv.n_shards + sv.rank;
      ++off;
    }
  }
  if (tid == 0) sv.meta[seq].n_active = n;
}

__global__ void __launch_bounds__(512) state_append_kernel(AppendArgs args) {
  __shared__ int sh_scan[40];
  __shared__ int sh_err;
  const StateView& sv = args.sv;
  const int seq = args.seq0 + blockIdx.x;
  const int tid = threadIdx.x, bs = blockDim.x;
  if (tid == 0) sh_err = 0;
  if (args.reset) {
    uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
    for (int w = tid; w < sv.words; w += bs) bm[w] = 0u;
    int32_t* ring = sv.ring + (long long)seq * sv.w_max;
    for (int s = tid; s < sv.w_max; s += bs) ring[s] = -1;
    if (sv.rule == 0) {
      int32_t* cnt = sv.cnt + (long long)seq * sv.v_local;
      for (int l = tid; l < sv.v_local; l += bs) cnt[l] = 0;
    }
  }
  __syncthreads();
  long long total = args.reset ? 0 : sv.meta[seq].total;
  const ListArg* lists[2] = {&args.a, &args.b};
  for (int q = 0; q < 2; ++q) {
    const ListArg& L = *lists[q];
    if (L.len <= 0 || L.ptr == nullptr) continue;
    const int32_t* p = L.ptr + (long long)(seq - args.seq0) * L.seq_stride;
    if (sv.rule == 0) append_window(sv, seq, p, L.len, L.dedup, total, sh_scan, &sh_err);
    else append_fifo(sv, seq, p, L.len, L.dedup, total, &sh_err);
  }
  __syncthreads();
  compact(sv, seq, sh_scan);
  if (tid == 0) {
    sv.meta[seq].total = total;
    if (args.reset) sv.meta[seq].err = sh_err;
    else if (sh_err) sv.meta[seq].err |= 1;
  }
}

// Per-step fast path of a2 (rule R1, no reset, both lists together <= 512
// ids and <= W_max, W_max <= 8192): one CTA per sequence.  The sequence's
// bitmap and the new ids are staged in shared memory; tuple(.) dedup is a
// shared-memory hash (min position per (list, id)); window counts are updated
// with returning atomics (all decrements, then all increments), so the bit
// flips are known without re-reading cnt; I is recompacted into shared memory
// and written back with coalesced stores.  Global round trips: {meta, bitmap,
// lists} -> ring slots -> decrements -> increments.
constexpr int kFastThreads = 512;
constexpr int kFastMaxW = 8192;
constexpr int kHashSlots = 2048;

__global__ void __launch_bounds__(kFastThreads) state_update_fast_kernel(AppendArgs args, unsigned long long* trace) {
  extern __shared__ uint32_t dyn[];
  __shared__ int32_t hkey[kHashSlots];
  __shared__ int32_t hpos[kHashSlots];
  __shared__ int sh_scan[40];
  __shared__ long long sh_total;
  __shared__ int sh_err;
  if (threadIdx.x == 0) trace_mark(trace, 9);  // state: start
  // let the dependent head kernel get resident and run its prologue meanwhile
  asm volatile("griddepcontrol.launch_dependents;");
  const StateView& sv = args.sv;
  const int seq = args.seq0 + blockIdx.x;
  const int tid = threadIdx.x;
  const int W = sv.w_max;
  uint32_t* bm_s = dyn;                                  // [words]
  int32_t* ids_s = reinterpret_cast<int32_t*>(dyn + sv.words);  // [W]
  const int la = (int)args.a.len, lb = (int)args.b.len;
  const int L = la + lb;
  uint32_t* bm = sv.bitmap + (long long)seq * sv.words;
  int32_t* ring = sv.ring + (long long)seq * W;
  int32_t* cnt = sv.cnt + (long long)seq * sv.v_local;
  if (tid == 0) { sh_total = sv.meta[seq].total; sh_err = 0; }
  int32_t e = -1;
  if (tid < la) e = args.a.ptr[(long long)(seq - args.seq0) * args.a.seq_stride + tid];
  else if (tid < L) e = args.b.ptr[(long long)(seq - args.seq0) * args.b.seq_stride + (tid - la)];
  {
    uint32_t tmp[32];  // all bitmap loads of this thread in flight at once (<= 16384 words)
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int w = tid + i * kFastThreads;
      if (w < sv.words) tmp[i] = bm[w];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int w = tid + i * kFastThreads;
      if (w < sv.words) bm_s[w] = tmp[i];
    }
  }
  for (int h = tid; h < kHashSlots; h += kFastThreads) { hkey[h] = -1; hpos[h] = 0x7fffffff; }
  __syncthreads();
  if (tid == 0) trace_mark(trace, 10);  // state: bitmap + lists staged
  // tuple(.): keep the first occurrence of every id within its own list
  const bool valid = tid < L && e >= 0 && e < sv.vocab;
  if (tid < L && !valid) sh_err = 1;
  int slot_h = -1;
  if (valid) {
    const int32_t key = e * 2 + (tid < la ? 0 : 1);
    int h = (int)(((uint32_t)key * 2654435761u) >> 21) & (kHashSlots - 1);
    while (true) {
      const int32_t old = atomicCAS(&hkey[h], -1, key);
      if (old == -1 || old == key) break;
      h = (h + 1) & (kHashSlots - 1);
    }
    atomicMin(&hpos[h], tid);
    slot_h = h;
  }
  __syncthreads();
  const bool keep = valid && hpos[slot_h] == tid;
  int nk;
  const int pos = block_exclusive_scan(keep ? 1 : 0, sh_scan, &nk);
  const long long total = sh_total;
  int slot = (int)(total % W) + pos;  // pos < W: one wrap at most
  if (slot >= W) slot -= W;
  int32_t old = -1;
  if (keep && total + pos >= W) old = ring[slot];
  // decrements for the evicted slots
  if (tid == 0) trace_mark(trace, 11);  // state: ring slots read
  if (old >= 0 && is_local(sv, old)) {
    const int32_t l = local_of(sv, old);
    if (atomicSub(&cnt[l], 1) == 1) atomicAnd(&bm_s[l >> 5], ~(1u << (l & 31)));
  }
  __syncthreads();
  // increments for the appended ids
  if (tid == 0) trace_mark(trace, 12);  // state: decrements done
  if (keep) {
    ring[slot] = e;
    if (is_local(sv, e)) {
      const int32_t l = local_of(sv, e);
      if (atomicAdd(&cnt[l], 1) == 0) atomicOr(&bm_s[l >> 5], 1u << (l & 31));
    }
  }
  __syncthreads();
  if (tid == 0) trace_mark(trace, 13);  // state: increments done
  // write the bitmap back; recompact I (ascending) into shared memory
  for (int w = tid; w < sv.words; w += kFastThreads) bm[w] = bm_s[w];
  const int per = (sv.words + kFastThreads - 1) / kFastThreads;
  const int w0 = tid * per, w1 = min(sv.words, w0 + per);
  int c = 0;
  for (int w = w0; w < w1; ++w) c += __popc(bm_s[w]);
  int n;
  int off = block_exclusive_scan(c, sh_scan, &n);
  if (tid == 0) trace_mark(trace, 15);  // state: bitmap written back, counts scanned
  for (int w = w0; w < w1; ++w) {
    uint32_t b = bm_s[w];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const int32_t l = (w << 5) + bit;
      if (off < W) ids_s[off] = sv.n_shards <= 1 ? l : l * sv.n_shards + sv.rank;
      ++off;
    }
  }
  __syncthreads();
  int32_t* ids = sv.ids + (long long)seq * W;
  const int nn = min(n, W);
  for (int j = tid; j < nn; j += kFastThreads) ids[j] = ids_s[j];  // coalesced
  if (tid == 0) {
    sv.meta[seq].total = total + nk;
    sv.meta[seq].n_active = n;
    if (sh_err) sv.meta[seq].err |= 1;
    trace_mark(trace, 14);  // state: done
  }
}

}  // namespace

cudaError_t launch_state_append(const StateView& sv, int seq0, int nseq, int reset,
                                const int32_t* a, long long a_len, long long a_stride, int a_dedup,
                                const int32_t* b, long long b_len, long long b_stride, int b_dedup,
                                cudaStream_t stream) {
  AppendArgs args;
  args.sv = sv;
  args.seq0 = seq0;
  args.reset = reset;
  args.a = ListArg{a, a_len, a_stride, a_dedup};
  args.b = ListArg{b, b_len, b_stride, b_dedup};
  const long long L = (a ? a_len : 0) + (b ? b_len : 0);
  if (!reset && sv.rule == 0 && a_dedup && b_dedup && L <= kFastThreads && L <= sv.w_max &&
      sv.words <= 16384 && sv.w_max <= kFastMaxW) {
    if (!a) args.a.len = 0;
    if (!b) args.b.len = 0;
    const size_t smem = sizeof(uint32_t) * ((size_t)sv.words + (size_t)sv.w_max);
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(state_update_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (16384 + kFastMaxW) * (int)sizeof(uint32_t));
      if (e != cudaSuccess) return e;
      attr = true;
    }
    state_update_fast_kernel<<<nseq, kFastThreads, smem, stream>>>(args, trace_buffer());
    return cudaGetLastError();
  }
  state_append_kernel<<<nseq, 512, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace nanospec
