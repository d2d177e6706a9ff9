// a1/a2 of the hot path: GPU-resident candidate-stream state.
//
// One CTA per sequence.  A call appends up to two id lists to the stream
// (init: prompt verbatim, then tuple(prefill union) -- Eq. 3; update:
// tuple(C_draft) then tuple(C_ver) -- Eq. 4), maintaining
//   ring[W]  the last W stream slots (slot = position % W),
//   cnt[V]   how often each id occurs in the window,
//   bitmap   bit g set  <=>  cnt[g] > 0        (I = Unique(Suffix(S, W)), Eq. 5)
// and keeps I in ids[0, n_active) as a stable slot table (pos[g] = slot of g):
// the general path (init, long lists, rule R2) recompacts ascending by a block
// prefix sum over the bitmap; the per-step fast path changes only the slots of
// the ids that leave / enter the window (O(changes), not O(V)).  Everything
// stays on the device; no host sync.
//
// tuple(.) deduplication (first occurrence within one list) uses first[V]:
// atomicMin of the list position per id, then "keep iff first[e] == i".
#include "common.cuh"
#include "internal.h"
#include "state_fast.cuh"

namespace nanospec {

namespace {

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
      if (off < sv.w_max) {
        ids[off] = sv.n_shards <= 1 ? l : l * sv.n_shards + sv.rank;
        if (sv.pos) sv.pos[(long long)seq * sv.v_local + l] = off;
      }
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

__global__ void __launch_bounds__(kFastThreads) state_update_fast_kernel(AppendArgs args, unsigned long long* trace) {
  __shared__ UpdSmem sm;
  // Programmatic dependent launch: this kernel may start while the previous
  // kernel on the stream (e.g. the last head call) is still running; it must
  // not touch the state before that kernel has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) trace_mark(trace, 9);  // state: start
  // let the dependent head kernel get resident and run its prologue meanwhile
  // (the launcher records this stream, so that head waits for this grid before
  // reading the state: note_update_launch)
  asm volatile("griddepcontrol.launch_dependents;");
  NoPublish hook;
  update_fast(args, args.seq0 + blockIdx.x, sm, hook, trace);
}

}  // namespace

bool state_fast_path(const StateView& sv, int reset, long long a_len, int a_dedup, long long b_len, int b_dedup) {
  const long long L = a_len + b_len;
  return !reset && sv.rule == 0 && sv.pos && a_dedup && b_dedup && L <= kFastThreads && L <= sv.w_max;
}

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
  if (!reset && sv.rule == 0 && sv.pos && a_dedup && b_dedup && L <= kFastThreads && L <= sv.w_max) {
    if (!a) args.a.len = 0;
    if (!b) args.b.len = 0;
    const size_t smem = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nseq);
    cfg.blockDim = dim3(kFastThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    unsigned long long* tr = trace_buffer();
    note_update_launch(stream);
    cudaError_t e = cudaLaunchKernelEx(&cfg, state_update_fast_kernel, args, tr);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      state_update_fast_kernel<<<nseq, kFastThreads, smem, stream>>>(args, tr);
      e = cudaGetLastError();
    }
    return e;
  }
  state_append_kernel<<<nseq, 512, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace nanospec
