// a5 of the hot path: per-node top-k over the active logits, mapped back to
// global token ids through I (SelectDraftTokens, Alg. 1),
// plus lse over the active set (softmax renormalised over I).
//
// One CTA per (sequence, node).  Exact radix select on an order-preserving
// 32-bit key (12 + 12 + 8 bits, early exit as soon as the threshold bin is
// taken whole), then the <= 32 winners are ordered by (value desc, id asc) with
// a warp bitonic sort.  Exact value ties at the threshold are resolved by a
// second radix select over the global ids (smallest ids first, Q10).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kSelThreads = 256;
constexpr int kStageCap = 32768;  // active rows staged in shared memory (128 KB)

struct SelOut {
  float* topk_logit;
  int32_t* topk_id;
  float* lse;
  int k;
};

struct Cand {
  uint32_t key;
  int32_t gid;
  float val;
  int valid;
};

__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  if (a.valid != b.valid) return a.valid;
  if (!a.valid) return false;
  if (a.key != b.key) return a.key > b.key;
  return a.gid < b.gid;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand r;
  r.key = __shfl_sync(0xffffffffu, c.key, src);
  r.gid = __shfl_sync(0xffffffffu, c.gid, src);
  r.val = __shfl_sync(0xffffffffu, c.val, src);
  r.valid = __shfl_sync(0xffffffffu, c.valid, src);
  return r;
}

// Bitonic sort of one candidate per lane, best first.
__device__ __forceinline__ Cand warp_sort(Cand me) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      Cand o = shfl_cand(me, lane ^ stride);
      const bool asc = (lane & size) == 0 || size == 32;
      const bool lower = (lane & stride) == 0;
      const bool take_best = (lower == asc);
      const bool o_first = before(o, me);
      if (take_best ? o_first : !o_first && before(me, o)) me = o;
    }
  }
  return me;
}

template <bool kStage>
__global__ void __launch_bounds__(kSelThreads) select_topk_kernel(HeadProblem p, SelOut o) {
  extern __shared__ float staged[];
  __shared__ int hist[4096];
  __shared__ int sh_scan[40];
  __shared__ float sh_red[40];
  __shared__ int sh_bin, sh_above, sh_n;
  __shared__ uint32_t cand_key[32];
  __shared__ int cand_idx[32];
  __shared__ float sh_max;

  const int tid = threadIdx.x, bs = blockDim.x;
  const int node = blockIdx.x, seq = blockIdx.y;
  const int m = p.nact_base[(long long)seq * p.nact_stride];
  const int32_t* ids = p.ids_base + (long long)seq * p.ids_stride;
  const float* row = p.logits + ((long long)seq * p.n + node) * p.max_ids;
  const long long ob = ((long long)seq * p.n + node) * o.k;
  const int kk = min(o.k, m);

  const float* vals = row;
  if (kStage) {
    for (int j = tid; j < m; j += bs) staged[j] = row[j];
    __syncthreads();
    vals = staged;
  }
  if (kk <= 0) {
    for (int r = tid; r < o.k; r += bs) { o.topk_logit[ob + r] = -INFINITY; o.topk_id[ob + r] = -1; }
    if (o.lse && tid == 0) o.lse[(long long)seq * p.n + node] = -INFINITY;
    return;
  }

  uint32_t prefix = 0u, pmask = 0u;
  int krem = kk;
  bool all_in = false;
  const int shifts[3] = {20, 8, 0};
  const int nbits[3] = {12, 12, 8};
  for (int ps = 0; ps < 3; ++ps) {
    const int nb = 1 << nbits[ps];
    const uint32_t mask = (uint32_t)nb - 1u;
    const int shift = shifts[ps];
    for (int b = tid; b < nb; b += bs) hist[b] = 0;
    __syncthreads();
    for (int j = tid; j < m; j += bs) {
      uint32_t key = float_key(vals[j]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & mask], 1);
    }
    __syncthreads();
    const int per = nb / bs;
    const int lo = tid * per;
    int s = 0;
    for (int b = lo; b < lo + per; ++b) s += hist[b];
    int T;
    const int excl = block_exclusive_scan(s, sh_scan, &T);
    const int above = T - excl - s;
    if (above < krem && above + s >= krem) {
      int acc = above;
      for (int b = lo + per - 1; b >= lo; --b) {
        if (acc + hist[b] >= krem) { sh_bin = b; sh_above = acc; break; }
        acc += hist[b];
      }
    }
    __syncthreads();
    const int b = sh_bin;
    krem -= sh_above;
    prefix |= (uint32_t)b << shift;
    pmask |= mask << shift;
    const int cnt_b = hist[b];
    __syncthreads();
    if (cnt_b == krem) { all_in = true; break; }
  }

  if (tid == 0) sh_n = 0;
  __syncthreads();
  for (int j = tid; j < m; j += bs) {
    uint32_t key = float_key(vals[j]);
    uint32_t mk = key & pmask;
    if (mk > prefix || (all_in && mk == prefix)) {
      int slot = atomicAdd(&sh_n, 1);
      cand_key[slot] = key;
      cand_idx[slot] = j;
    }
  }
  __syncthreads();
  if (!all_in) {
    // Exact value ties at the threshold: take the krem smallest global ids
    // among them (Q10; ids[] is a slot table, not sorted) -- a second radix
    // select, over the ids, restricted to the tied elements.
    const uint32_t tie_key = prefix;  // all 32 bits resolved
    uint32_t gpre = 0u, gmask = 0u;
    int need = krem;
    bool gall = false;
    for (int ps = 0; ps < 3 && !gall; ++ps) {
      const int nb = 1 << nbits[ps];
      const uint32_t mask = (uint32_t)nb - 1u;
      const int shift = shifts[ps];
      for (int b = tid; b < nb; b += bs) hist[b] = 0;
      __syncthreads();
      for (int j = tid; j < m; j += bs) {
        const uint32_t g = (uint32_t)ids[j];
        if (float_key(vals[j]) == tie_key && (g & gmask) == gpre) atomicAdd(&hist[(g >> shift) & mask], 1);
      }
      __syncthreads();
      const int per = nb / bs;
      const int lo = tid * per;
      int sv = 0;
      for (int b = lo; b < lo + per; ++b) sv += hist[b];
      int T;
      const int below = block_exclusive_scan(sv, sh_scan, &T);
      if (below < need && below + sv >= need) {
        int acc = below;
        for (int b = lo; b < lo + per; ++b) {
          if (acc + hist[b] >= need) { sh_bin = b; sh_above = acc; break; }
          acc += hist[b];
        }
      }
      __syncthreads();
      const int b = sh_bin;
      need -= sh_above;
      gpre |= (uint32_t)b << shift;
      gmask |= mask << shift;
      gall = hist[b] == need;
      __syncthreads();
    }
    for (int j = tid; j < m; j += bs) {
      const uint32_t key = float_key(vals[j]);
      const uint32_t g = (uint32_t)ids[j] & gmask;
      if (key == tie_key && (g < gpre || g == gpre)) {
        const int slot = atomicAdd(&sh_n, 1);
        cand_key[slot] = key;
        cand_idx[slot] = j;
      }
    }
    __syncthreads();
  }

  if (warp_id() == 0) {
    const int lane = lane_id();
    Cand c;
    c.valid = lane < kk;
    c.key = c.valid ? cand_key[lane] : 0u;
    c.gid = c.valid ? ids[cand_idx[lane]] : 0x7fffffff;
    c.val = c.valid ? vals[cand_idx[lane]] : -INFINITY;
    c = warp_sort(c);
    if (lane < o.k) {
      o.topk_logit[ob + lane] = c.valid ? c.val : -INFINITY;
      o.topk_id[ob + lane] = c.valid ? c.gid : -1;
    }
    if (lane == 0) sh_max = c.val;
  }
  if (o.lse) {
    __syncthreads();
    const float mx = sh_max;
    float s = 0.f;
    for (int j = tid; j < m; j += bs) s += expf(vals[j] - mx);
    s = block_sum(s, sh_red);
    if (tid == 0) o.lse[(long long)seq * p.n + node] = mx + logf(s);
  }
}

// Exact merge of per-shard top-k lists (vocab-parallel), rank by counting.
__global__ void merge_topk_kernel(const float* cl, const int32_t* ci, const float* cls, int S, int rows, int k,
                                  float* ol, int32_t* oi, float* olse) {
  __shared__ float v[1024];
  __shared__ int32_t id[1024];
  __shared__ int sh_nvalid;
  const int row = blockIdx.x, tid = threadIdx.x, N = S * k;
  if (tid == 0) sh_nvalid = 0;
  float myv = -INFINITY;
  int32_t myid = -1;
  if (tid < N) {
    const int s = tid / k, r = tid - (tid / k) * k;
    const long long off = ((long long)s * rows + row) * k + r;
    myv = cl[off];
    myid = ci[off];
    v[tid] = myv;
    id[tid] = myid;
  }
  __syncthreads();
  if (tid < N && myid >= 0) {
    atomicAdd(&sh_nvalid, 1);
    int rank = 0;
    for (int j = 0; j < N; ++j) {
      if (id[j] < 0) continue;
      if (v[j] > myv || (v[j] == myv && id[j] < myid)) ++rank;
    }
    if (rank < k) {
      ol[(long long)row * k + rank] = myv;
      oi[(long long)row * k + rank] = myid;
    }
  }
  __syncthreads();
  for (int r = sh_nvalid + tid; r < k; r += blockDim.x) {
    ol[(long long)row * k + r] = -INFINITY;
    oi[(long long)row * k + r] = -1;
  }
  if (olse && tid == 0) {
    float mx = -INFINITY;
    for (int s = 0; s < S; ++s) mx = fmaxf(mx, cls[(long long)s * rows + row]);
    float sum = 0.f;
    if (mx != -INFINITY)
      for (int s = 0; s < S; ++s) sum += expf(cls[(long long)s * rows + row] - mx);
    olse[row] = mx == -INFINITY ? -INFINITY : mx + logf(sum);
  }
}

}  // namespace

cudaError_t launch_select_topk(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                               cudaStream_t stream) {
  SelOut o{topk_logit, topk_id, lse, k};
  dim3 grid(p.n, p.batch);
  if (p.max_ids <= kStageCap) {
    size_t smem = (size_t)p.max_ids * sizeof(float);
    static bool attr_set[64] = {false};  // the attribute is per (function, device)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!attr_set[dev]) {
      cudaError_t e = cudaFuncSetAttribute(select_topk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kStageCap * (int)sizeof(float));
      if (e != cudaSuccess) return e;
      attr_set[dev] = true;
    }
    select_topk_kernel<true><<<grid, kSelThreads, smem, stream>>>(p, o);
  } else {
    select_topk_kernel<false><<<grid, kSelThreads, 0, stream>>>(p, o);
  }
  return cudaGetLastError();
}

cudaError_t launch_merge_topk(const float* cand_logit, const int32_t* cand_id, const float* cand_lse,
                              int n_shards, int n_rows, int k, float* out_logit, int32_t* out_id, float* out_lse,
                              cudaStream_t stream) {
  int N = n_shards * k;
  int threads = ((N + 31) / 32) * 32;
  if (threads < 32) threads = 32;
  merge_topk_kernel<<<n_rows, threads, 0, stream>>>(cand_logit, cand_id, cand_lse, n_shards, n_rows, k, out_logit,
                                                    out_id, out_lse);
  return cudaGetLastError();
}

}  // namespace nanospec
