// EAGLE-2-style draft-tree bookkeeping on the device (the
// SelectDraftTokens / "append x_draft to draft tree" loop of Alg. 1, P:523-530,
// with the paper's tree of depth 5 and at most 60 draft tokens):
//
//   expand:  every frontier node f (cumulative log-probability s_f, 0 at the
//            root) gets its k children from the head's top-k over the active
//            set, child score s_f + (z - lse_f) -- the log-softmax over I
//             -- appended to a node pool; the n_next best children of
//            this level (score desc, pool index asc) become the next frontier;
//   rerank:  the m best nodes of the whole pool (same order) are the draft
//            tree; their tokens are C_draft for the state update.
//
// One CTA each, k * n_front <= 1024 children per level, pool <= 4096 nodes;
// ranking by counting in shared memory (every candidate by its own thread).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kTreeThreads = 1024;
constexpr int kPoolCap = 4096;

// a before b in (score desc, index asc); NaN never occurs (logits are finite,
// padding children carry -inf and rank last)
__device__ __forceinline__ bool before(float sa, int ia, float sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

__global__ void __launch_bounds__(kTreeThreads) tree_expand_kernel(TreeLevel t) {
  __shared__ float sc[1024];
  const int tid = threadIdx.x;
  const int nc = t.n_front * t.k;
  if (tid < nc) {
    const int f = tid / t.k, j = tid - f * t.k;
    const float ps = t.front_score ? t.front_score[f] : 0.f;
    const float z = t.topk_logit[(long long)f * t.k + j];
    const int32_t id = t.topk_id[(long long)f * t.k + j];
    const float s = (id >= 0) ? ps + (z - t.lse[f]) : -INFINITY;
    const int pi = t.pool_offset + tid;
    t.pool_score[pi] = s;
    t.pool_id[pi] = id;
    t.pool_parent[pi] = t.front_index ? t.front_index[f] : -1;
    sc[tid] = s;
  }
  __syncthreads();
  if (tid < nc) {
    const float me = sc[tid];
    int rk = 0;
    for (int e = 0; e < nc; ++e) rk += before(sc[e], e, me, tid) ? 1 : 0;
    if (rk < t.n_next) {
      t.next_index[rk] = t.pool_offset + tid;
      t.next_score[rk] = me;
    }
  }
}

__global__ void __launch_bounds__(kTreeThreads) tree_rerank_kernel(const float* score, const int32_t* id, int n,
                                                                  int m, int32_t* out_index, int32_t* out_id) {
  __shared__ float sc[kPoolCap];
  for (int e = threadIdx.x; e < n; e += kTreeThreads) sc[e] = score[e];
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += kTreeThreads) {
    const float me = sc[e];
    int rk = 0;
    for (int f = 0; f < n; ++f) rk += before(sc[f], f, me, e) ? 1 : 0;
    if (rk < m) {
      out_index[rk] = e;
      out_id[rk] = id[e];
    }
  }
}

}  // namespace

cudaError_t launch_tree_expand(const TreeLevel& t, cudaStream_t stream) {
  if (t.n_front < 1 || t.k < 1 || t.n_front * t.k > 1024 || t.n_next < 0 || t.n_next > t.n_front * t.k)
    return cudaErrorInvalidValue;
  tree_expand_kernel<<<1, kTreeThreads, 0, stream>>>(t);
  return cudaGetLastError();
}

cudaError_t launch_tree_rerank(const float* score, const int32_t* id, int n, int m, int32_t* out_index,
                               int32_t* out_id, cudaStream_t stream) {
  if (n < 1 || n > kPoolCap || m < 1 || m > n) return cudaErrorInvalidValue;
  tree_rerank_kernel<<<1, kTreeThreads, 0, stream>>>(score, id, n, m, out_index, out_id);
  return cudaGetLastError();
}

}  // namespace nanospec
