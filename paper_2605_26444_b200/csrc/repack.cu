// The paper's asynchronous repack (T6 `repack_buf`), built as
// a measured variant of the fused direct gather: after an update, the rows of
// the slots whose id changed (the entering ids) are copied from W_head into a
// dense [w_max x d] buffer, on whatever stream the caller picks (the paper's
// copy stream); the head then streams contiguous packed rows
// (nanospec_draft_logits_topk_packed).  One warp per slot: a slot whose tag
// equals its id is skipped after one 4-byte compare, a changed slot moves its
// d * 2 bytes with 16-byte loads and stores.
#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kRepackWarps = 8;

__global__ void __launch_bounds__(kRepackWarps * 32) repack_kernel(StateView sv, int seq, const uint16_t* w,
                                                                   long long ldw, int d, uint16_t* packed,
                                                                   long long ldp, int32_t* tags) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * kRepackWarps + warp;
  const int n = sv.meta[seq].n_active;
  if (j >= n || j >= sv.w_max) return;
  const int32_t g = sv.ids[(long long)seq * sv.w_max + j];
  int32_t* tag = tags + (long long)seq * sv.w_max + j;
  if (*tag == g) return;
  const long long row = sv.n_shards > 1 ? g / sv.n_shards : g;
  const uint4* src = reinterpret_cast<const uint4*>(w + row * ldw);
  uint4* dst = reinterpret_cast<uint4*>(packed + ((long long)seq * sv.w_max + j) * ldp);
  for (int c = lane; c < d / 8; c += 32) dst[c] = __ldcs(src + c);
  if (lane == 0) *tag = g;
}

}  // namespace

cudaError_t launch_repack(const StateView& sv, int seq, const uint16_t* w, long long ldw, int d, uint16_t* packed,
                          long long ldp, int32_t* tags, cudaStream_t stream) {
  const int blocks = (sv.w_max + kRepackWarps - 1) / kRepackWarps;
  repack_kernel<<<blocks, kRepackWarps * 32, 0, stream>>>(sv, seq, w, ldw, d, packed, ldp, tags);
  return cudaGetLastError();
}

}  // namespace nanospec
