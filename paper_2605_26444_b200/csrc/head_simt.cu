// a3+a4 on CUDA cores: gathered GEMV/skinny GEMM, fp32 accumulate.
//
//   logits[b][i][j] = sum_c W[row(ids_b[j])][c] * H[b][i][c]      (Eq. 2 on I)
//
// One warp per active row (the gather is a plain 16-byte-vectorised, coalesced
// read of that row straight from W_head: no repack buffer).  Lanes
// stride the row in 16-byte chunks, keep fp32 partial sums for a block of up to
// 8 nodes, and reduce across the warp with shuffles in a fixed order (so equal
// rows give bit-equal logits).  Used for narrow trees (n <= 8) and as the
// reference GPU path; the tensor-core kernel (head_tc.cu) covers wide trees.
#include "common.cuh"
#include "internal.h"

namespace nanospec {

namespace {

constexpr int kNB = 8;        // nodes per pass
constexpr int kThreads = 256;

__device__ __forceinline__ float dot8(const uint4& w, const uint4& h) {
  float s = bf16lo(w.x) * bf16lo(h.x);
  s = fmaf(bf16hi(w.x), bf16hi(h.x), s);
  s = fmaf(bf16lo(w.y), bf16lo(h.y), s);
  s = fmaf(bf16hi(w.y), bf16hi(h.y), s);
  s = fmaf(bf16lo(w.z), bf16lo(h.z), s);
  s = fmaf(bf16hi(w.z), bf16hi(h.z), s);
  s = fmaf(bf16lo(w.w), bf16lo(h.w), s);
  s = fmaf(bf16hi(w.w), bf16hi(h.w), s);
  return s;
}

__global__ void __launch_bounds__(kThreads) head_simt_kernel(HeadProblem p) {
  const int lane = lane_id();
  const long long gw = (long long)blockIdx.x * (kThreads / 32) + warp_id();
  const long long tw = (long long)gridDim.x * (kThreads / 32);
  const long long slots = (long long)p.batch * p.max_ids;
  const int chunks = p.d >> 3;
  for (long long slot = gw; slot < slots; slot += tw) {
    const int seq = (int)(slot / p.max_ids);
    const int j = (int)(slot - (long long)seq * p.max_ids);
    const int nact = p.nact_base[(long long)seq * p.nact_stride];
    if (j >= nact) continue;  // warp-uniform
    const int32_t g = p.ids_base[(long long)seq * p.ids_stride + j];
    const long long row = p.n_shards > 1 ? g / p.n_shards : g;
    const uint16_t* wrow = p.w + row * p.ldw;
    const uint16_t* hseq = p.h + (long long)seq * p.n * p.d;
    for (int nb = 0; nb < p.n; nb += kNB) {
      float acc[kNB];
#pragma unroll
      for (int q = 0; q < kNB; ++q) acc[q] = 0.f;
#pragma unroll 4
      for (int c = lane; c < chunks; c += 32) {
        const uint4 wv = ldg_stream(wrow + (long long)c * 8);
#pragma unroll
        for (int q = 0; q < kNB; ++q) {
          if (nb + q < p.n) {
            const uint4 hv = __ldg(reinterpret_cast<const uint4*>(hseq + (long long)(nb + q) * p.d) + c);
            acc[q] += dot8(wv, hv);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kNB; ++q) {
        float v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && nb + q < p.n) p.logits[((long long)seq * p.n + nb + q) * p.max_ids + j] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_head_simt(const HeadProblem& p, int num_sms, cudaStream_t stream) {
  long long warps_needed = (long long)p.batch * p.max_ids;
  long long blocks = (warps_needed + (kThreads / 32) - 1) / (kThreads / 32);
  long long cap = (long long)num_sms * 8;  // 8 CTAs x 8 warps per SM resident
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  head_simt_kernel<<<(unsigned)blocks, kThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace nanospec
