// Internal (non-ABI) launchers of the NanoSpec CUDA path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace nanospec {

cudaError_t launch_state_append(const StateView& sv, int seq0, int nseq, int reset,
                                const int32_t* a, long long a_len, long long a_stride, int a_dedup,
                                const int32_t* b, long long b_len, long long b_stride, int b_dedup,
                                cudaStream_t stream);

// Active rows of one head call: for sequence s, ids = ids_base + s*ids_stride,
// n_active = *(nact_base + s*nact_stride).
struct HeadProblem {
  const uint16_t* w;        // bf16 bits [rows x ldw]
  long long ldw;
  int d;
  const uint16_t* h;        // bf16 bits [batch x n x d]
  int n;
  int batch;
  const int32_t* ids_base;
  long long ids_stride;
  const int32_t* nact_base;
  long long nact_stride;
  int max_ids;              // ids capacity per sequence (row stride of logits)
  int n_shards;             // row(g) = g / n_shards
  float* logits;            // fp32 [batch x n x max_ids]
  unsigned long long* trace; // debug phase trace or null
};

// Debug phase-trace buffer (nanospec_debug_set_trace); null = off.
unsigned long long* trace_buffer();

// Phase 1 (a3+a4): gathered contraction into the fp32 logits staging buffer.
cudaError_t launch_head_simt(const HeadProblem& p, int num_sms, cudaStream_t stream);
// Tensor-core variant, a3+a4+a5 fused in one kernel (writes the top-k, lse and,
// if p.logits != null, the debug logits).  Returns cudaErrorNotSupported when
// the shape is not covered (the caller falls back to SIMT only for AUTO).
cudaError_t launch_head_tc(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                           void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream);
size_t head_tc_scratch_bytes(int batch, int max_ids, int n);
struct AppendArgs;
// Fused step: the fast-path update `upd` (one sequence, rule R1) and the head of
// that sequence in one launch (p.batch == 1, p points at that sequence).
// cudaErrorNotSupported when the shape cannot be fused (caller: update + head).
// dry_run: only decide (cudaSuccess = would fuse), launch nothing.
cudaError_t launch_step_tc(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit, int32_t* topk_id,
                           float* lse, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream,
                           bool dry_run = false);
// Pair-split tensor-core head (head_pair.cu): the one-wave regime (every row
// tile resident at once).  Scratch shared with head_tc.cu's layout.
constexpr int kMaxPairSMs = 256;
struct PairScratch {
  uint2* cand;          // pair_cand_bytes(n): row keys, ids, tile maxima and lse partials
  unsigned* node_ctr;   // [batch * n], zero between launches
  unsigned* grid_word;  // grid barrier word (generation << 12 | arrivals), shared with head_tc.cu
  unsigned* step_ctr;   // fused: publication generation
  unsigned* arrive_ctr; // fused: zero between launches
  uint32_t* stale;      // fused: [max_ids / 32]
  int32_t* enter_ids;   // fused: [kFastThreads]
  int* enter_meta;      // fused: [4]
};
size_t pair_cand_bytes(int n);
cudaError_t launch_head_pair(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                             const PairScratch& s, int num_sms, cudaStream_t stream);
cudaError_t launch_step_pair(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit,
                             int32_t* topk_id, float* lse, const PairScratch& s, int num_sms, cudaStream_t stream,
                             bool dry_run);
void set_head_pair_enabled(int on);
// Two-kernel head (head_split.cu): stream kernel A (gather + UMMA + partials to
// L2) and select kernel B (sum + top-k + lse), chained by programmatic
// dependent launch.  Scratch: head_split_scratch_bytes at the start of `scratch`.
size_t head_split_scratch_bytes(int batch, int max_ids, int n);
cudaError_t launch_head_split(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                              void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream);
cudaError_t launch_step_split(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit,
                              int32_t* topk_id, float* lse, void* scratch, size_t scratch_bytes, int num_sms,
                              cudaStream_t stream, bool dry_run);
void set_head_split_pdl(int on);
// The fused step through the split head only (the debug-logits call); scratch as launch_step_tc.
cudaError_t launch_step_split_only(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit,
                                   int32_t* topk_id, float* lse, void* scratch, size_t scratch_bytes, int num_sms,
                                   cudaStream_t stream);
// Whether launch_state_append would take the per-step fast path for these lists.
bool state_fast_path(const StateView& sv, int reset, long long a_len, int a_dedup, long long b_len, int b_dedup);
// Debug: force the fused head's reduction mode (-1 auto, 0 finisher, 1 poll, 2 cluster).
void set_head_tc_mode(int mode);
// Debug: cap the cluster (K-split) size the cluster / fused modes try (0 = no cap).
void set_head_tc_cluster_cap(int s);

// Phase 2 (a5): per (sequence, node) top-k by (value desc, id asc) + lse.
cudaError_t launch_select_topk(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                               cudaStream_t stream);

cudaError_t launch_merge_topk(const float* cand_logit, const int32_t* cand_id, const float* cand_lse,
                              int n_shards, int n_rows, int k, float* out_logit, int32_t* out_id, float* out_lse,
                              cudaStream_t stream);

}  // namespace nanospec
