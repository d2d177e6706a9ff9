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
  const uint16_t* packed;   // repacked rows or null: slot j of sequence b at packed + (b * max_ids + j) * ldp
  long long ldp;
};

// The paper's repack (T6 `repack_buf` P:451) as a measured variant:
// copy W_head[ids[j]] into packed row j for every slot j < n_active whose tag
// (the id the packed row holds) differs from ids[j] -- the delta of one update
// is the entering ids' slots -- and update the tags.  tags: int32 [w_max] per
// sequence, -1 initially.
cudaError_t launch_repack(const StateView& sv, int seq, const uint16_t* w, long long ldw, int d, uint16_t* packed,
                          long long ldp, int32_t* tags, cudaStream_t stream);

// Debug phase-trace buffer (nanospec_debug_set_trace); null = off.
unsigned long long* trace_buffer();

// Phase 1 (a3+a4): gathered contraction into the fp32 logits staging buffer.
cudaError_t launch_head_simt(const HeadProblem& p, int num_sms, cudaStream_t stream);
// Tensor-core head, a3+a4+a5 (head_split.cu): stream kernel A (gather +
// tcgen05 UMMA, K-split partial tiles to L2) chained by programmatic dependent
// launch to select kernel B (sum in K order, top-k, lse; writes the top-k, lse
// and, if p.logits != null, the debug logits).  Returns cudaErrorNotSupported
// when the shape is not covered (the caller falls back to SIMT only for AUTO).
cudaError_t launch_head_tc(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                           void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream);
size_t head_tc_scratch_bytes(int batch, int max_ids, int n);
struct AppendArgs;
// Fused step: the fast-path update `upd` (one sequence, rule R1) and the head of
// that sequence in one pair of launches (p.batch == 1, p points at that
// sequence; p.logits != null: the streamed rows' logits, nanospec_step_debug).
// cudaErrorNotSupported when the shape cannot be fused (caller: update + head).
// dry_run: only decide (cudaSuccess = would fuse), launch nothing.
cudaError_t launch_step_tc(const HeadProblem& p, const AppendArgs& upd, int k, float* topk_logit, int32_t* topk_id,
                           float* lse, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t stream,
                           bool dry_run = false);
// The state update kernel lets its dependent start early; a tensor-core head
// launched right after it on the same stream must then wait for it before
// reading the state.  note_update_launch records (device, stream);
// take_update_launch reports and clears it (head_split.cu).
void note_update_launch(cudaStream_t stream);
bool take_update_launch(cudaStream_t stream);
// Whether launch_state_append would take the per-step fast path for these lists.
bool state_fast_path(const StateView& sv, int reset, long long a_len, int a_dedup, long long b_len, int b_dedup);
// Debug: -1 default; 0 = launch the head's kernels without programmatic
// dependent launch (plain stream order); 1 = the stream kernel alone (timing
// only: no outputs).
void set_head_tc_mode(int mode);

// Phase 2 (a5): per (sequence, node) top-k by (value desc, id asc) + lse.
cudaError_t launch_select_topk(const HeadProblem& p, int k, float* topk_logit, int32_t* topk_id, float* lse,
                               cudaStream_t stream);

// Draft-tree bookkeeping (tree.cu).
struct TreeLevel {
  const float* front_score;   // [n_front] cumulative log-probabilities (null: the root, 0)
  const int32_t* front_index; // [n_front] pool indices of the frontier nodes (null: the root, parent -1)
  const float* topk_logit;    // [n_front][k] the head's top-k over I
  const int32_t* topk_id;
  const float* lse;           // [n_front] lse over I
  int n_front, k;
  float* pool_score;          // the node pool: children appended at pool_offset
  int32_t* pool_id;
  int32_t* pool_parent;
  int pool_offset;
  int n_next;                 // children kept as the next frontier
  int32_t* next_index;        // [n_next] pool indices, best first
  float* next_score;          // [n_next]
};
cudaError_t launch_tree_expand(const TreeLevel& t, cudaStream_t stream);
cudaError_t launch_tree_rerank(const float* score, const int32_t* id, int n, int m, int32_t* out_index,
                               int32_t* out_id, cudaStream_t stream);

cudaError_t launch_merge_topk(const float* cand_logit, const int32_t* cand_id, const float* cand_lse,
                              int n_shards, int n_rows, int k, float* out_logit, int32_t* out_id, float* out_lse,
                              cudaStream_t stream);

}  // namespace nanospec
