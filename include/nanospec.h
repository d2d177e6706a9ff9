/*
 * nanospec.h -- C ABI of the B200-native NanoSpec hot path
 * (arxiv 2605.26444, "NanoSpec: Accelerating Speculative Decoding using
 * Minimalist In-Context Vocabularies").  P:n = PAPER.md line n, S:n = SPEC.md
 * line n; Q-numbers are the readings listed in DESIGN.md section 3.
 *
 * The path:
 *   a1  state init     S0 = prompt (+) tuple(U_i TopK_pre(z_i))          Eq. 3
 *   a2  state update   S  = S (+) tuple(C_draft) (+) tuple(C_ver)         Eq. 4
 *                      I  = Unique(Suffix(S, W_max))                      Eq. 5
 *                      kept GPU-resident as a bitmap + compacted id list
 *   a3  gather of the active rows W_head[I, :]
 *   a4  z' = W_head[I, :] h   (bf16 in, fp32 accumulate)                   Eq. 2
 *   a5  per-node top-k over z', mapped back to global ids through I (+lse) P:527-528
 *
 * Conventions (all entry points):
 *   - Ownership: the CALLER owns every device buffer (weights, hidden states,
 *     outputs, state workspace, head scratch).  The library owns only the small
 *     host handle behind nanospec_state (malloc'd in create, freed in destroy).
 *   - Layout: row-major everywhere.  bf16 arrays are passed as `const void*`
 *     (IEEE bfloat16 bit patterns); their rows must be 16-byte aligned
 *     (d_model % 8 == 0, ldw % 8 == 0, base pointer 16-byte aligned).
 *   - Asynchrony: every call except nanospec_state_read / nanospec_state_check
 *     is asynchronous on `stream`, never synchronises the host and never copies
 *     the active-set size to the host.  Update -> head ordering is
 *     stream order.  The tensor-core head kernels are launched with
 *     programmatic dependent launch and read their INPUTS (state, hidden
 *     states, update lists) as soon as the previous kernel on the stream lets
 *     them start; they wait for that kernel to complete only before writing
 *     the head scratch.  This library's select kernels let a dependent start
 *     only after the state's last writer completed; its state update kernel
 *     lets the next kernel start early, and the library then makes the next
 *     tensor-core head launched on that stream wait before reading the state.
 *     A caller mixing in its own programmatic-launch kernels that
 *     produce these inputs must not trigger (griddepcontrol.launch_dependents)
 *     before those outputs are written.  Ordinary kernels, copies and event
 *     waits need nothing.
 *   - Errors: host-side validation -> NANOSPEC_EINVAL (nothing launched);
 *     launch failure -> NANOSPEC_ECUDA.  An out-of-range token id cannot be
 *     checked on the host: the kernels drop it (it is never appended) and set a
 *     per-sequence device flag that nanospec_state_check reports as
 *     NANOSPEC_EDEVICE.  No C++ exception crosses this ABI.
 *   - Threading: a state handle is single-writer; distinct handles may
 *     be used concurrently on different streams.
 */
#ifndef NANOSPEC_H_
#define NANOSPEC_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

#define NANOSPEC_ABI_VERSION 1
#define NANOSPEC_MAX_K 32       /* draft top-k: 1 <= k <= 32 (Q9)                  */
#define NANOSPEC_MAX_NODES 256  /* draft-tree nodes per call: 1 <= n <= 256         */

typedef struct nanospec_state_s* nanospec_state;

typedef enum {
  NANOSPEC_OK = 0,
  NANOSPEC_EINVAL = 1,       /* bad argument (null, range, alignment, size)          */
  NANOSPEC_EEMPTY = 2,       /* empty prompt ("empty prompt")                 */
  NANOSPEC_ECUDA = 3,        /* a CUDA runtime call or launch failed                 */
  NANOSPEC_EDEVICE = 4,      /* a kernel saw an out-of-range token id        */
  NANOSPEC_EUNSUPPORTED = 5  /* valid but not implemented (e.g. R2 + vocab sharding) */
} nanospec_status;

/* Which reading of the window rule the state maintains (Q1). */
typedef enum {
  NANOSPEC_RULE_WINDOW = 0,      /* R1, default: Eq. 5 literally -- I is the set of
                                    distinct ids among the last W_max stream slots   */
  NANOSPEC_RULE_UNIQUE_FIFO = 1  /* R2: only ids not already in the queue are pushed;
                                    FIFO eviction at W_max            */
} nanospec_rule;

/* Contraction kernel choice for the head (a3+a4).  AUTO picks the tensor-core
 * path (tcgen05) when compiled in, else the CUDA-core path. */
typedef enum {
  NANOSPEC_HEAD_AUTO = 0,
  NANOSPEC_HEAD_SIMT = 1,  /* CUDA cores, 16-byte vector loads, fp32 FMA          */
  NANOSPEC_HEAD_TC = 2     /* 5th-gen tensor cores (tcgen05.mma, TMEM accumulators) */
} nanospec_head_impl;

int32_t nanospec_abi_version(void);
const char* nanospec_status_str(nanospec_status s);

/* ------------------------------------------------------------------ state --
 * Device workspace for `batch` independent sequences, each with vocabulary
 * `vocab` and window `w_max` (D1-D4 of SURVEY 2.2).  Per sequence it holds:
 *   bitmap  uint32[ceil(V_local/32)]  membership of I (the paper's `token_ids`,
 *                                     16,032 B at V = 128256, T6 P:449, Q14)
 *   ids     int32[w_max]              I as a slot table (first n_active valid): stable slots,
 *                                     an id keeps its slot while it stays in I; the general
 *                                     path (init) lays it out ascending (Q4)
 *   pos     int32[V_local]            R1 only: slot of every active id
 *   ring    int32[w_max]              the last w_max stream slots (R1) / queue (R2)
 *   cnt     int32[V_local]            R1 only: occurrences of each id in the window
 *   first   int32[vocab]              dedup scratch for tuple(.) (Eq. 3/4)
 *   meta    {int64 total; int32 n_active; int32 err}
 * Vocab-parallel sharding (n_shards > 1): the ring is replicated and every rank
 * receives the same update lists, but bitmap/ids/cnt cover only ids g with
 * g % n_shards == shard_rank; the head then reads local weight row g / n_shards.
 * V_local = ceil((vocab - shard_rank) / n_shards).  (0, 1) = unsharded.
 * Returns 0 on invalid arguments. */
size_t nanospec_state_workspace_bytes(int32_t vocab, int32_t w_max, int32_t batch, nanospec_rule rule,
                                      int32_t shard_rank, int32_t n_shards);

/* Creates a handle over caller-owned `d_workspace` (>= workspace_bytes, 256-B
 * aligned) and clears it asynchronously on `stream` (every sequence starts with
 * an empty stream and I = {}).  EINVAL on bad sizes / pointers, EUNSUPPORTED for
 * R2 with n_shards > 1. */
nanospec_status nanospec_state_create(nanospec_state* out, int32_t vocab, int32_t w_max, int32_t batch,
                                      nanospec_rule rule, int32_t shard_rank, int32_t n_shards,
                                      void* d_workspace, size_t ws_bytes, cudaStream_t stream);
nanospec_status nanospec_state_destroy(nanospec_state st);

/* a1 -- Eq. 3: resets sequence `seq` and sets
 *   S0 = (x_1..x_L) (+) tuple(flatten_rowmajor(prefill_topk)),
 * prompt ids verbatim (duplicates kept), the [L x k_pre] candidate table
 * deduplicated by first occurrence within itself only (Q3), then
 * I = Unique(Suffix(S0, W_max)) (window applies immediately, Q7).
 *   d_prompt       int32[prompt_len] device; prompt_len == 0 -> EEMPTY
 *   d_prefill_topk int32[prompt_len x k_pre] device, rank order; NULL iff k_pre == 0
 * Ids outside [0, vocab) are dropped and flagged (see Errors). */
nanospec_status nanospec_state_init(nanospec_state st, int32_t seq, const int32_t* d_prompt, int64_t prompt_len,
                                    const int32_t* d_prefill_topk, int32_t k_pre, cudaStream_t stream);

/* a2 -- Eq. 4 + Eq. 5: appends tuple(C_draft) then tuple(C_ver)
 * (each deduplicated by first occurrence within itself, Q5) to sequence
 * `seq`'s stream, slides the window, updates the bitmap and recompacts I.
 *   d_draft_ids  int32[n_draft] device: the draft-tree tokens in node order (Q6)
 *   d_verify_topk int32[k_ver] device: the target's top-K_ver ids in rank order
 * Either list may be empty (NULL with count 0).  One launch, no host sync. */
nanospec_status nanospec_state_update(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                                      const int32_t* d_verify_topk, int32_t k_ver, cudaStream_t stream);

/* a2 for every sequence of the state in one launch (data-parallel decode):
 *   d_draft_ids [batch x n_draft], d_verify_topk [batch x k_ver]. */
nanospec_status nanospec_state_update_batch(nanospec_state st, const int32_t* d_draft_ids, int32_t n_draft,
                                            const int32_t* d_verify_topk, int32_t k_ver, cudaStream_t stream);

/* SYNCHRONISES `stream`; for tests and debugging.  Copies sequence `seq`'s
 * state to host buffers (any may be NULL): h_ids int32[w_max] (the slot table,
 * first *h_n_active valid; sort it for the canonical ascending order), h_bitmap uint32[ceil(V_local/32)], h_ring int32[w_max] (-1 = never
 * written), h_total = |S| (R1) or pushes (R2), h_err = the device flag. */
nanospec_status nanospec_state_read(const nanospec_state st, int32_t seq, int32_t* h_ids, int32_t* h_n_active,
                                    uint32_t* h_bitmap, int32_t* h_ring, int64_t* h_total, int32_t* h_err,
                                    cudaStream_t stream);

/* SYNCHRONISES `stream`; EDEVICE if any sequence's error flag is set. */
nanospec_status nanospec_state_check(const nanospec_state st, cudaStream_t stream);

/* Device pointers into the state, for callers that chain their own kernels
 * (e.g. the bench's dense comparator).  ids of sequence seq: int32[w_max];
 * n_active of sequence seq: one int32.  NULL on bad arguments. */
const int32_t* nanospec_state_ids_ptr(const nanospec_state st, int32_t seq);
const int32_t* nanospec_state_n_active_ptr(const nanospec_state st, int32_t seq);

/* ------------------------------------------------------------------- head --
 * Scratch the head needs for `batch` sequences of up to `max_ids` active rows
 * and `n_nodes` draft nodes (fp32 logits staging + split-K partials + counters).
 * The scratch must be zero-initialised ONCE before its first use (the kernels
 * leave their counters at zero on exit); 0 on invalid arguments. */
size_t nanospec_head_scratch_bytes(int32_t batch, int32_t max_ids, int32_t n_nodes);

/* a3+a4+a5 for every sequence of the state, one call:
 *   z'[b][i][j] = sum_c W_head[row(ids_b[j])][c] * H[b][i][c]   (fp32 accumulate)
 * then per (b, i) the k largest z' ranked by (value desc, global id asc)
 * (Q10), as global token ids.  Full-vocabulary logits are never materialised.
 *   d_w_head      bf16 [V_local x ldw] device; row(g) = g / n_shards (g when unsharded)
 *   d_model       hidden size d (% 8 == 0); ldw >= d, % 8 == 0
 *   d_hidden      bf16 [batch x n_nodes x d_model] device
 *   k             1..NANOSPEC_MAX_K; slots beyond n_active are (-inf, -1)
 *   d_topk_logit  fp32 [batch x n_nodes x k], d_topk_id int32 [batch x n_nodes x k]
 *   d_lse         fp32 [batch x n_nodes] = log sum_{j in I} exp(z'_j) (Q13) or NULL
 *   d_debug_logits fp32 [batch x n_nodes x w_max] (first n_active of each row
 *                 valid) or NULL -- for tests; costs extra writes
 *   d_scratch     >= nanospec_head_scratch_bytes(batch, w_max, n_nodes)
 * Reads n_active and ids from device memory (no host sync). */
nanospec_status nanospec_draft_logits_topk(const nanospec_state st, const void* d_w_head, int32_t d_model,
                                           int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                           float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                           float* d_debug_logits, void* d_scratch, size_t scratch_bytes,
                                           cudaStream_t stream);

/* Same, choosing the contraction kernel explicitly (tests, bench). */
nanospec_status nanospec_draft_logits_topk_ex(const nanospec_state st, const void* d_w_head, int32_t d_model,
                                              int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                              float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                              float* d_debug_logits, void* d_scratch, size_t scratch_bytes,
                                              nanospec_head_impl impl, cudaStream_t stream);

/* The head over an explicit, caller-supplied ascending id list instead of a
 * state: a static set (FR-Spec-style 32k list) or [0, V) -- the dense
 * full-vocabulary head of Eq. 2, used as the dense comparator.
 *   d_ids int32[max_ids] device (global ids, row(g) = g / n_shards)
 *   d_n_ids one int32 on device: how many of d_ids are valid (<= max_ids)
 *   d_hidden bf16 [n_nodes x d_model]; outputs as above with batch = 1;
 *   d_debug_logits fp32 [n_nodes x max_ids] or NULL. */
nanospec_status nanospec_logits_topk_ids(const int32_t* d_ids, const int32_t* d_n_ids, int32_t max_ids,
                                         int32_t n_shards, const void* d_w_head, int32_t d_model, int64_t ldw,
                                         const void* d_hidden, int32_t n_nodes, int32_t k, float* d_topk_logit,
                                         int32_t* d_topk_id, float* d_lse, float* d_debug_logits,
                                         void* d_scratch, size_t scratch_bytes, nanospec_head_impl impl,
                                         cudaStream_t stream);

/* Vocab-parallel merge: the exact top-k and lse over the union
 * of n_shards disjoint shards' results.
 *   d_cand_logit fp32 [n_shards x n_rows x k], d_cand_id int32 [n_shards x n_rows x k]
 *   (padding (-inf, -1) allowed), d_cand_lse fp32 [n_shards x n_rows] or NULL.
 *   Outputs [n_rows x k] and [n_rows]; ties ranked by ascending id.
 *   n_shards * k <= 1024. */
nanospec_status nanospec_merge_topk(const float* d_cand_logit, const int32_t* d_cand_id, const float* d_cand_lse,
                                    int32_t n_shards, int32_t n_rows, int32_t k, float* d_out_logit,
                                    int32_t* d_out_id, float* d_out_lse, cudaStream_t stream);

/* One decode step of sequence `seq`, fused where possible: the state update
 * (Eq. 4 + Eq. 5; exactly nanospec_state_update) followed by the
 * restricted head over the UPDATED active set (Eq. 2 on I, P:205;
 * SelectDraftTokens P:527-528; exactly nanospec_draft_logits_topk on that
 * sequence).  Fused, the head's stream kernel gathers the rows of the
 * pre-update slots plus the update-list entries (a superset of the new I
 * known without waiting for the update) while one of its CTAs applies the
 * update, and the select kernel drops the rows that are not in the new I, so
 * the update is off the critical path (two kernels, no CTA waits for another
 * except the updating CTA for the streaming ones).  Shapes it cannot fuse
 * (rule R2, lists > 512 ids, more row tiles than SMs) run as update + head
 * with identical results.
 *   d_draft_ids int32[n_draft], d_verify_topk int32[k_ver]  (as state_update)
 *   d_hidden    bf16 [n_nodes x d_model] (this sequence's tree nodes)
 *   d_topk_logit / d_topk_id [n_nodes x k], d_lse [n_nodes] or NULL
 *   d_scratch  >= nanospec_head_scratch_bytes(1, w_max, n_nodes), zeroed once.
 * Errors as nanospec_state_update + nanospec_draft_logits_topk. */
nanospec_status nanospec_step(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                              const int32_t* d_verify_topk, int32_t k_ver, const void* d_w_head, int32_t d_model,
                              int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k, float* d_topk_logit,
                              int32_t* d_topk_id, float* d_lse, void* d_scratch, size_t scratch_bytes,
                              cudaStream_t stream);

/* nanospec_step that also writes the logits of every row the fused launch
 * streamed (tests: the fused launch's contraction checked element by element).
 *   d_debug_logits fp32 [n_nodes x (w_max + n_draft + k_ver)], row i:
 *     columns [0, w_max)          the PRE-update slots ids[0, n_old) (n_old = |I|
 *                                 before the step; later columns unspecified);
 *     columns [w_max, w_max + e)  the update-list entries, draft then verify.
 *   Only the rows in the updated active set feed the top-k / lse (the others
 *   are rows whose id left I, repeats, or ids that were already active).
 * EUNSUPPORTED when the step cannot run fused (then nothing is
 * done); otherwise exactly nanospec_step. */
nanospec_status nanospec_step_debug(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                                    const int32_t* d_verify_topk, int32_t k_ver, const void* d_w_head,
                                    int32_t d_model, int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                    float* d_topk_logit, int32_t* d_topk_id, float* d_lse, float* d_debug_logits,
                                    void* d_scratch, size_t scratch_bytes, cudaStream_t stream);

/* nanospec_step with HOST buffers (the end-to-end call): one host->device copy
 * of the packed inputs, the step, one device->host copy of the packed results,
 * all asynchronous on `stream` (pinned host memory for real overlap).
 *   h_in  = [hidden bf16 n_nodes x d_model][draft int32 n_draft][verify int32 k_ver]
 *   h_out = [topk_logit fp32 n_nodes x k][topk_id int32 n_nodes x k][lse fp32 n_nodes]
 *   d_io  : caller-owned device staging, >= nanospec_step_host_io_bytes(...)
 *   d_scratch as for nanospec_step.  h_out is valid after the stream syncs. */
size_t nanospec_step_host_io_bytes(int32_t n_nodes, int32_t d_model, int32_t n_draft, int32_t k_ver, int32_t k,
                                   size_t* in_bytes, size_t* out_bytes);
nanospec_status nanospec_step_host(nanospec_state st, int32_t seq, const void* h_in, int32_t n_draft, int32_t k_ver,
                                   const void* d_w_head, int32_t d_model, int64_t ldw, int32_t n_nodes, int32_t k,
                                   void* h_out, void* d_io, size_t io_bytes, void* d_scratch, size_t scratch_bytes,
                                   cudaStream_t stream);

/* nanospec_step_host for a pipeline of steps: the host->device copy runs on
 * `copy_stream` (it overlaps the previous step's kernels), the step and the
 * device->host copy on `stream`, ordered by two caller-created events.  A
 * caller alternates >= 2 staging slots (d_io, h_out, ev_in, ev_done each):
 * the copy into a slot first waits for ev_done, recorded by the previous step
 * that used the slot (an event never recorded means no wait); the step waits
 * for ev_in.  Results of a step are in its h_out once its ev_done completes.
 * Same layouts and results as nanospec_step_host; EINVAL on bad arguments or
 * copy_stream == stream, ECUDA on a failed copy / event call. */
nanospec_status nanospec_step_host_async(nanospec_state st, int32_t seq, const void* h_in, int32_t n_draft,
                                         int32_t k_ver, const void* d_w_head, int32_t d_model, int64_t ldw,
                                         int32_t n_nodes, int32_t k, void* h_out, void* d_io, size_t io_bytes,
                                         void* d_scratch, size_t scratch_bytes, cudaStream_t stream,
                                         cudaStream_t copy_stream, cudaEvent_t ev_in, cudaEvent_t ev_done);

/* 1 if nanospec_step with these sizes runs fused (the update inside the head's
 * stream kernel) on the current device, 0 if it runs as update + head (same
 * results).  Host-only query. */
int32_t nanospec_step_fused(const nanospec_state st, int32_t n_draft, int32_t k_ver, int32_t d_model,
                            int32_t n_nodes, int32_t k);

/* The paper's repack design (T6 `repack_buf`), built as a
 * measured alternative to the fused direct gather.
 * nanospec_repack: for every slot j < n_active of sequence `seq` whose tag
 * differs from ids[j], copy row W_head[ids[j]] (d_model bf16) into packed row
 * j and set the tag -- after an update that is the delta of the entering
 * ids.  d_packed bf16 [batch x w_max x ldp] and d_tags int32 [batch x w_max]
 * (all -1 initially) are caller-owned; run it on a copy stream and order the
 * packed head after it with an event.
 * nanospec_draft_logits_topk_packed: nanospec_draft_logits_topk (tensor-core
 * head) with every active row read from its packed slot instead of W_head --
 * contiguous rows; results identical.  Asynchronous; EINVAL on bad arguments,
 * EUNSUPPORTED where the tensor-core head does not take the shape. */
nanospec_status nanospec_repack(const nanospec_state st, int32_t seq, const void* d_w_head, int32_t d_model,
                                int64_t ldw, void* d_packed, int64_t ldp, int32_t* d_tags, cudaStream_t stream);
nanospec_status nanospec_draft_logits_topk_packed(const nanospec_state st, const void* d_packed, int32_t d_model,
                                                  int64_t ldp, const void* d_hidden, int32_t n_nodes, int32_t k,
                                                  float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                                  void* d_scratch, size_t scratch_bytes, cudaStream_t stream);

/* Draft-tree bookkeeping of one EAGLE-2-style round (the
 * SelectDraftTokens loop of Alg. 1; tree depth 5 / 60 draft tokens,
 * P:286), on the device so a whole round is one CUDA graph.
 *
 * nanospec_tree_expand: the k children of each of the n_front frontier nodes
 * (the head's top-k over I: d_topk_logit / d_topk_id [n_front x k], d_lse
 * [n_front]) are appended to a node pool at pool_offset with cumulative score
 * s_parent + (z - lse_parent) -- the log-softmax over the active set;
 * the root has d_front_score = d_front_index = NULL (score 0, parent -1).
 * The n_next best children of the level (score desc, pool index asc) are
 * written as the next frontier (d_next_index: pool indices, d_next_score).
 * Padding children (id -1) score -inf.  n_front * k <= 1024; pool_offset +
 * n_front * k <= pool_cap <= 4096.  Pool arrays: d_pool_score fp32,
 * d_pool_id / d_pool_parent int32 [pool_cap], caller-owned.
 *
 * nanospec_tree_rerank: the m best nodes of pool[0, pool_n) (same order):
 * d_out_index = their pool indices, d_out_id = their token ids (C_draft).
 * Both asynchronous on `stream`; EINVAL on bad sizes. */
nanospec_status nanospec_tree_expand(const float* d_front_score, const int32_t* d_front_index, int32_t n_front,
                                     const float* d_topk_logit, const int32_t* d_topk_id, const float* d_lse,
                                     int32_t k, float* d_pool_score, int32_t* d_pool_id, int32_t* d_pool_parent,
                                     int32_t pool_offset, int32_t pool_cap, int32_t n_next, int32_t* d_next_index,
                                     float* d_next_score, cudaStream_t stream);
nanospec_status nanospec_tree_rerank(const float* d_pool_score, const int32_t* d_pool_id, int32_t pool_n, int32_t m,
                                     int32_t* d_out_index, int32_t* d_out_id, cudaStream_t stream);

/* Debug: phase trace.  d_buf = device uint64[ctas * 16] (ctas >= 256; rows for
 * the stream kernel's grid plus the select kernel's) or NULL (off, the
 * default).  While set, the tensor-core head writes %globaltimer (ns) marks:
 * stream-kernel CTA b at d_buf[b*16 + e] (0 start, 1 dependency resolved, 7
 * row ids staged, 2 first loads, 3 last load landed, 4 last MMA done, 9
 * drained, 11 update published; 12/13/14/15 clock64), select-kernel CTA c at
 * row (stream grid + c) (0 start, 1 dependency resolved, 5 partials loaded,
 * 6/2 histogram, 7 candidates, 9 ranked, 4 done; 12 = 0xB marks the row;
 * scripts/split_dev.py prints them).  Process-wide; not thread-safe; for
 * profiling only. */
nanospec_status nanospec_debug_set_trace(unsigned long long* d_buf, int32_t ctas);

/* Debug: -1 (default) launches the tensor-core head's two kernels (stream
 * kernel A, select kernel B) with programmatic dependent launch, so each one's
 * prologue overlaps its predecessor; 0 launches them in plain stream order
 * (same results); 1 launches the stream kernel alone (timing breakdowns only:
 * no outputs are written).  Process-wide; tests and bench. */
nanospec_status nanospec_debug_set_head_mode(int32_t mode);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* NANOSPEC_H_ */
