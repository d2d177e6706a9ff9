// The C ABI (include/nanospec.h): argument validation, workspace layout and
// dispatch to the kernels.  No torch types anywhere; plain pointers + sizes.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>

#include "nanospec.h"
#include "common.cuh"
#include "internal.h"
#include "state_fast.cuh"

using namespace nanospec;

struct nanospec_state_s {
  StateView sv;
  void* ws;
  size_t ws_bytes;
};

namespace nanospec {
static unsigned long long* g_trace = nullptr;
unsigned long long* trace_buffer() { return g_trace; }
}  // namespace nanospec

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
  size_t meta, bitmap, ids, ring, cnt, pos, first, total;
};

bool geometry(int32_t vocab, int32_t w_max, int32_t batch, int rule, int32_t rank, int32_t n_shards,
              int32_t* v_local, int32_t* words) {
  if (vocab <= 0 || w_max <= 0 || batch <= 0) return false;
  if (rule != NANOSPEC_RULE_WINDOW && rule != NANOSPEC_RULE_UNIQUE_FIFO) return false;
  if (n_shards < 1 || rank < 0 || rank >= n_shards || rank >= vocab) return false;
  if (w_max > (1 << 28)) return false;
  *v_local = n_shards > 1 ? (vocab - rank + n_shards - 1) / n_shards : vocab;
  *words = (*v_local + 31) / 32;
  return true;
}

Layout layout(int32_t vocab, int32_t w_max, int32_t batch, int rule, int32_t v_local, int32_t words) {
  Layout L;
  size_t off = 0;
  L.meta = off;   off += align_up(sizeof(Meta) * (size_t)batch);
  L.bitmap = off; off += align_up(sizeof(uint32_t) * (size_t)words * batch);
  L.ids = off;    off += align_up(sizeof(int32_t) * (size_t)w_max * batch);
  L.ring = off;   off += align_up(sizeof(int32_t) * (size_t)w_max * batch);
  L.cnt = off;    off += rule == NANOSPEC_RULE_WINDOW ? align_up(sizeof(int32_t) * (size_t)v_local * batch) : 0;
  L.pos = off;    off += rule == NANOSPEC_RULE_WINDOW ? align_up(sizeof(int32_t) * (size_t)v_local * batch) : 0;
  L.first = off;  off += align_up(sizeof(int32_t) * (size_t)vocab * batch);
  L.total = off;
  return L;
}

int sm_count() {
  static int cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

inline nanospec_status cuda_status(cudaError_t e) { return e == cudaSuccess ? NANOSPEC_OK : NANOSPEC_ECUDA; }

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

size_t logits_bytes(int32_t batch, int32_t max_ids, int32_t n) {
  return align_up(sizeof(float) * (size_t)batch * (size_t)n * (size_t)max_ids);
}

nanospec_status run_head(HeadProblem hp, int32_t k, float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                         float* d_debug_logits, void* d_scratch, size_t scratch_bytes, nanospec_head_impl impl,
                         cudaStream_t stream) {
  const size_t lb = logits_bytes(hp.batch, hp.max_ids, hp.n);
  if (!d_scratch || scratch_bytes < nanospec_head_scratch_bytes(hp.batch, hp.max_ids, hp.n)) return NANOSPEC_EINVAL;
  char* rest = (char*)d_scratch + lb;
  size_t rest_bytes = scratch_bytes - lb;
  if (impl == NANOSPEC_HEAD_TC || impl == NANOSPEC_HEAD_AUTO) {
    hp.logits = d_debug_logits;  // fused kernel: logits only if the caller wants them
    cudaError_t e = launch_head_tc(hp, k, d_topk_logit, d_topk_id, d_lse, rest, rest_bytes, sm_count(), stream);
    if (e == cudaSuccess) return NANOSPEC_OK;
    if (e != cudaErrorNotSupported) return NANOSPEC_ECUDA;
    if (impl == NANOSPEC_HEAD_TC) return NANOSPEC_EUNSUPPORTED;
  }
  hp.logits = d_debug_logits ? d_debug_logits : (float*)d_scratch;
  cudaError_t e = launch_head_simt(hp, sm_count(), stream);
  if (e != cudaSuccess) return NANOSPEC_ECUDA;
  return cuda_status(launch_select_topk(hp, k, d_topk_logit, d_topk_id, d_lse, stream));
}

}  // namespace

extern "C" {

int32_t nanospec_abi_version(void) { return NANOSPEC_ABI_VERSION; }

const char* nanospec_status_str(nanospec_status s) {
  switch (s) {
    case NANOSPEC_OK: return "ok";
    case NANOSPEC_EINVAL: return "invalid argument";
    case NANOSPEC_EEMPTY: return "empty prompt";
    case NANOSPEC_ECUDA: return "CUDA error";
    case NANOSPEC_EDEVICE: return "out-of-range token id seen on device";
    case NANOSPEC_EUNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

size_t nanospec_state_workspace_bytes(int32_t vocab, int32_t w_max, int32_t batch, nanospec_rule rule,
                                      int32_t shard_rank, int32_t n_shards) {
  int32_t vl, words;
  if (!geometry(vocab, w_max, batch, rule, shard_rank, n_shards, &vl, &words)) return 0;
  return layout(vocab, w_max, batch, rule, vl, words).total;
}

nanospec_status nanospec_state_create(nanospec_state* out, int32_t vocab, int32_t w_max, int32_t batch,
                                      nanospec_rule rule, int32_t shard_rank, int32_t n_shards, void* d_workspace,
                                      size_t ws_bytes, cudaStream_t stream) {
  if (!out) return NANOSPEC_EINVAL;
  *out = nullptr;
  int32_t vl, words;
  if (!geometry(vocab, w_max, batch, rule, shard_rank, n_shards, &vl, &words)) return NANOSPEC_EINVAL;
  if (rule == NANOSPEC_RULE_UNIQUE_FIFO && n_shards > 1) return NANOSPEC_EUNSUPPORTED;
  Layout L = layout(vocab, w_max, batch, rule, vl, words);
  if (!d_workspace || ws_bytes < L.total || ((uintptr_t)d_workspace % kAlign) != 0) return NANOSPEC_EINVAL;
  nanospec_state st = (nanospec_state)malloc(sizeof(nanospec_state_s));
  if (!st) return NANOSPEC_EINVAL;
  char* base = (char*)d_workspace;
  StateView& sv = st->sv;
  sv.vocab = vocab;
  sv.v_local = vl;
  sv.w_max = w_max;
  sv.words = words;
  sv.rank = shard_rank;
  sv.n_shards = n_shards;
  sv.rule = (int32_t)rule;
  sv.batch = batch;
  sv.meta = (Meta*)(base + L.meta);
  sv.bitmap = (uint32_t*)(base + L.bitmap);
  sv.ids = (int32_t*)(base + L.ids);
  sv.ring = (int32_t*)(base + L.ring);
  sv.cnt = rule == NANOSPEC_RULE_WINDOW ? (int32_t*)(base + L.cnt) : nullptr;
  sv.pos = rule == NANOSPEC_RULE_WINDOW ? (int32_t*)(base + L.pos) : nullptr;
  sv.first = (int32_t*)(base + L.first);
  st->ws = d_workspace;
  st->ws_bytes = ws_bytes;
  cudaError_t e = cudaSuccess;
  // meta, bitmap, ids, cnt, pos -> 0; ring -> -1 (0xff bytes); first -> 0x7f7f7f7f
  if (e == cudaSuccess) e = cudaMemsetAsync(base + L.meta, 0, L.ring - L.meta, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(base + L.ring, 0xff, (L.cnt ? L.cnt : L.first) - L.ring, stream);
  if (e == cudaSuccess && rule == NANOSPEC_RULE_WINDOW) e = cudaMemsetAsync(base + L.cnt, 0, L.first - L.cnt, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(base + L.first, 0x7f, L.total - L.first, stream);
  if (e != cudaSuccess) {
    free(st);
    return NANOSPEC_ECUDA;
  }
  *out = st;
  return NANOSPEC_OK;
}

nanospec_status nanospec_state_destroy(nanospec_state st) {
  if (!st) return NANOSPEC_EINVAL;
  free(st);
  return NANOSPEC_OK;
}

nanospec_status nanospec_state_init(nanospec_state st, int32_t seq, const int32_t* d_prompt, int64_t prompt_len,
                                    const int32_t* d_prefill_topk, int32_t k_pre, cudaStream_t stream) {
  if (!st || seq < 0 || seq >= st->sv.batch || prompt_len < 0 || k_pre < 0) return NANOSPEC_EINVAL;
  if (prompt_len == 0) return NANOSPEC_EEMPTY;
  if (!d_prompt || (k_pre > 0 && !d_prefill_topk)) return NANOSPEC_EINVAL;
  if (prompt_len > 0x3fffffff || prompt_len * (int64_t)k_pre > 0x3fffffff) return NANOSPEC_EINVAL;
  return cuda_status(launch_state_append(st->sv, seq, 1, /*reset=*/1, d_prompt, prompt_len, 0, /*dedup=*/0,
                                         d_prefill_topk, prompt_len * (int64_t)k_pre, 0, /*dedup=*/1, stream));
}

nanospec_status nanospec_state_update(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                                      const int32_t* d_verify_topk, int32_t k_ver, cudaStream_t stream) {
  if (!st || seq < 0 || seq >= st->sv.batch || n_draft < 0 || k_ver < 0) return NANOSPEC_EINVAL;
  if ((n_draft > 0 && !d_draft_ids) || (k_ver > 0 && !d_verify_topk)) return NANOSPEC_EINVAL;
  return cuda_status(launch_state_append(st->sv, seq, 1, 0, d_draft_ids, n_draft, 0, 1, d_verify_topk, k_ver, 0, 1,
                                         stream));
}

nanospec_status nanospec_state_update_batch(nanospec_state st, const int32_t* d_draft_ids, int32_t n_draft,
                                            const int32_t* d_verify_topk, int32_t k_ver, cudaStream_t stream) {
  if (!st || n_draft < 0 || k_ver < 0) return NANOSPEC_EINVAL;
  if ((n_draft > 0 && !d_draft_ids) || (k_ver > 0 && !d_verify_topk)) return NANOSPEC_EINVAL;
  return cuda_status(launch_state_append(st->sv, 0, st->sv.batch, 0, d_draft_ids, n_draft, n_draft, 1,
                                         d_verify_topk, k_ver, k_ver, 1, stream));
}

nanospec_status nanospec_state_read(const nanospec_state st, int32_t seq, int32_t* h_ids, int32_t* h_n_active,
                                    uint32_t* h_bitmap, int32_t* h_ring, int64_t* h_total, int32_t* h_err,
                                    cudaStream_t stream) {
  if (!st || seq < 0 || seq >= st->sv.batch) return NANOSPEC_EINVAL;
  const StateView& sv = st->sv;
  Meta m;
  cudaError_t e = cudaMemcpyAsync(&m, sv.meta + seq, sizeof m, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess && h_ids)
    e = cudaMemcpyAsync(h_ids, sv.ids + (size_t)seq * sv.w_max, sizeof(int32_t) * sv.w_max, cudaMemcpyDeviceToHost,
                        stream);
  if (e == cudaSuccess && h_bitmap)
    e = cudaMemcpyAsync(h_bitmap, sv.bitmap + (size_t)seq * sv.words, sizeof(uint32_t) * sv.words,
                        cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess && h_ring)
    e = cudaMemcpyAsync(h_ring, sv.ring + (size_t)seq * sv.w_max, sizeof(int32_t) * sv.w_max,
                        cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return NANOSPEC_ECUDA;
  if (h_n_active) *h_n_active = m.n_active;
  if (h_total) *h_total = m.total;
  if (h_err) *h_err = m.err;
  return NANOSPEC_OK;
}

nanospec_status nanospec_state_check(const nanospec_state st, cudaStream_t stream) {
  if (!st) return NANOSPEC_EINVAL;
  const int B = st->sv.batch;
  Meta* h = (Meta*)malloc(sizeof(Meta) * (size_t)B);
  if (!h) return NANOSPEC_EINVAL;
  cudaError_t e = cudaMemcpyAsync(h, st->sv.meta, sizeof(Meta) * (size_t)B, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  nanospec_status r = e == cudaSuccess ? NANOSPEC_OK : NANOSPEC_ECUDA;
  for (int b = 0; r == NANOSPEC_OK && b < B; ++b)
    if (h[b].err) r = NANOSPEC_EDEVICE;
  free(h);
  return r;
}

const int32_t* nanospec_state_ids_ptr(const nanospec_state st, int32_t seq) {
  if (!st || seq < 0 || seq >= st->sv.batch) return nullptr;
  return st->sv.ids + (size_t)seq * st->sv.w_max;
}

const int32_t* nanospec_state_n_active_ptr(const nanospec_state st, int32_t seq) {
  if (!st || seq < 0 || seq >= st->sv.batch) return nullptr;
  return &st->sv.meta[seq].n_active;
}

size_t nanospec_head_scratch_bytes(int32_t batch, int32_t max_ids, int32_t n_nodes) {
  if (batch <= 0 || max_ids <= 0 || n_nodes <= 0 || n_nodes > NANOSPEC_MAX_NODES) return 0;
  return logits_bytes(batch, max_ids, n_nodes) + align_up(head_tc_scratch_bytes(batch, max_ids, n_nodes));
}

nanospec_status nanospec_draft_logits_topk_ex(const nanospec_state st, const void* d_w_head, int32_t d_model,
                                              int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                              float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                              float* d_debug_logits, void* d_scratch, size_t scratch_bytes,
                                              nanospec_head_impl impl, cudaStream_t stream) {
  if (!st || !d_w_head || !d_hidden || !d_topk_logit || !d_topk_id) return NANOSPEC_EINVAL;
  if (d_model <= 0 || d_model % 8 != 0 || ldw < d_model || ldw % 8 != 0) return NANOSPEC_EINVAL;
  if (n_nodes < 1 || n_nodes > NANOSPEC_MAX_NODES || k < 1 || k > NANOSPEC_MAX_K) return NANOSPEC_EINVAL;
  if (!aligned16(d_w_head) || !aligned16(d_hidden)) return NANOSPEC_EINVAL;
  if (impl != NANOSPEC_HEAD_AUTO && impl != NANOSPEC_HEAD_SIMT && impl != NANOSPEC_HEAD_TC) return NANOSPEC_EINVAL;
  const StateView& sv = st->sv;
  HeadProblem hp = {};
  hp.w = (const uint16_t*)d_w_head;
  hp.ldw = ldw;
  hp.d = d_model;
  hp.h = (const uint16_t*)d_hidden;
  hp.n = n_nodes;
  hp.batch = sv.batch;
  hp.ids_base = sv.ids;
  hp.ids_stride = sv.w_max;
  hp.nact_base = &sv.meta[0].n_active;
  hp.nact_stride = sizeof(Meta) / sizeof(int32_t);
  hp.max_ids = sv.w_max;
  hp.n_shards = sv.n_shards;
  hp.logits = nullptr;
  hp.trace = trace_buffer();
  return run_head(hp, k, d_topk_logit, d_topk_id, d_lse, d_debug_logits, d_scratch, scratch_bytes, impl, stream);
}

nanospec_status nanospec_draft_logits_topk(const nanospec_state st, const void* d_w_head, int32_t d_model,
                                           int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                           float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                           float* d_debug_logits, void* d_scratch, size_t scratch_bytes,
                                           cudaStream_t stream) {
  return nanospec_draft_logits_topk_ex(st, d_w_head, d_model, ldw, d_hidden, n_nodes, k, d_topk_logit, d_topk_id,
                                       d_lse, d_debug_logits, d_scratch, scratch_bytes, NANOSPEC_HEAD_AUTO, stream);
}

namespace {
nanospec_status step_impl(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                          const int32_t* d_verify_topk, int32_t k_ver, const void* d_w_head, int32_t d_model,
                          int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k, float* d_topk_logit,
                          int32_t* d_topk_id, float* d_lse, float* d_debug_logits, void* d_scratch,
                          size_t scratch_bytes, cudaStream_t stream) {
  if (!st || seq < 0 || seq >= st->sv.batch || n_draft < 0 || k_ver < 0) return NANOSPEC_EINVAL;
  if ((n_draft > 0 && !d_draft_ids) || (k_ver > 0 && !d_verify_topk)) return NANOSPEC_EINVAL;
  if (!d_w_head || !d_hidden || !d_topk_logit || !d_topk_id) return NANOSPEC_EINVAL;
  if (d_model <= 0 || d_model % 8 != 0 || ldw < d_model || ldw % 8 != 0) return NANOSPEC_EINVAL;
  if (n_nodes < 1 || n_nodes > NANOSPEC_MAX_NODES || k < 1 || k > NANOSPEC_MAX_K) return NANOSPEC_EINVAL;
  if (!aligned16(d_w_head) || !aligned16(d_hidden)) return NANOSPEC_EINVAL;
  const StateView& sv = st->sv;
  if (!d_scratch || scratch_bytes < nanospec_head_scratch_bytes(1, sv.w_max, n_nodes)) return NANOSPEC_EINVAL;
  HeadProblem hp = {};
  hp.w = (const uint16_t*)d_w_head;
  hp.ldw = ldw;
  hp.d = d_model;
  hp.h = (const uint16_t*)d_hidden;
  hp.n = n_nodes;
  hp.batch = 1;
  hp.ids_base = sv.ids + (size_t)seq * sv.w_max;
  hp.ids_stride = sv.w_max;
  hp.nact_base = &sv.meta[seq].n_active;
  hp.nact_stride = sizeof(Meta) / sizeof(int32_t);
  hp.max_ids = sv.w_max;
  hp.n_shards = sv.n_shards;
  hp.logits = d_debug_logits;
  hp.trace = trace_buffer();
  if (state_fast_path(sv, 0, d_draft_ids ? n_draft : 0, 1, d_verify_topk ? k_ver : 0, 1)) {
    AppendArgs upd;
    upd.sv = sv;
    upd.seq0 = seq;
    upd.reset = 0;
    upd.a = ListArg{d_draft_ids, d_draft_ids ? n_draft : 0, 0, 1};
    upd.b = ListArg{d_verify_topk, d_verify_topk ? k_ver : 0, 0, 1};
    const size_t lb = logits_bytes(1, sv.w_max, n_nodes);
    cudaError_t e = launch_step_tc(hp, upd, k, d_topk_logit, d_topk_id, d_lse, (char*)d_scratch + lb,
                                   scratch_bytes - lb, sm_count(), stream);
    if (e == cudaSuccess) return NANOSPEC_OK;
    if (e != cudaErrorNotSupported) return NANOSPEC_ECUDA;
  }
  if (d_debug_logits) return NANOSPEC_EUNSUPPORTED;  // the superset-row layout exists only in the fused launch
  hp.logits = nullptr;
  // not fusable: the update, then the head on that sequence (two launches)
  nanospec_status r = nanospec_state_update(st, seq, d_draft_ids, n_draft, d_verify_topk, k_ver, stream);
  if (r != NANOSPEC_OK) return r;
  return run_head(hp, k, d_topk_logit, d_topk_id, d_lse, nullptr, d_scratch, scratch_bytes, NANOSPEC_HEAD_AUTO,
                  stream);
}
}  // namespace

nanospec_status nanospec_step(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                              const int32_t* d_verify_topk, int32_t k_ver, const void* d_w_head, int32_t d_model,
                              int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k, float* d_topk_logit,
                              int32_t* d_topk_id, float* d_lse, void* d_scratch, size_t scratch_bytes,
                              cudaStream_t stream) {
  return step_impl(st, seq, d_draft_ids, n_draft, d_verify_topk, k_ver, d_w_head, d_model, ldw, d_hidden, n_nodes, k,
                   d_topk_logit, d_topk_id, d_lse, nullptr, d_scratch, scratch_bytes, stream);
}

nanospec_status nanospec_step_debug(nanospec_state st, int32_t seq, const int32_t* d_draft_ids, int32_t n_draft,
                                    const int32_t* d_verify_topk, int32_t k_ver, const void* d_w_head,
                                    int32_t d_model, int64_t ldw, const void* d_hidden, int32_t n_nodes, int32_t k,
                                    float* d_topk_logit, int32_t* d_topk_id, float* d_lse, float* d_debug_logits,
                                    void* d_scratch, size_t scratch_bytes, cudaStream_t stream) {
  if (!d_debug_logits) return NANOSPEC_EINVAL;
  return step_impl(st, seq, d_draft_ids, n_draft, d_verify_topk, k_ver, d_w_head, d_model, ldw, d_hidden, n_nodes, k,
                   d_topk_logit, d_topk_id, d_lse, d_debug_logits, d_scratch, scratch_bytes, stream);
}

size_t nanospec_step_host_io_bytes(int32_t n_nodes, int32_t d_model, int32_t n_draft, int32_t k_ver, int32_t k,
                                   size_t* in_bytes, size_t* out_bytes) {
  if (n_nodes < 1 || d_model <= 0 || n_draft < 0 || k_ver < 0 || k < 1) return 0;
  const size_t ib = align_up((size_t)n_nodes * d_model * 2 + (size_t)(n_draft + k_ver) * 4);
  const size_t ob = align_up((size_t)n_nodes * k * 8 + (size_t)n_nodes * 4);
  if (in_bytes) *in_bytes = ib;
  if (out_bytes) *out_bytes = ob;
  return ib + ob;
}

nanospec_status nanospec_step_host(nanospec_state st, int32_t seq, const void* h_in, int32_t n_draft, int32_t k_ver,
                                   const void* d_w_head, int32_t d_model, int64_t ldw, int32_t n_nodes, int32_t k,
                                   void* h_out, void* d_io, size_t io_bytes, void* d_scratch, size_t scratch_bytes,
                                   cudaStream_t stream) {
  if (!h_in || !h_out || !d_io) return NANOSPEC_EINVAL;
  size_t ib = 0, ob = 0;
  if (nanospec_step_host_io_bytes(n_nodes, d_model, n_draft, k_ver, k, &ib, &ob) == 0 || io_bytes < ib + ob)
    return NANOSPEC_EINVAL;
  char* din = (char*)d_io;
  char* dout = din + ib;
  const size_t hb = (size_t)n_nodes * d_model * 2;
  const size_t in_used = hb + (size_t)(n_draft + k_ver) * 4;
  const size_t out_used = (size_t)n_nodes * k * 8 + (size_t)n_nodes * 4;
  if (cudaMemcpyAsync(din, h_in, in_used, cudaMemcpyHostToDevice, stream) != cudaSuccess) return NANOSPEC_ECUDA;
  const int32_t* dd = n_draft > 0 ? (const int32_t*)(din + hb) : nullptr;
  const int32_t* dv = k_ver > 0 ? (const int32_t*)(din + hb) + n_draft : nullptr;
  float* ol = (float*)dout;
  int32_t* oi = (int32_t*)(dout + (size_t)n_nodes * k * 4);
  float* os = (float*)(dout + (size_t)n_nodes * k * 8);
  nanospec_status r = nanospec_step(st, seq, dd, n_draft, dv, k_ver, d_w_head, d_model, ldw, din, n_nodes, k, ol, oi,
                                    os, d_scratch, scratch_bytes, stream);
  if (r != NANOSPEC_OK) return r;
  return cuda_status(cudaMemcpyAsync(h_out, dout, out_used, cudaMemcpyDeviceToHost, stream));
}

nanospec_status nanospec_step_host_async(nanospec_state st, int32_t seq, const void* h_in, int32_t n_draft,
                                         int32_t k_ver, const void* d_w_head, int32_t d_model, int64_t ldw,
                                         int32_t n_nodes, int32_t k, void* h_out, void* d_io, size_t io_bytes,
                                         void* d_scratch, size_t scratch_bytes, cudaStream_t stream,
                                         cudaStream_t copy_stream, cudaEvent_t ev_in, cudaEvent_t ev_done) {
  if (!h_in || !h_out || !d_io || !ev_in || !ev_done || copy_stream == stream) return NANOSPEC_EINVAL;
  size_t ib = 0, ob = 0;
  if (nanospec_step_host_io_bytes(n_nodes, d_model, n_draft, k_ver, k, &ib, &ob) == 0 || io_bytes < ib + ob)
    return NANOSPEC_EINVAL;
  char* din = (char*)d_io;
  char* dout = din + ib;
  const size_t hb = (size_t)n_nodes * d_model * 2;
  const size_t in_used = hb + (size_t)(n_draft + k_ver) * 4;
  const size_t out_used = (size_t)n_nodes * k * 8 + (size_t)n_nodes * 4;
  // the previous step that used this staging slot (and h_out) is complete
  // before the copy overwrites it (an event never recorded: no wait)
  if (cudaStreamWaitEvent(copy_stream, ev_done, 0) != cudaSuccess) return NANOSPEC_ECUDA;
  if (cudaMemcpyAsync(din, h_in, in_used, cudaMemcpyHostToDevice, copy_stream) != cudaSuccess) return NANOSPEC_ECUDA;
  if (cudaEventRecord(ev_in, copy_stream) != cudaSuccess) return NANOSPEC_ECUDA;
  if (cudaStreamWaitEvent(stream, ev_in, 0) != cudaSuccess) return NANOSPEC_ECUDA;
  const int32_t* dd = n_draft > 0 ? (const int32_t*)(din + hb) : nullptr;
  const int32_t* dv = k_ver > 0 ? (const int32_t*)(din + hb) + n_draft : nullptr;
  float* ol = (float*)dout;
  int32_t* oi = (int32_t*)(dout + (size_t)n_nodes * k * 4);
  float* os = (float*)(dout + (size_t)n_nodes * k * 8);
  nanospec_status r = nanospec_step(st, seq, dd, n_draft, dv, k_ver, d_w_head, d_model, ldw, din, n_nodes, k, ol, oi,
                                    os, d_scratch, scratch_bytes, stream);
  if (r != NANOSPEC_OK) return r;
  if (cudaMemcpyAsync(h_out, dout, out_used, cudaMemcpyDeviceToHost, stream) != cudaSuccess) return NANOSPEC_ECUDA;
  return cuda_status(cudaEventRecord(ev_done, stream));
}

int32_t nanospec_step_fused(const nanospec_state st, int32_t n_draft, int32_t k_ver, int32_t d_model,
                            int32_t n_nodes, int32_t k) {
  if (!st || n_draft < 0 || k_ver < 0 || d_model <= 0 || d_model % 8 != 0) return 0;
  if (n_nodes < 1 || n_nodes > NANOSPEC_MAX_NODES || k < 1 || k > NANOSPEC_MAX_K) return 0;
  const StateView& sv = st->sv;
  if (!state_fast_path(sv, 0, n_draft, 1, k_ver, 1)) return 0;
  HeadProblem hp = {};
  hp.d = d_model;
  hp.ldw = d_model;
  hp.n = n_nodes;
  hp.batch = 1;
  hp.max_ids = sv.w_max;
  AppendArgs upd = {};
  upd.sv = sv;
  upd.a.len = n_draft;
  upd.b.len = k_ver;
  return launch_step_tc(hp, upd, k, nullptr, nullptr, nullptr, nullptr, 0, sm_count(), 0, true) == cudaSuccess ? 1 : 0;
}

nanospec_status nanospec_logits_topk_ids(const int32_t* d_ids, const int32_t* d_n_ids, int32_t max_ids,
                                         int32_t n_shards, const void* d_w_head, int32_t d_model, int64_t ldw,
                                         const void* d_hidden, int32_t n_nodes, int32_t k, float* d_topk_logit,
                                         int32_t* d_topk_id, float* d_lse, float* d_debug_logits, void* d_scratch,
                                         size_t scratch_bytes, nanospec_head_impl impl, cudaStream_t stream) {
  if (!d_ids || !d_n_ids || max_ids <= 0 || n_shards < 1) return NANOSPEC_EINVAL;
  if (!d_w_head || !d_hidden || !d_topk_logit || !d_topk_id) return NANOSPEC_EINVAL;
  if (d_model <= 0 || d_model % 8 != 0 || ldw < d_model || ldw % 8 != 0) return NANOSPEC_EINVAL;
  if (n_nodes < 1 || n_nodes > NANOSPEC_MAX_NODES || k < 1 || k > NANOSPEC_MAX_K) return NANOSPEC_EINVAL;
  if (!aligned16(d_w_head) || !aligned16(d_hidden)) return NANOSPEC_EINVAL;
  if (impl != NANOSPEC_HEAD_AUTO && impl != NANOSPEC_HEAD_SIMT && impl != NANOSPEC_HEAD_TC) return NANOSPEC_EINVAL;
  HeadProblem hp = {};
  hp.w = (const uint16_t*)d_w_head;
  hp.ldw = ldw;
  hp.d = d_model;
  hp.h = (const uint16_t*)d_hidden;
  hp.n = n_nodes;
  hp.batch = 1;
  hp.ids_base = d_ids;
  hp.ids_stride = 0;
  hp.nact_base = d_n_ids;
  hp.nact_stride = 0;
  hp.max_ids = max_ids;
  hp.n_shards = n_shards;
  hp.logits = nullptr;
  hp.trace = trace_buffer();
  return run_head(hp, k, d_topk_logit, d_topk_id, d_lse, d_debug_logits, d_scratch, scratch_bytes, impl, stream);
}

nanospec_status nanospec_debug_set_trace(unsigned long long* d_buf, int32_t ctas) {
  if (d_buf && ctas < 256) return NANOSPEC_EINVAL;
  g_trace = d_buf;
  return NANOSPEC_OK;
}

nanospec_status nanospec_debug_set_head_mode(int32_t mode) {
  if (mode < -1 || mode > 1) return NANOSPEC_EINVAL;
  set_head_tc_mode(mode);
  return NANOSPEC_OK;
}

nanospec_status nanospec_merge_topk(const float* d_cand_logit, const int32_t* d_cand_id, const float* d_cand_lse,
                                    int32_t n_shards, int32_t n_rows, int32_t k, float* d_out_logit,
                                    int32_t* d_out_id, float* d_out_lse, cudaStream_t stream) {
  if (!d_cand_logit || !d_cand_id || !d_out_logit || !d_out_id) return NANOSPEC_EINVAL;
  if (n_shards < 1 || n_rows < 1 || k < 1 || k > NANOSPEC_MAX_K || n_shards * k > 1024) return NANOSPEC_EINVAL;
  if (d_out_lse && !d_cand_lse) return NANOSPEC_EINVAL;
  return cuda_status(launch_merge_topk(d_cand_logit, d_cand_id, d_cand_lse, n_shards, n_rows, k, d_out_logit,
                                       d_out_id, d_out_lse, stream));
}

nanospec_status nanospec_repack(const nanospec_state st, int32_t seq, const void* d_w_head, int32_t d_model,
                                int64_t ldw, void* d_packed, int64_t ldp, int32_t* d_tags, cudaStream_t stream) {
  if (!st || seq < 0 || seq >= st->sv.batch || !d_w_head || !d_packed || !d_tags) return NANOSPEC_EINVAL;
  if (d_model <= 0 || d_model % 8 != 0 || ldw < d_model || ldw % 8 != 0 || ldp < d_model || ldp % 8 != 0)
    return NANOSPEC_EINVAL;
  if (!aligned16(d_w_head) || !aligned16(d_packed)) return NANOSPEC_EINVAL;
  return cuda_status(launch_repack(st->sv, seq, (const uint16_t*)d_w_head, ldw, d_model, (uint16_t*)d_packed, ldp,
                                   d_tags, stream));
}

nanospec_status nanospec_draft_logits_topk_packed(const nanospec_state st, const void* d_packed, int32_t d_model,
                                                  int64_t ldp, const void* d_hidden, int32_t n_nodes, int32_t k,
                                                  float* d_topk_logit, int32_t* d_topk_id, float* d_lse,
                                                  void* d_scratch, size_t scratch_bytes, cudaStream_t stream) {
  if (!st || !d_packed || !d_hidden || !d_topk_logit || !d_topk_id) return NANOSPEC_EINVAL;
  if (d_model <= 0 || d_model % 8 != 0 || ldp < d_model || ldp % 8 != 0) return NANOSPEC_EINVAL;
  if (n_nodes < 1 || n_nodes > NANOSPEC_MAX_NODES || k < 1 || k > NANOSPEC_MAX_K) return NANOSPEC_EINVAL;
  if (!aligned16(d_packed) || !aligned16(d_hidden)) return NANOSPEC_EINVAL;
  const StateView& sv = st->sv;
  HeadProblem hp = {};
  hp.w = (const uint16_t*)d_packed;  // not dereferenced: rows come from `packed`
  hp.ldw = ldp;
  hp.d = d_model;
  hp.h = (const uint16_t*)d_hidden;
  hp.n = n_nodes;
  hp.batch = sv.batch;
  hp.ids_base = sv.ids;
  hp.ids_stride = sv.w_max;
  hp.nact_base = &sv.meta[0].n_active;
  hp.nact_stride = sizeof(Meta) / sizeof(int32_t);
  hp.max_ids = sv.w_max;
  hp.n_shards = sv.n_shards;
  hp.trace = trace_buffer();
  hp.packed = (const uint16_t*)d_packed;
  hp.ldp = ldp;
  return run_head(hp, k, d_topk_logit, d_topk_id, d_lse, nullptr, d_scratch, scratch_bytes, NANOSPEC_HEAD_TC, stream);
}

nanospec_status nanospec_tree_expand(const float* d_front_score, const int32_t* d_front_index, int32_t n_front,
                                     const float* d_topk_logit, const int32_t* d_topk_id, const float* d_lse,
                                     int32_t k, float* d_pool_score, int32_t* d_pool_id, int32_t* d_pool_parent,
                                     int32_t pool_offset, int32_t pool_cap, int32_t n_next, int32_t* d_next_index,
                                     float* d_next_score, cudaStream_t stream) {
  if (!d_topk_logit || !d_topk_id || !d_lse || !d_pool_score || !d_pool_id || !d_pool_parent) return NANOSPEC_EINVAL;
  if ((d_front_score == nullptr) != (d_front_index == nullptr)) return NANOSPEC_EINVAL;
  if (n_front < 1 || k < 1 || k > NANOSPEC_MAX_K || n_front * k > 1024 || pool_offset < 0) return NANOSPEC_EINVAL;
  if ((long long)pool_offset + (long long)n_front * k > pool_cap || pool_cap > 4096) return NANOSPEC_EINVAL;
  if (n_next < 0 || n_next > n_front * k || (n_next > 0 && (!d_next_index || !d_next_score))) return NANOSPEC_EINVAL;
  TreeLevel t;
  t.front_score = d_front_score;
  t.front_index = d_front_index;
  t.topk_logit = d_topk_logit;
  t.topk_id = d_topk_id;
  t.lse = d_lse;
  t.n_front = n_front;
  t.k = k;
  t.pool_score = d_pool_score;
  t.pool_id = d_pool_id;
  t.pool_parent = d_pool_parent;
  t.pool_offset = pool_offset;
  t.n_next = n_next;
  t.next_index = d_next_index;
  t.next_score = d_next_score;
  return cuda_status(launch_tree_expand(t, stream));
}

nanospec_status nanospec_tree_rerank(const float* d_pool_score, const int32_t* d_pool_id, int32_t pool_n, int32_t m,
                                     int32_t* d_out_index, int32_t* d_out_id, cudaStream_t stream) {
  if (!d_pool_score || !d_pool_id || !d_out_index || !d_out_id) return NANOSPEC_EINVAL;
  if (pool_n < 1 || pool_n > 4096 || m < 1 || m > pool_n) return NANOSPEC_EINVAL;
  return cuda_status(launch_tree_rerank(d_pool_score, d_pool_id, pool_n, m, d_out_index, d_out_id, stream));
}

}  // extern "C"
