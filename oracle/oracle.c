/*
 * NanoSpec CPU oracle  --  TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load or call this library.  The product path
 * (paper_2605_26444_b200/) never touches it and shares no code, header, table
 * or helper with it.
 *
 * A plain, slow, obviously correct CPU implementation of what the hot path
 * computes, written from the paper (PAPER.md, arxiv 2605.26444).  All floating
 * point is fp64.  Every function cites the passage it follows ("P:n" is a
 * PAPER.md line, "S:n" a SPEC.md line).
 *
 *   Eq. 3  stream initialisation  S0 = prompt (+) tuple(U_i TopK_pre(z_i))
 *   Eq. 4  stream update          S  = S (+) tuple(C_draft) (+) tuple(C_ver)
 *   Eq. 5  active set             I  = Unique(Suffix(S, W_max))
 *   Eq. 2  LM head restricted to I: z_j = W_head[I_j,:] . h
 *   Alg. 1 line 528    SelectDraftTokens: top-k over the pruned logits, mapped
 *                      back to global ids through I
 *
 * Readings of the paper this file takes (DESIGN.md lists them all):
 *   Q1  rule R1 = Eq. 5 literally (window counts stream slots); rule R2 =
 *       unique-FIFO ("pushing unique new candidates"; "FIFO eviction",
 *       P:641) as a secondary flag.
 *   Q3  tuple(set) = first-occurrence order of the list it came from; the
 *       prefill union is flattened row-major (position, then rank).
 *   Q4  I is reported in ascending global id.
 *   Q10 ties in top-k are broken by ascending global id.
 *   Q13 lse is over the active set only.
 *   ids outside [0, V) are dropped (never appended) and flagged in *err.
 *
 * Parity pins (tests/test_oracle_*.py) are listed in DESIGN.md section 3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EEMPTY 2

/* bf16 -> double, exactly: a bf16 is the top 16 bits of an IEEE binary32. */
double oracle_bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* tuple(set): keep the first occurrence of every id of `in`, in order (Q3).
 * Ids outside [0, V) are dropped and set *err = 1.  Returns the output length. */
static int64_t dedup_first(const int32_t* in, int64_t m, int32_t V, int32_t* out, int32_t* err) {
  int64_t n = 0;
  for (int64_t i = 0; i < m; ++i) {
    int32_t e = in[i];
    if (e < 0 || e >= V) { *err = 1; continue; }
    int seen = 0;
    for (int64_t j = 0; j < n; ++j)
      if (out[j] == e) { seen = 1; break; }
    if (!seen) out[n++] = e;
  }
  return n;
}

/* Eq. 3: S0 = (x_1..x_L) (+) tuple(U_{i=1..L} T_Kpre(z_i)).
 * prefill is [L x k_pre], row i = the top-k_pre ids of z_i in rank order
 * (computing T_Kpre from target logits is outside the hot path).
 * Prompt tokens are kept verbatim, duplicates included.
 * `out` must hold L + L*k_pre ids.  Returns |S0|, or -ORACLE_EEMPTY for L == 0
 * ("empty prompt"). */
int64_t oracle_stream_init(const int32_t* prompt, int64_t L, const int32_t* prefill, int32_t k_pre,
                           int32_t V, int32_t* out, int32_t* err) {
  if (L <= 0) return -ORACLE_EEMPTY;
  int64_t n = 0;
  for (int64_t i = 0; i < L; ++i) {
    int32_t e = prompt[i];
    if (e < 0 || e >= V) { *err = 1; continue; }
    out[n++] = e;
  }
  if (k_pre > 0) n += dedup_first(prefill, L * (int64_t)k_pre, V, out + n, err);
  return n;
}

/* Eq. 4: the segment appended at a decode step,
 * tuple(C_draft) (+) tuple(C_ver); C_draft first (Q5). Each tuple is
 * deduplicated only within itself.  `out` must hold n_draft + k_ver ids. */
int64_t oracle_stream_update(const int32_t* draft, int32_t n_draft, const int32_t* verify, int32_t k_ver,
                             int32_t V, int32_t* out, int32_t* err) {
  int64_t n = dedup_first(draft, n_draft, V, out, err);
  n += dedup_first(verify, k_ver, V, out + n, err);
  return n;
}

/* Eq. 5: I = Unique(Suffix(S, W_max)) -- rule R1 (rule == 0).
 * Rule R2 (rule == 1), unique-FIFO: replay S from the start; an element
 * already in the queue Q is skipped, otherwise it is pushed at the back and,
 * if |Q| > W_max, the front is popped.
 * Vocab-parallel shard (n_shards > 1): only ids g with g % n_shards ==
 * shard_rank are reported; the bitmap is indexed by the local id g / n_shards.
 * ids_out gets I in ascending global id (Q4); bitmap_out (may be NULL) gets
 * ceil(V_local/32) words, bit b of word w set iff local id 32w+b is in I.
 * Returns |I| (of this shard). */
int32_t oracle_active_set(const int32_t* S, int64_t len, int32_t V, int32_t W, int32_t rule,
                          int32_t shard_rank, int32_t n_shards, int32_t* ids_out, uint32_t* bitmap_out) {
  unsigned char* in_set = (unsigned char*)calloc((size_t)V, 1);
  if (rule == 0) {
    int64_t start = len - W > 0 ? len - W : 0;              /* Suffix(S, W_max) */
    for (int64_t p = start; p < len; ++p) in_set[S[p]] = 1;  /* Unique(.) */
  } else {
    int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len + 1));
    int64_t head = 0, tail = 0;                              /* Q = q[head, tail) */
    for (int64_t p = 0; p < len; ++p) {
      int32_t e = S[p];
      if (in_set[e]) continue;
      q[tail++] = e;
      in_set[e] = 1;
      if (tail - head > W) in_set[q[head++]] = 0;
    }
    free(q);
  }
  int32_t n_local = n_shards > 1 ? (V - shard_rank + n_shards - 1) / n_shards : V;
  int32_t n_words = (n_local + 31) / 32;
  if (bitmap_out) memset(bitmap_out, 0, sizeof(uint32_t) * (size_t)n_words);
  int32_t n = 0;
  for (int32_t g = 0; g < V; ++g) {
    if (!in_set[g]) continue;
    if (n_shards > 1 && g % n_shards != shard_rank) continue;
    ids_out[n++] = g;
    int32_t l = n_shards > 1 ? g / n_shards : g;
    if (bitmap_out) bitmap_out[l / 32] |= 1u << (l % 32);
  }
  free(in_set);
  return n;
}

/* The W_max-slot ring a GPU-resident R1 state keeps: stream
 * position p lives in slot p % W for the last min(len, W) positions; never
 * written slots hold -1.  For R2 the ring holds the last W pushed elements in
 * push order (push i in slot i % W).  Returns the number of pushes (R2) or
 * len (R1): the state's `total`. */
int64_t oracle_ring(const int32_t* S, int64_t len, int32_t V, int32_t W, int32_t rule, int32_t* ring_out) {
  for (int32_t s = 0; s < W; ++s) ring_out[s] = -1;
  if (rule == 0) {
    int64_t start = len - W > 0 ? len - W : 0;
    for (int64_t p = start; p < len; ++p) ring_out[p % W] = S[p];
    return len;
  }
  unsigned char* in_q = (unsigned char*)calloc((size_t)V, 1);
  int64_t pushes = 0;
  for (int64_t p = 0; p < len; ++p) {
    int32_t e = S[p];
    if (in_q[e]) continue;
    if (pushes >= W) in_q[ring_out[pushes % W]] = 0;
    ring_out[pushes % W] = e;
    in_q[e] = 1;
    ++pushes;
  }
  free(in_q);
  return pushes;
}

/* Eq. 2 restricted to I:
 *   z[i][j] = sum_{c=0}^{d-1} W_head[ids[j]][c] * H[i][c]     (ascending c, fp64)
 *   A[i][j] = sum_{c} |W_head[ids[j]][c] * H[i][c]|            (conditioning, tolerance floor)
 * W is [V x ldw] bf16 bits row-major, H is [n x d] bf16 bits; z, A are [n x n_ids]. */
void oracle_logits(const uint16_t* W, int64_t ldw, int32_t d, const uint16_t* H, int32_t n,
                   const int32_t* ids, int32_t n_ids, double* z, double* A) {
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t j = 0; j < n_ids; ++j) {
      const uint16_t* w = W + (int64_t)ids[j] * ldw;
      const uint16_t* h = H + (int64_t)i * d;
      double s = 0.0, a = 0.0;
      for (int32_t c = 0; c < d; ++c) {
        double p = oracle_bf16_to_double(w[c]) * oracle_bf16_to_double(h[c]);
        s += p;
        a += fabs(p);
      }
      z[(int64_t)i * n_ids + j] = s;
      if (A) A[(int64_t)i * n_ids + j] = a;
    }
  }
}

/* SelectDraftTokens (Alg. 1) in its top-k form: for every
 * node i, the k entries of z[i][.] ranked by (value descending, global id
 * ascending) (Q10), mapped to global ids through ids[].  Slots beyond
 * n_ids are padded with (-inf, -1).  Plain repeated arg-max. */
void oracle_topk(const double* z, const int32_t* ids, int32_t n_ids, int32_t n, int32_t k,
                 double* val_out, int32_t* id_out) {
  unsigned char* taken = (unsigned char*)malloc((size_t)(n_ids > 0 ? n_ids : 1));
  for (int32_t i = 0; i < n; ++i) {
    memset(taken, 0, (size_t)(n_ids > 0 ? n_ids : 1));
    const double* zi = z + (int64_t)i * n_ids;
    for (int32_t r = 0; r < k; ++r) {
      int32_t best = -1;
      for (int32_t j = 0; j < n_ids; ++j) {
        if (taken[j]) continue;
        if (best < 0 || zi[j] > zi[best] || (zi[j] == zi[best] && ids[j] < ids[best])) best = j;
      }
      if (best < 0) {
        val_out[(int64_t)i * k + r] = -INFINITY;
        id_out[(int64_t)i * k + r] = -1;
      } else {
        taken[best] = 1;
        val_out[(int64_t)i * k + r] = zi[best];
        id_out[(int64_t)i * k + r] = ids[best];
      }
    }
  }
  free(taken);
}

/* log sum_j exp(z[i][j]) over the active set (softmax renormalised over the
 * pruned vocabulary, Q13): m = max_j z; lse = m + log sum_j exp(z - m). */
void oracle_lse(const double* z, int32_t n_ids, int32_t n, double* lse_out) {
  for (int32_t i = 0; i < n; ++i) {
    const double* zi = z + (int64_t)i * n_ids;
    if (n_ids <= 0) { lse_out[i] = -INFINITY; continue; }
    double m = zi[0];
    for (int32_t j = 1; j < n_ids; ++j) if (zi[j] > m) m = zi[j];
    double s = 0.0;
    for (int32_t j = 0; j < n_ids; ++j) s += exp(zi[j] - m);
    lse_out[i] = m + log(s);
  }
}

/* EAGLE-2 draft-tree bookkeeping (SelectDraftTokens / "append x_draft to draft
 * tree", Alg. 1; depth 5 and at most 60 draft tokens).
 * Level expansion: child (f, j) of frontier node f gets the cumulative
 * log-probability parent_score[f] + (val[f][j] - lse[f]) -- the log-softmax
 * over the active set; the root has parent_score == NULL (score 0,
 * parent -1).  Children are appended to the pool at pool_n in (f, j) order;
 * padding children (id < 0) score -inf.  The n_next best children of this
 * level, by (score desc, pool index asc), become the next frontier: repeated
 * arg-max, plain loops. */
void oracle_tree_expand(const double* parent_score, const int32_t* parent_index, int32_t n_front,
                        const double* val, const int32_t* id, const double* lse, int32_t k, double* pool_score,
                        int32_t* pool_id, int32_t* pool_parent, int32_t pool_n, int32_t n_next,
                        int32_t* next_index, double* next_score) {
  const int32_t nc = n_front * k;
  for (int32_t f = 0; f < n_front; ++f)
    for (int32_t j = 0; j < k; ++j) {
      const int32_t c = pool_n + f * k + j;
      const int32_t tok = id[(int64_t)f * k + j];
      const double ps = parent_score ? parent_score[f] : 0.0;
      pool_score[c] = tok >= 0 ? ps + (val[(int64_t)f * k + j] - lse[f]) : -INFINITY;
      pool_id[c] = tok;
      pool_parent[c] = parent_index ? parent_index[f] : -1;
    }
  char* taken = (char*)calloc((size_t)(nc > 0 ? nc : 1), 1);
  for (int32_t r = 0; r < n_next; ++r) {
    int32_t best = -1;
    for (int32_t c = 0; c < nc; ++c) {
      if (taken[c]) continue;
      if (best < 0 || pool_score[pool_n + c] > pool_score[pool_n + best]) best = c;  /* ties: lower index kept */
    }
    taken[best] = 1;
    next_index[r] = pool_n + best;
    next_score[r] = pool_score[pool_n + best];
  }
  free(taken);
}

/* Rerank: the m best nodes of the pool by (score desc, pool index asc): the
 * draft tree, whose tokens form C_draft.  Repeated arg-max. */
void oracle_tree_rerank(const double* pool_score, int32_t n, int32_t m, int32_t* out_index) {
  char* taken = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int32_t r = 0; r < m; ++r) {
    int32_t best = -1;
    for (int32_t c = 0; c < n; ++c) {
      if (taken[c]) continue;
      if (best < 0 || pool_score[c] > pool_score[best]) best = c;
    }
    taken[best] = 1;
    out_index[r] = best;
  }
  free(taken);
}
