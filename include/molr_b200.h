/*
 * molr_b200.h — C-ABI of the B200-native MoL + h-indexer retrieval hot path.
 *
 * The reference (arXiv 2306.04039 `molr`, /root/reference/pkg/src/molr) is pure Python/NumPy,
 * so its "plugin API" for this path is the Python module surface of molr.mol / molr.hindexer /
 * molr.quant.  Each entry point below replaces the NumPy body of one of those functions; the
 * Python mirror in paper_2306_04039_b200/{mol,hindexer,quant}.py keeps the reference names,
 * argument meaning and exception classes and calls through here (ctypes; GIL released).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every data pointer may be HOST or DEVICE memory (UVA):
 *    host inputs are staged to the device inside the call, host outputs are written back
 *    before the call returns; device pointers are used in place (no copies).
 *  - `stream` is a cudaStream_t passed as void* (NULL = the context's own stream).  Calls are
 *    re-entrant: scratch is stream-ordered (cudaMallocAsync), handles are immutable after
 *    creation, so any number of host threads may query one cache concurrently (engine.py:6).
 *  - Item ids are int64 on the boundary (reference dtype), < 2^31 inside.
 *  - Return value: MOLR_OK or one of the error codes; molr_last_error() gives a thread-local
 *    message.  Codes map 1:1 onto molr.errors classes (errors.py:4-24).
 */
#ifndef MOLR_B200_H
#define MOLR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

enum molr_status {
  MOLR_OK = 0,
  MOLR_ERR_DIMENSION = 1,      /* DimensionMismatchError  errors.py:12 */
  MOLR_ERR_OUT_OF_RANGE = 2,   /* OutOfRangeError         errors.py:16 */
  MOLR_ERR_EMPTY_CANDIDATES = 3,/* EmptyCandidatesError   errors.py:24 */
  MOLR_ERR_ZERO_NORM = 4,      /* ZeroNormError           errors.py:8  */
  MOLR_ERR_LENGTH_OVERFLOW = 5,/* LengthOverflowError     errors.py:20 */
  MOLR_ERR_CAPACITY = 6,       /* candidate buffer too small (new; caller retries larger) */
  MOLR_ERR_CUDA = 7,           /* CUDA / NCCL runtime failure */
  MOLR_ERR_INVALID = 8         /* bad argument (ValueError in the reference) */
};

/* stage-1 view / scoring mode — hindexer.py:94-112 */
enum molr_s1_mode {
  MOLR_S1_FLOAT = 0,     /* view @ q in fp32                                  (hindexer.py:112) */
  MOLR_S1_INT8 = 1,      /* int32 acc * row scale, bit-exact                  (hindexer.py:111) */
  MOLR_S1_INT8_RAW = 2   /* raw int32 accumulators (raw_int_ordering=True)    (hindexer.py:109-110) */
};

enum molr_comparator { MOLR_INCLUSIVE = 0, MOLR_STRICT = 1 }; /* hindexer.py:159-162 */

typedef struct molr_ctx molr_ctx;
typedef struct molr_cache molr_cache;
typedef struct molr_gating molr_gating;

const char* molr_last_error(void);
const char* molr_version(void);

/* ---- context: one device + a stream + the kernel registry -------------------------------- */
int molr_ctx_create(int device, molr_ctx** out);
int molr_ctx_destroy(molr_ctx* ctx);
int molr_ctx_sync(molr_ctx* ctx, void* stream);
/* number of hot-path kernel launches this context has issued (all threads) */
int64_t molr_ctx_launch_count(molr_ctx* ctx);
/* Per-kernel CUDA-event timing (off by default).  When on, the hot kernels are bracketed by
 * events on their own launch stream; read back (name, launches, total ms, algorithmic work in
 * bytes or flops) per kernel name by index until MOLR_ERR_OUT_OF_RANGE. */
int molr_ctx_set_profiling(molr_ctx* ctx, int on);
int molr_ctx_prof_read(molr_ctx* ctx, int idx, char* name, int name_len, int64_t* count,
                       double* total_ms, double* work);
int molr_ctx_prof_reset(molr_ctx* ctx);

/* ---- ItemCache: immutable device snapshot — mol.py:216-291 ---------------------------------
 * item_embs (X, k_x, d) f32, item_gate_pre (X, G) f32, stage1_embs (X, d1) f32 or NULL,
 * stage1 int8 codes (X, d1) + scales (X,) or NULL.  Storage on device: item_embs and gate_pre
 * as bf16 when every value is bf16-representable, else f32 — the device copy is always exact,
 * so scoring sees the caller's fp32 inputs bit for bit.  Replaces ItemCache.__init__ validation and
 * the arrays' residency. */
int molr_cache_create(molr_ctx* ctx, int64_t n_items, int k_x, int d, int n_logits,
                      const float* item_embs, const float* item_gate_pre,
                      int d1, const float* stage1_embs, const int8_t* stage1_codes,
                      const float* stage1_scales, molr_cache** out);
/* Two-step construction for corpora built on the device in chunks (no f32 copy of the whole
 * corpus ever exists): allocate with explicit storage, then fill row ranges.  storage bits:
 * MOLR_STORE_EMBS_F32 keeps item_embs in f32 (default bf16); MOLR_STORE_GP_F32 keeps gate_pre
 * in f32 (default bf16); MOLR_STORE_S1_F32 / MOLR_STORE_S1_INT8 select the stage-1 views.  A fill whose values
 * are not representable in the chosen storage fails with MOLR_ERR_INVALID (no silent loss). */
enum molr_storage {
  MOLR_STORE_EMBS_F32 = 1,
  MOLR_STORE_GP_F32 = 2,
  MOLR_STORE_S1_F32 = 4,
  MOLR_STORE_S1_INT8 = 8
};
int molr_cache_alloc(molr_ctx* ctx, int64_t n_items, int k_x, int d, int n_logits, int d1,
                     int storage, molr_cache** out);
int molr_cache_fill(molr_cache* cache, int64_t row0, int64_t n, const float* item_embs,
                    const float* item_gate_pre, const float* stage1_embs,
                    const int8_t* stage1_codes, const float* stage1_scales, void* stream);
int molr_cache_destroy(molr_cache* cache);
/* Device-side build_item_cache (mol.py:294-326) for rows [row0, row0+n): item_table (n, d_x) ->
 * item_proj MLP (d_x -> proj_hidden -> k_x*d) -> per-component L2 normalisation (numerics.py:41-50,
 * ZERO_NORM if a norm <= eps) -> item_net MLP (d_x -> net_hidden -> G) -> stage-1 = mean over the
 * k_x components -> rowwise int8 (quant.py:49-57) when the cache has an int8 view -> cache rows.
 * flags: MOLR_BUILD_L2_NORMALIZE (MoLConfig.l2_normalized), MOLR_BUILD_ROUND_BF16 (round the item
 * components and gate pre-activations to bf16 before the stage-1 mean: the production bf16 cache).
 * Weights and table may be host or device pointers.  Replaces mol.py:294-326 for device corpora. */
enum { MOLR_BUILD_L2_NORMALIZE = 1, MOLR_BUILD_ROUND_BF16 = 2 };
int molr_cache_build_rows(molr_cache* cache, int64_t row0, int64_t n, int d_x, const float* item_table,
                          int proj_hidden, const float* proj_w1, const float* proj_b1, const float* proj_w2,
                          int net_hidden, const float* net_w1, const float* net_b1, const float* net_w2,
                          int flags, float eps, void* stream);
/* read rows back as f32 (exact: storage is lossless); any output pointer may be NULL */
int molr_cache_read(const molr_cache* cache, int64_t row0, int64_t n, float* item_embs,
                    float* item_gate_pre, float* stage1_embs, int8_t* stage1_codes,
                    float* stage1_scales, void* stream);
/* storage: the molr_storage bits the cache was built with */
int molr_cache_info(const molr_cache* cache, int64_t* n_items, int* storage, int64_t* device_bytes);
/* 1 if MoL scoring of this (cache, gating, k_u) runs on the fused tcgen05 kernel (production shape
 * k_u = k_x = 8, d = 64, G = 64, H = 128; bf16-exact caches, or f32-stored caches through their
 * bf16 hi + lo image), 0 if on the generic SIMT fp32 kernel; < 0 on a null argument. */
int molr_mol_uses_tensor_cores(const molr_cache* cache, const molr_gating* gating, int k_u);

/* Elementwise primitives (numerics.py:69-81): op 0 sigmoid (scipy expit), 1 silu, 2 silu_grad;
 * dtype 0 = f32, 2 = f64 (the input's NumPy dtype). */
int molr_eltwise(molr_ctx* ctx, int op, int dtype, int64_t n, const void* x, void* out, void* stream);
/* Max-shifted softmax along the last axis (numerics.py:61-66). */
int molr_softmax_rows(molr_ctx* ctx, int dtype, int64_t rows, int dim, const void* x, void* out, void* stream);

/* Batched user-side query prep (engine.py:113-115 -> model.py:179-208 user_forward, and
 * mol.py:186 user_net): user_embs (B, k_u, d) = per-component L2-normalised user_proj(feats)
 * (when l2_normalized; ZERO_NORM if a norm <= eps), uw (B, G) = user_net(feats).  Both MLPs are
 * silu(x W1 + b1) W2 (mol.py:62-85).  Inputs/outputs host or device. */
int molr_query_prep(molr_ctx* ctx, int B, int d_u, const float* feats, int proj_hidden, const float* proj_w1,
                    const float* proj_b1, const float* proj_w2, int k_u, int d, int l2_normalized, int net_hidden,
                    const float* net_w1, const float* net_b1, const float* net_w2, int G, float eps,
                    float* user_embs, float* uw, void* stream);

/* ---- gating weights (cross_net G->H->G, user_net du->Hu->G) — mol.py:62-109 ---------------- */
int molr_gating_create(molr_ctx* ctx, int G, int H, const float* cross_w1, const float* cross_b1,
                       const float* cross_w2, int d_u, int H_u, const float* user_w1,
                       const float* user_b1, const float* user_w2, molr_gating** out);
int molr_gating_destroy(molr_gating* g);

/* ---- MoL primitives (generic shapes) ------------------------------------------------------ */
/* component_logits — mol.py:139-158: user (k_u,d), items (n,k_x,d) -> (n, k_u*k_x) / tau.
 * Arrays are f32, or f64 when is_f64 (computed in the input precision, like NumPy). */
int molr_component_logits(molr_ctx* ctx, int n, int k_u, int k_x, int d, const void* user_embs,
                          const void* item_embs, double tau, int is_f64, void* out, void* stream);
/* user_net / any Mlp forward: silu(x@w1+b1)@w2 — mol.py:84-85 (rows, in) -> (rows, out) */
int molr_mlp_forward(molr_ctx* ctx, int rows, int in_dim, int hidden, int out_dim,
                     const float* w1, const float* b1, const float* w2, const float* x, float* out,
                     void* stream);
/* decomposed_gating (inference) — mol.py:161-194: uw (G,), item_gate_pre (n,G), cl (n,G) -> pi */
int molr_decomposed_gating(molr_ctx* ctx, const molr_gating* g, int n, const float* uw,
                           const float* item_gate_pre, const float* cross_logits, float* out,
                           void* stream);
/* mol_score — mol.py:197-205 (f32, or f64 when is_f64) */
int molr_mol_score(molr_ctx* ctx, int n, int G, const void* pi, const void* cl, int is_f64, void* out,
                   void* stream);

/* ---- fused MoL scoring over a cache (K1) --------------------------------------------------
 * score_candidates / mol_top_k batched over B queries — mol.py:329-345, 389-408.
 * user_embs (B,k_u,d) f32; uw (B,G) f32 = user_net(gate_features) (mol.py:186).
 * Candidates in CSR: cand_offsets (B+1) int64, cand_ids int64; cand_offsets==NULL means
 * "every item of the cache" for every query (engine.full_top_k / batch_score_all).
 * score: out_scores laid out like cand_ids (or (B,X) when dense).
 * top_k: out_ids (B,k) int64, out_scores (B,k) f32, score desc, ties -> smaller id. */
int molr_score(molr_ctx* ctx, const molr_cache* cache, const molr_gating* g, int B, int k_u,
               const float* user_embs, const float* uw, float tau, const int64_t* cand_offsets,
               const int64_t* cand_ids, float* out_scores, void* stream);
int molr_mol_top_k(molr_ctx* ctx, const molr_cache* cache, const molr_gating* g, int B, int k_u,
                   const float* user_embs, const float* uw, float tau, const int64_t* cand_offsets,
                   const int64_t* cand_ids, int k, int64_t* out_ids, float* out_scores,
                   void* stream);

/* l2_normalize_rows — numerics.py:41-50 (MOLR_ERR_ZERO_NORM if any norm <= eps) */
int molr_l2_normalize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, float eps,
                           float* out, void* stream);
/* mean over the middle axis of (n, k, d) -> (n, d) — build_item_cache stage-1 (mol.py:318) */
int molr_mean_rows(molr_ctx* ctx, int64_t n, int k, int d, const float* x, float* out,
                   void* stream);

/* ---- quantization — quant.py:49-63, 83-90 ------------------------------------------------- */
int molr_quantize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, int8_t* codes,
                       float* scales, void* stream);
/* QuantizedRows.dequantize — quant.py:45-46 */
int molr_dequantize_rows(molr_ctx* ctx, int64_t rows, int dim, const int8_t* codes,
                         const float* scales, float* out, void* stream);
/* int8_matvec over arbitrary rows (codes (n,d) x query codes (d,)) -> int32 (n,) */
int molr_int8_matvec(molr_ctx* ctx, int64_t n, int dim, const int8_t* codes, const int8_t* q,
                     int32_t* out, void* stream);

/* ---- stage 1 over a cache (K2/K3) — hindexer.py:94-178 ------------------------------------ */
/* stage1_scores: B queries (B,d1) f32 -> (B,X) f32 (mode FLOAT/INT8) or int32 (INT8_RAW) */
int molr_stage1_scores(molr_ctx* ctx, const molr_cache* cache, int mode, int B, const float* q,
                       void* out, void* stream);
/* nth_largest (hindexer.py:77-82) of B rows of `n_values` values; dtype 0 f32, 1 i32, 2 f64, 3 i64 */
int molr_nth_largest(molr_ctx* ctx, int B, int64_t n_values, const void* values, int dtype,
                     int64_t n, double* out, void* stream);
/* estimate_threshold (hindexer.py:115-132): n-th largest score over the sampled rows */
int molr_estimate_threshold(molr_ctx* ctx, const molr_cache* cache, int mode, int B,
                            const float* q, int64_t lam, const int64_t* sample, int64_t n_rank,
                            double* out_t, void* stream);
/* h_indexer (hindexer.py:135-163) with host-drawn samples: sample (B,lam) int64 row ids of the
 * seeded permutation prefix; n_rank = max(1, round(k'*lam/X)).  Writes threshold per query,
 * passer counts and ascending ids (CSR into out_ids with capacity `cap` per query; count>cap
 * returns MOLR_ERR_CAPACITY with out_counts filled so the caller can retry). */
int molr_h_indexer(molr_ctx* ctx, const molr_cache* cache, int mode, int B, const float* q,
                   int64_t lam, const int64_t* sample, int64_t n_rank, int comparator,
                   double* out_t, int64_t* out_counts, int64_t* out_ids, int64_t cap,
                   void* stream);
/* exact_top_k (hindexer.py:166-178): (B,k) ids, ties -> smaller id */
int molr_stage1_exact_top_k(molr_ctx* ctx, const molr_cache* cache, int mode, int B,
                            const float* q, int k, int64_t* out_ids, void* stream);
/* index_select (hindexer.py:181-201) — new cache of the given ascending rows (device gather) */
int molr_index_select(molr_ctx* ctx, const molr_cache* cache, int64_t n, const int64_t* ids,
                      molr_cache** out);

/* ---- fused batched two-stage retrieval (engine.py:117-138 batched) ------------------------
 * Per query: stage-1 query = mean_a user_embs[a] (engine.py:131); threshold from a device-drawn
 * sample of lam rows shared by the batch (seeded Feistel permutation prefix); passers scored
 * by MoL; top-k.  A shard of a larger corpus passes id_offset (global id of row 0) so the
 * returned ids are global.  out_ids (B,k), out_scores (B,k); out_cand (B,) candidate counts. */
int molr_two_stage_top_k(molr_ctx* ctx, const molr_cache* cache, const molr_gating* g, int B,
                         int k_u, const float* user_embs, const float* uw, float tau, int mode,
                         int64_t k_prime, int64_t lam, uint64_t seed, int comparator, int k,
                         int64_t id_offset, int64_t* out_ids, float* out_scores,
                         int64_t* out_cand, void* stream);

/* ---- sharded retrieval with the single-device threshold (SURVEY §8(e) "single-GPU-equivalent
 * threshold") --------------------------------------------------------------------------------
 * A shard holding global rows [row_lo, row_lo + X_shard) of an X_global corpus:
 * 1. molr_sample_top_keys: draws the SAME global sample as a single device (seeded Feistel prefix
 *    of lam rows of X_global, hindexer.py:125), scores the rows that fall in this shard and writes
 *    each query's n_keep largest ascending-order score keys (f32_key / i32_key; padded with 0).
 * 2. the caller all-gathers the (B, n_keep) keys of the P shards into (B, P*n_keep) rows and
 *    molr_select_nth_keys picks the n-th largest per row: n = max(1, round(k'*lam/X_global)) gives
 *    exactly the single-device threshold (hindexer.py:131; the n-th largest of the union of every
 *    shard's top n is the n-th largest of the whole sample).
 * 3. molr_two_stage_top_k_at filters this shard with those thresholds (keys), scores the passers
 *    by MoL and returns the shard's top-k with global ids and its passer counts; no corpus
 *    fallback (the caller falls back when the GLOBAL count is < k, engine.py:134-135, by calling
 *    it again with the key below every score: f32_key(-inf) = 0x007FFFFF, or 0 for raw int32).  cap_hint sizes the candidate buffer. */
int molr_sample_top_keys(molr_ctx* ctx, const molr_cache* cache, int B, int k_u, const float* user_embs,
                         int mode, int64_t X_global, int64_t row_lo, int64_t lam, uint64_t seed,
                         int64_t n_keep, uint32_t* out_keys, void* stream);
int molr_select_nth_keys(molr_ctx* ctx, int B, int64_t m, const uint32_t* keys, int64_t n,
                         uint32_t* out_keys, void* stream);
int molr_two_stage_top_k_at(molr_ctx* ctx, const molr_cache* cache, const molr_gating* g, int B,
                            int k_u, const float* user_embs, const float* uw, float tau, int mode,
                            int64_t cap_hint, const uint32_t* tkeys, int comparator, int k,
                            int64_t id_offset, int64_t* out_ids, float* out_scores,
                            int64_t* out_cand, void* stream);

/* ---- multi-GPU merge (C1): P ranks' (B,k) lists (already all-gathered, rank-major) ------- */
int molr_merge_top_k(molr_ctx* ctx, int P, int B, int k_in, const int64_t* ids,
                     const float* scores, int k, int64_t* out_ids, float* out_scores,
                     void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* MOLR_B200_H */
