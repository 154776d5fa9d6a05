// Internal (C++) entry points shared between translation units.
#pragma once
#include "common.cuh"

namespace molr {

// Segments of candidates per query: query b owns [begin[b], end[b]) of the id/score arrays.
// ids == nullptr means "dense": candidate j of query b is item j (segment [0, X)).
template <class Id>
struct Segs {
  const int64_t* begin = nullptr;  // (B,) device; nullptr => dense over X
  const int64_t* end = nullptr;    // (B,)
  const Id* ids = nullptr;
  int64_t X = 0;                   // dense length
};

// Fused MoL scoring over a cache (generic SIMT fp32 path, any shape within SMEM limits).
template <class Id>
int mol_score_generic(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u,
                      const float* user_embs, const float* uw, float tau, Segs<Id> segs,
                      float* out_scores, int64_t out_dense_ld, cudaStream_t s);

// True when the tcgen05 production kernel handles this shape (k_u=k_x=8, d=64, G=64, H=128).
bool mol_tc_supported(const molr_cache* c, const molr_gating* g, int k_u);
template <class Id>
int mol_score_tc(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B,
                 const float* user_embs, const float* uw, float tau, Segs<Id> segs, float* out_scores,
                 int64_t out_dense_ld, cudaStream_t s);

// Segmented top-k by (score desc, id asc).  Scores laid out like the segments
// (dense: scores[b*ld + j]).  id_offset is added to emitted ids.
template <class Id>
int segmented_top_k(molr_ctx* ctx, int B, Segs<Id> segs, const float* scores, int64_t dense_ld,
                    int k, int64_t id_offset, int64_t* out_ids, float* out_scores, cudaStream_t s);

// Radix-select n-th largest for B rows of keys given as f32 or int32 values, optionally through
// an index gather (values[b*ld + idx[b*lam + j]]).
int nth_largest_rows(molr_ctx* ctx, int B, int64_t n_values, const void* values, int is_int,
                     int64_t ld, const int64_t* gather, int64_t gather_ld, int64_t n,
                     uint32_t* out_keys, cudaStream_t s);

// n-th largest of rows of pre-computed ascending keys (row b: keys[b*cap, b*cap + counts[b])).
// Rows holding fewer than n keys set *short_rows (left untouched otherwise) and get no key.
int nth_largest_keys(molr_ctx* ctx, int B, int64_t cap, const uint32_t* keys, const int64_t* counts, int64_t n,
                     uint32_t* out_keys, int* short_rows, cudaStream_t s);

__global__ void mlp_forward_kernel(int rows, int in_dim, int hidden, int out_dim, const float* __restrict__ w1,
                                   const float* __restrict__ b1, const float* __restrict__ w2,
                                   const float* __restrict__ x, float* __restrict__ out);

int quantize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, int8_t* codes, float* scales,
                  cudaStream_t s);

}  // namespace molr
