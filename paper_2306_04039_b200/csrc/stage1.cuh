// Stage-1 building blocks shared by stage1.cu and pipeline.cu.
#pragma once
#include "kernels.cuh"

namespace molr {

int scan_scores(molr_ctx* ctx, int mode, int64_t n, int dim, const float* vf, const int8_t* codes, bool ilv,
                const int32_t* inv, const float* scales, const int64_t* rows_idx, int B, const float* qf, const int8_t* qc, void* out,
                int64_t ld, cudaStream_t s);
int compact_passers(molr_ctx* ctx, int B, int64_t n, const void* sc, int is_int, int64_t ld, const uint32_t* tkey,
                    int strict, int64_t cap, int64_t id_base, int64_t* out_ids, int64_t* totals, cudaStream_t s);
int gather_rows(molr_ctx* ctx, int64_t m, int64_t dim_bytes, const void* src, const int64_t* idx, void* dst,
                cudaStream_t s);
int prepare_queries(molr_ctx* ctx, int mode, int B, int dim, const float* q, int8_t* qc, float* qs, cudaStream_t s);
int check_view(const molr_cache* c, int mode);
// Deferred overflow check for the filter scans of one batched call: instead of reading back the
// largest per-CTA passer segment after each scan (a host round trip), the scan records it in
// *seg_need (device, atomicMax) and reports the segment length it used in *seg_used (host); the
// caller compares the two after its single end-of-call synchronisation and reruns with
// seg_min = *seg_need if a segment overflowed (rare: passers of one query concentrated in one
// CTA's block of the corpus).
struct S1Deferred {
  int* seg_need = nullptr;   // device
  int64_t seg_min = 0;       // floor for the segment length
  int64_t* seg_used = nullptr;  // host: max segment length used by the scans that reported here
};
bool s1_tc_supported(const molr_cache* c, int mode);
int s1_tc_scan(molr_ctx* ctx, int mode, const int8_t* codes, const float* scales, const float2* mm,
               const int32_t* perm, int64_t n, int B,
               const int8_t* qcodes, const uint32_t* tkeys, int strict, int64_t cap, int32_t* cand, int64_t* counts,
               void* out, int64_t ld, cudaStream_t s, bool emit_keys = false, const S1Deferred* defer = nullptr);
// chunk (min, max) scale reciprocals of 32-row chunks [c0, c1) of a scale vector (filter bound)
int encode_rows_tmap(CUtensorMap* tm, const void* base, int64_t rows);
int chunk_minmax(molr_ctx* ctx, const float* scales, int64_t c0, int64_t c1, float2* mm, cudaStream_t s);
int s1_update_chunk_mm(molr_cache* c, int64_t row0, int64_t n, cudaStream_t s);
int s1_seal(molr_cache* c, cudaStream_t s);
// rows [row0, row0 + n) of an f32-stored cache's bf16 hi + lo image, from its embs_f32 (abi.cu)
int build_embs_hilo(molr_cache* c, int64_t row0, int64_t n, cudaStream_t s);
// float view (MOLR_S1_FLOAT) on the tensor cores: bf16 MMA pre-test + exact fp32 re-check of the
// band the bf16 rounding cannot decide (same candidate set as the fp32 scan)
bool s1_bf_supported(const molr_cache* c, int mode);
struct F16View {  // fp16 image of an fp32 row matrix (d = 64) for s1_f16_filter
  const __half* h;
  const float* nrm;  // per-row ||v||_2 (rounded up)
  const float* cmx;  // per-32-row max of nrm
  float sv;          // power-of-two scale of the image
  const float* f32;  // the fp32 rows (exact re-check)
  int64_t n;
};
int s1_f16_filter(molr_ctx* ctx, const F16View& V, int B, const float* q, const uint32_t* tkeys, int strict,
                  int64_t cap, int32_t* cand, int64_t* counts, cudaStream_t s, const char* timer);
int s1_f16_image(molr_ctx* ctx, const molr_cache* c, const int64_t* rows, int64_t n, Scratch& f32, Scratch& h,
                 Scratch& nrm, Scratch& cmx, F16View* out, cudaStream_t s);
int s1_passer_keys(molr_ctx* ctx, int B, int64_t cap, const int32_t* ids, const int64_t* counts, const float* vf,
                   const float* q, uint32_t* keys, cudaStream_t s);
int s1_bf_scan(molr_ctx* ctx, const molr_cache* c, int B, const float* q, const uint32_t* tkeys, int strict,
               int64_t cap, int32_t* cand, int64_t* counts, cudaStream_t s);
int int_to_float_inplace(molr_ctx* ctx, int32_t* p, int64_t n, cudaStream_t s);

}  // namespace molr
