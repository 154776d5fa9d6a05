// Stage 1 of the h-indexer (hindexer.py:94-178, quant.py:49-90): bit-exact rowwise int8
// quantisation, corpus scans in the float / int8 / raw-int32 views, the sampled threshold and
// order-preserving compaction of the passers.
#include <algorithm>
#include <cmath>

#include "kernels.cuh"
#include "stage1.cuh"

namespace molr {

// ------------------------------------------------------------------------------------------
// quantize_rowwise — quant.py:49-57 (bit-exact: IEEE division, rint half-even, clip +-127)
// ------------------------------------------------------------------------------------------
__global__ void quantize_rows_kernel(int64_t rows, int dim, const float* __restrict__ x, int8_t* __restrict__ codes,
                                     float* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw) {
    const float* xr = x + r * dim;
    float m = 0.f;
    for (int k = lane; k < dim; k += 32) m = fmaxf(m, fabsf(xr[k]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float sc = m > 0.0f ? __fdiv_rn(m, 127.0f) : 1.0f;
    for (int k = lane; k < dim; k += 32) {
      float q = rintf(__fdiv_rn(xr[k], sc));
      q = fminf(fmaxf(q, -127.0f), 127.0f);
      codes[r * dim + k] = (int8_t)(int)q;
    }
    if (lane == 0) scales[r] = sc;
  }
}

int quantize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, int8_t* codes, float* scales,
                  cudaStream_t s) {
  if (rows <= 0) return MOLR_OK;
  int blocks = (int)imin64((rows + 7) / 8, int64_t(ctx->num_sms) * 16);
  quantize_rows_kernel<<<blocks, 256, 0, s>>>(rows, dim, x, codes, scales);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

// ------------------------------------------------------------------------------------------
// scans: out[b*ld + r] for B queries against rows [0, n) of a stage-1 view
// ------------------------------------------------------------------------------------------
// int8 dot of stage-1 row r (cache layout, see s1_chunk_offset) with a linear query
__device__ __forceinline__ int32_t dot_row_i8(const int8_t* __restrict__ codes, int64_t r, const int8_t* __restrict__ q,
                                              int dim, bool ilv) {
  int32_t acc = 0;
  if ((dim & 15) == 0 && ((uintptr_t)q & 15) == 0 && (ilv || ((uintptr_t)codes & 15) == 0)) {
    for (int c = 0; c < dim / 16; ++c) {
      const int4 x = *reinterpret_cast<const int4*>(codes + (ilv ? s1_chunk_offset(r, c, dim) : r * dim + c * 16));
      const int4 y = *reinterpret_cast<const int4*>(q + c * 16);
      acc = __dp4a(x.x, y.x, acc);
      acc = __dp4a(x.y, y.y, acc);
      acc = __dp4a(x.z, y.z, acc);
      acc = __dp4a(x.w, y.w, acc);
    }
  } else {
    const int8_t* a = codes + r * dim;
    for (int k = 0; k < dim; ++k) acc += int32_t(a[k]) * int32_t(q[k]);
  }
  return acc;
}

// mode: MOLR_S1_FLOAT (f32 out), MOLR_S1_INT8 (f32 out = acc.f32 * scale), MOLR_S1_INT8_RAW (i32 out)
__global__ void scan_scores_kernel(int mode, int64_t n, int dim, const float* __restrict__ vf,
                                   const int8_t* __restrict__ codes, bool ilv, const int32_t* __restrict__ inv,
                                   const float* __restrict__ scales,
                                   const int64_t* __restrict__ rows_idx, int B, const float* __restrict__ qf,
                                   const int8_t* __restrict__ qc, void* __restrict__ out, int64_t ld) {
  extern __shared__ __align__(16) unsigned char sq[];
  // stage the B queries (codes or floats) in shared memory
  const int qbytes = mode == MOLR_S1_FLOAT ? B * dim * 4 : B * dim;
  const unsigned char* src = mode == MOLR_S1_FLOAT ? (const unsigned char*)qf : (const unsigned char*)qc;
  for (int i = threadIdx.x; i < qbytes; i += blockDim.x) sq[i] = src[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows_idx ? rows_idx[i] : i;
    if (mode == MOLR_S1_FLOAT && dim == 64) {
      // the row stays in registers across the queries (s1_dot64: NumPy/OpenBLAS order)
      float v[64];
      const float4* v4 = reinterpret_cast<const float4*>(vf + r * 64);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float4 x = __ldg(v4 + k);
        v[4 * k] = x.x, v[4 * k + 1] = x.y, v[4 * k + 2] = x.z, v[4 * k + 3] = x.w;
      }
      for (int b = 0; b < B; ++b)
        reinterpret_cast<float*>(out)[b * ld + i] = s1_dot64(v, reinterpret_cast<const float*>(sq) + b * 64);
    } else if (mode == MOLR_S1_FLOAT) {
      const float* v = vf + r * dim;
      for (int b = 0; b < B; ++b) {
        const float* q = reinterpret_cast<const float*>(sq) + b * dim;
        reinterpret_cast<float*>(out)[b * ld + i] = s1_dot_f32(v, q, dim);
      }
    } else {
      const int64_t pos = inv ? inv[r] : r;  // stored position of item r (sealed, scale-sorted tiles)
      const float scale = mode == MOLR_S1_INT8 ? scales[pos] : 0.f;
      for (int b = 0; b < B; ++b) {
        int32_t acc = dot_row_i8(codes, pos, reinterpret_cast<const int8_t*>(sq) + b * dim, dim, ilv);
        if (mode == MOLR_S1_INT8_RAW) reinterpret_cast<int32_t*>(out)[b * ld + i] = acc;
        else reinterpret_cast<float*>(out)[b * ld + i] = __fmul_rn((float)acc, scale);
      }
    }
  }
}

int scan_scores(molr_ctx* ctx, int mode, int64_t n, int dim, const float* vf, const int8_t* codes, bool ilv,
                const int32_t* inv, const float* scales, const int64_t* rows_idx, int B, const float* qf, const int8_t* qc, void* out,
                int64_t ld, cudaStream_t s) {
  if (n <= 0 || B <= 0) return MOLR_OK;
  // shared memory holds up to 48 KB of queries per launch; chunk the batch otherwise
  const int per_q = mode == MOLR_S1_FLOAT ? dim * 4 : dim;
  const int bchunk = std::max(1, std::min(B, (48 * 1024) / per_q));
  if (per_q > 48 * 1024) MOLR_FAIL(MOLR_ERR_DIMENSION, "stage-1 dim %d too large", dim);
  for (int b0 = 0; b0 < B; b0 += bchunk) {
    int bb = std::min(bchunk, B - b0);
    int blocks = (int)imin64((n + 255) / 256, int64_t(ctx->num_sms) * 8);
    size_t esz = mode == MOLR_S1_INT8_RAW ? 4 : 4;
    void* o = reinterpret_cast<char*>(out) + size_t(b0) * ld * esz;
    scan_scores_kernel<<<blocks, 256, size_t(bb) * per_q, s>>>(
        mode, n, dim, vf, codes, ilv, inv, scales, rows_idx, bb, qf ? qf + size_t(b0) * dim : nullptr,
        qc ? qc + size_t(b0) * dim : nullptr, o, ld);
    MOLR_LAUNCHED(ctx);
  }
  return MOLR_OK;
}

// ------------------------------------------------------------------------------------------
// order-preserving compaction of {r : key(score[b, r]) >= / > key(t_b)} (np.nonzero, ascending)
// ------------------------------------------------------------------------------------------
constexpr int kCompactChunk = 4096;
constexpr int kCompactThreads = 256;

__device__ __forceinline__ uint32_t score_key(const void* sc, int is_int, int64_t idx) {
  return is_int ? i32_key(reinterpret_cast<const int32_t*>(sc)[idx]) : f32_key(reinterpret_cast<const float*>(sc)[idx]);
}

__global__ void compact_count_kernel(int64_t n, const void* __restrict__ sc, int is_int, int64_t ld,
                                     const uint32_t* __restrict__ tkey, int strict, int64_t nchunks,
                                     int64_t* __restrict__ counts) {
  const int b = blockIdx.y;
  const int64_t c0 = blockIdx.x * (int64_t)kCompactChunk;
  const uint32_t t = tkey[b];
  int cnt = 0;
  for (int64_t i = c0 + threadIdx.x; i < min(n, c0 + kCompactChunk); i += blockDim.x) {
    uint32_t k = score_key(sc, is_int, b * ld + i);
    cnt += strict ? (k > t) : (k >= t);
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int wsum[kCompactThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) s += wsum[w];
    counts[b * nchunks + blockIdx.x] = s;
  }
}

// exclusive scan of chunk counts per query (one block per query); total -> totals[b]
__global__ void compact_scan_kernel(int64_t nchunks, int64_t* __restrict__ counts, int64_t* __restrict__ totals) {
  const int b = blockIdx.x;
  int64_t* c = counts + b * nchunks;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nchunks; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nchunks ? c[i] : 0;
    // block inclusive scan (Hillis-Steele in shared memory)
    __shared__ int64_t tmp[1024];
    tmp[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
      int64_t add = threadIdx.x >= (unsigned)o ? tmp[threadIdx.x - o] : 0;
      __syncthreads();
      tmp[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < nchunks) c[i] = carry + tmp[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += tmp[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[b] = carry;
}

__global__ void compact_write_kernel(int64_t n, const void* __restrict__ sc, int is_int, int64_t ld,
                                     const uint32_t* __restrict__ tkey, int strict, int64_t nchunks,
                                     const int64_t* __restrict__ offs, int64_t cap, int64_t id_base,
                                     int64_t* __restrict__ out_ids) {
  const int b = blockIdx.y;
  const int64_t c0 = blockIdx.x * (int64_t)kCompactChunk;
  const uint32_t t = tkey[b];
  __shared__ int wsum[kCompactThreads / 32];
  __shared__ int64_t run;
  if (threadIdx.x == 0) run = offs[b * nchunks + blockIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = c0; base < min(n, c0 + kCompactChunk); base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    bool pass = false;
    if (i < min(n, c0 + kCompactChunk)) {
      uint32_t k = score_key(sc, is_int, b * ld + i);
      pass = strict ? (k > t) : (k >= t);
    }
    unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) {
      before += w < warp ? wsum[w] : 0;
      total += wsum[w];
    }
    if (pass) {
      int64_t pos = run + before + __popc(bal & ((1u << lane) - 1));
      if (pos < cap) out_ids[b * cap + pos] = i + id_base;
    }
    __syncthreads();
    if (threadIdx.x == 0) run += total;
    __syncthreads();
  }
}

int compact_passers(molr_ctx* ctx, int B, int64_t n, const void* sc, int is_int, int64_t ld, const uint32_t* tkey,
                    int strict, int64_t cap, int64_t id_base, int64_t* out_ids, int64_t* totals, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  const int64_t nchunks = std::max<int64_t>(1, (n + kCompactChunk - 1) / kCompactChunk);
  Scratch counts;
  MOLR_TRY(counts.alloc(size_t(B) * nchunks * 8, s));
  dim3 grid((unsigned)nchunks, (unsigned)B);
  compact_count_kernel<<<grid, kCompactThreads, 0, s>>>(n, sc, is_int, ld, tkey, strict, nchunks,
                                                        counts.as<int64_t>());
  MOLR_LAUNCHED(ctx);
  compact_scan_kernel<<<B, 1024, 0, s>>>(nchunks, counts.as<int64_t>(), totals);
  MOLR_LAUNCHED(ctx);
  compact_write_kernel<<<grid, kCompactThreads, 0, s>>>(n, sc, is_int, ld, tkey, strict, nchunks,
                                                        counts.as<int64_t>(), cap, id_base, out_ids);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

__global__ void gather_rows_kernel(int64_t m, int64_t dim_bytes, const unsigned char* __restrict__ src,
                                   const int64_t* __restrict__ idx, unsigned char* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * dim_bytes;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / dim_bytes, c = i % dim_bytes;
    dst[i] = src[idx[r] * dim_bytes + c];
  }
}

int gather_rows(molr_ctx* ctx, int64_t m, int64_t dim_bytes, const void* src, const int64_t* idx, void* dst,
                cudaStream_t s) {
  if (m <= 0) return MOLR_OK;
  int blocks = (int)imin64((m * dim_bytes + 255) / 256, int64_t(ctx->num_sms) * 16);
  gather_rows_kernel<<<blocks, 256, 0, s>>>(m, dim_bytes, (const unsigned char*)src, idx, (unsigned char*)dst);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

__global__ void int_to_float_kernel(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    reinterpret_cast<float*>(p)[i] = (float)p[i];
}

int int_to_float_inplace(molr_ctx* ctx, int32_t* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return MOLR_OK;
  int_to_float_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(p, n);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

// queries for the int8 views: bit-exact quantize_vector (quant.py:60-63) of each row
int prepare_queries(molr_ctx* ctx, int mode, int B, int dim, const float* q, int8_t* qc, float* qs, cudaStream_t s) {
  if (mode == MOLR_S1_FLOAT) return MOLR_OK;
  return quantize_rows(ctx, B, dim, q, qc, qs, s);
}

int check_view(const molr_cache* c, int mode) {
  if (mode != MOLR_S1_FLOAT && c->s1_codes) MOLR_TRY(s1_seal(const_cast<molr_cache*>(c), c->ctx->stream));
  if (mode == MOLR_S1_FLOAT && !c->s1_f32) MOLR_FAIL(MOLR_ERR_INVALID, "cache has no float stage-1 view");
  if (mode != MOLR_S1_FLOAT && !c->s1_codes)
    MOLR_FAIL(MOLR_ERR_INVALID, "cache was built without quantized stage-1 embeddings");
  if (mode < 0 || mode > 2) MOLR_FAIL(MOLR_ERR_INVALID, "bad stage-1 mode %d", mode);
  return MOLR_OK;
}

}  // namespace molr

using namespace molr;

extern "C" {

int molr_quantize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, int8_t* codes, float* scales,
                       void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (rows < 0 || dim < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "expected 2-D matrix");
  if (dim > 131070) MOLR_FAIL(MOLR_ERR_LENGTH_OVERFLOW, "row length %d exceeds int32-safe bound 131070", dim);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (rows == 0) return MOLR_OK;
  In xi;
  Out c, sc;
  MOLR_TRY(xi.stage(x, size_t(rows) * dim * 4, s));
  MOLR_TRY(c.stage(codes, size_t(rows) * dim, s));
  MOLR_TRY(sc.stage(scales, size_t(rows) * 4, s));
  MOLR_TRY(quantize_rows(ctx, rows, dim, xi.as<float>(), c.as<int8_t>(), sc.as<float>(), s));
  return finish_outputs(s, {&c, &sc});
}

int molr_int8_matvec(molr_ctx* ctx, int64_t n, int dim, const int8_t* codes, const int8_t* q, int32_t* out,
                     void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (dim > 131070) MOLR_FAIL(MOLR_ERR_LENGTH_OVERFLOW, "row length %d exceeds int32-safe bound 131070", dim);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n <= 0) return MOLR_OK;
  In c, qq;
  Out o;
  MOLR_TRY(c.stage(codes, size_t(n) * dim, s));
  MOLR_TRY(qq.stage(q, size_t(dim), s));
  MOLR_TRY(o.stage(out, size_t(n) * 4, s));
  // raw mode over an ad-hoc view: scales unused
  MOLR_TRY(scan_scores(ctx, MOLR_S1_INT8_RAW, n, dim, nullptr, c.as<int8_t>(), false, nullptr, nullptr, nullptr, 1, nullptr,
                       qq.as<int8_t>(), o.dptr, n, s));
  return finish_outputs(s, {&o});
}


int molr_stage1_scores(molr_ctx* ctx, const molr_cache* c, int mode, int B, const float* q, void* out, void* stream) {
  if (!ctx || !c) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_TRY(check_view(c, mode));
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  In qi;
  Out o;
  MOLR_TRY(qi.stage(q, size_t(B) * c->d1 * 4, s));
  MOLR_TRY(o.stage(out, size_t(B) * c->X * 4, s));
  Scratch qc, qs;
  if (mode != MOLR_S1_FLOAT) {
    MOLR_TRY(qc.alloc(size_t(B) * c->d1, s));
    MOLR_TRY(qs.alloc(size_t(B) * 4, s));
    MOLR_TRY(prepare_queries(ctx, mode, B, c->d1, qi.as<float>(), qc.as<int8_t>(), qs.as<float>(), s));
  }
  MOLR_TRY(scan_scores(ctx, mode, c->X, c->d1, c->s1_f32, c->s1_codes, s1_interleaved(c->d1), c->s1_inv, c->s1_scales, nullptr, B, qi.as<float>(),
                       qc.as<int8_t>(), o.dptr, c->X, s));
  return finish_outputs(s, {&o});
}

int molr_h_indexer(molr_ctx* ctx, const molr_cache* c, int mode, int B, const float* q, int64_t lam,
                   const int64_t* sample, int64_t n_rank, int comparator, double* out_t, int64_t* out_counts,
                   int64_t* out_ids, int64_t cap, void* stream) {
  if (!ctx || !c) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_TRY(check_view(c, mode));
  if (lam < 1 || lam > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "lambda %lld outside [1, %lld]", (long long)lam,
                                       (long long)c->X);
  if (n_rank < 1 || n_rank > lam) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n=%lld outside [1, %lld]", (long long)n_rank,
                                            (long long)lam);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  const int is_int = mode == MOLR_S1_INT8_RAW;
  // 1. score the corpus once (hindexer.py:155)
  Scratch scores;
  MOLR_TRY(scores.alloc(size_t(B) * c->X * 4, s));
  In qi, si;
  MOLR_TRY(qi.stage(q, size_t(B) * c->d1 * 4, s));
  MOLR_TRY(si.stage(sample, size_t(B) * lam * 8, s));
  Scratch qc, qs;
  if (mode != MOLR_S1_FLOAT) {
    MOLR_TRY(qc.alloc(size_t(B) * c->d1, s));
    MOLR_TRY(qs.alloc(size_t(B) * 4, s));
    MOLR_TRY(prepare_queries(ctx, mode, B, c->d1, qi.as<float>(), qc.as<int8_t>(), qs.as<float>(), s));
  }
  MOLR_TRY(scan_scores(ctx, mode, c->X, c->d1, c->s1_f32, c->s1_codes, s1_interleaved(c->d1), c->s1_inv, c->s1_scales, nullptr, B, qi.as<float>(),
                       qc.as<int8_t>(), scores.p, c->X, s));
  // 2. threshold = n-th largest of the SAME score array at the sampled rows (hindexer.py:156-158)
  Scratch tkey;
  MOLR_TRY(tkey.alloc(size_t(B) * 4, s));
  MOLR_TRY(nth_largest_rows(ctx, B, lam, scores.p, is_int, c->X, si.as<int64_t>(), lam, n_rank,
                            tkey.as<uint32_t>(), s));
  // 3. passers in ascending id order (hindexer.py:159-163)
  Out ids, cnt;
  MOLR_TRY(ids.stage(out_ids, size_t(B) * cap * 8, s));
  MOLR_TRY(cnt.stage(out_counts, size_t(B) * 8, s));
  MOLR_TRY(compact_passers(ctx, B, c->X, scores.p, is_int, c->X, tkey.as<uint32_t>(), comparator == MOLR_STRICT,
                           cap, 0, ids.as<int64_t>(), cnt.as<int64_t>(), s));
  std::vector<uint32_t> hk(B);
  MOLR_CUDA(cudaMemcpyAsync(hk.data(), tkey.p, size_t(B) * 4, cudaMemcpyDeviceToHost, s));
  MOLR_TRY(finish_outputs(s, {&ids, &cnt}));
  MOLR_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) out_t[b] = is_int ? double(key_i32(hk[b])) : double(key_f32(hk[b]));
  // capacity check (reference never truncates: the caller retries with the reported counts)
  std::vector<int64_t> hc(B);
  MOLR_CUDA(cudaMemcpy(hc.data(), cnt.dptr, size_t(B) * 8, cudaMemcpyDefault));
  for (int b = 0; b < B; ++b)
    if (hc[b] > cap) MOLR_FAIL(MOLR_ERR_CAPACITY, "query %d has %lld passers > capacity %lld", b,
                               (long long)hc[b], (long long)cap);
  return MOLR_OK;
}

int molr_stage1_exact_top_k(molr_ctx* ctx, const molr_cache* c, int mode, int B, const float* q, int k,
                            int64_t* out_ids, void* stream) {
  if (!ctx || !c) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_TRY(check_view(c, mode));
  if (k < 1 || k > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "k=%d outside [1, %lld]", k, (long long)c->X);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  Scratch scores;
  MOLR_TRY(scores.alloc(size_t(B) * c->X * 4, s));
  MOLR_TRY(molr_stage1_scores(ctx, c, mode, B, q, scores.p, s));
  if (mode == MOLR_S1_INT8_RAW) {  // rank raw ints as floats: exact (|acc| < 2^24)
    MOLR_TRY(int_to_float_inplace(ctx, scores.as<int32_t>(), int64_t(B) * c->X, s));
  }
  Out ids;
  MOLR_TRY(ids.stage(out_ids, size_t(B) * k * 8, s));
  Scratch osc;
  MOLR_TRY(osc.alloc(size_t(B) * k * 4, s));
  Segs<int64_t> segs;
  segs.X = c->X;
  MOLR_TRY(segmented_top_k<int64_t>(ctx, B, segs, scores.as<float>(), c->X, k, 0, ids.as<int64_t>(),
                                    osc.as<float>(), s));
  return finish_outputs(s, {&ids});
}

}  // extern "C"
