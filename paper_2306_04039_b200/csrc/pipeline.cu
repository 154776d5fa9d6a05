// Cache-level MoL entry points (score_candidates / mol_top_k / batch_score_all, mol.py:329-408),
// index_select (hindexer.py:181-201) and the fused batched two-stage retrieval
// (RetrievalEngine.query batched, engine.py:117-138).
#include <algorithm>
#include <cmath>

#include "kernels.cuh"
#include "stage1.cuh"

namespace molr {

// Dispatch: tcgen05 production kernel for the production shape, generic SIMT otherwise.
template <class Id>
int mol_score_any(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
                  const float* uw, float tau, Segs<Id> segs, float* out, int64_t out_ld, cudaStream_t s) {
  if (mol_tc_supported(c, g, k_u)) return mol_score_tc<Id>(ctx, c, g, B, ue, uw, tau, segs, out, out_ld, s);
  return mol_score_generic<Id>(ctx, c, g, B, k_u, ue, uw, tau, segs, out, out_ld, s);
}

// begin[b] = off[b], end[b] = off[b+1]
__global__ void csr_to_segs_kernel(int B, const int64_t* __restrict__ off, int64_t* __restrict__ beg,
                                   int64_t* __restrict__ end) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    beg[b] = off[b];
    end[b] = off[b + 1];
  }
}

__global__ void validate_ids_kernel(int64_t n, const int64_t* __restrict__ ids, int64_t X, int* __restrict__ bad) {
  int b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b |= (ids[i] < 0 || ids[i] >= X);
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// mean over k_u component rows -> stage-1 query (engine.py:131; numpy axis-0 reduction is a
// sequential fp32 sum over rows followed by one division)
__global__ void s1_query_kernel(int B, int k_u, int d, const float* __restrict__ ue, float* __restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < int64_t(B) * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / d, k = i % d;
    float acc = ue[(b * k_u) * d + k];
    for (int a = 1; a < k_u; ++a) acc = __fadd_rn(acc, ue[(b * k_u + a) * d + k]);
    q[i] = __fdiv_rn(acc, (float)k_u);
  }
}

// ---- device sampling: seeded Feistel permutation of [0, X), prefix of length lam -------------
__device__ __forceinline__ uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__global__ void feistel_sample_kernel(int64_t X, int64_t lam, uint64_t seed, int half_bits, int64_t* __restrict__ out) {
  const uint32_t mask = (1u << half_bits) - 1u;
  const uint32_t k0 = mix32(uint32_t(seed) ^ 0x9e3779b9u), k1 = mix32(uint32_t(seed >> 32) ^ 0x7f4a7c15u);
  const uint32_t keys[4] = {k0, k1, mix32(k0 + 0x632be59bu), mix32(k1 + 0x3c6ef372u)};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < lam; j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)j;
    do {  // cycle-walk until inside [0, X)
      uint32_t L = uint32_t(x >> half_bits), R = uint32_t(x) & mask;
      for (int r = 0; r < 4; ++r) {
        uint32_t nL = R;
        R = L ^ (mix32(R * 0x9e3779b1u ^ keys[r]) & mask);
        L = nL;
      }
      x = (uint64_t(L) << half_bits) | R;
    } while (x >= (uint64_t)X);
    out[j] = (int64_t)x;
  }
}

// filter scan: every row against every query; append passers (int32 local ids) per query
template <int MODE>
__global__ void __launch_bounds__(256)
filter_scan_kernel(int64_t n, int dim, const float* __restrict__ vf, const int8_t* __restrict__ codes,
                   const int32_t* __restrict__ inv, const float* __restrict__ scales, int B, const float* __restrict__ qf,
                   const int8_t* __restrict__ qc, const uint32_t* __restrict__ tkey, int strict, int64_t cap,
                   int32_t* __restrict__ cand, int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char sq[];
  uint32_t* tk = reinterpret_cast<uint32_t*>(sq);
  unsigned char* qs = sq + ((B * 4 + 15) / 16) * 16;
  const int qbytes = MODE == MOLR_S1_FLOAT ? B * dim * 4 : B * dim;
  const unsigned char* src = MODE == MOLR_S1_FLOAT ? (const unsigned char*)qf : (const unsigned char*)qc;
  for (int i = threadIdx.x; i < qbytes; i += blockDim.x) qs[i] = src[i];
  for (int i = threadIdx.x; i < B; i += blockDim.x) tk[i] = tkey[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    for (int b = 0; b < B; ++b) {
      uint32_t key;
      if (MODE == MOLR_S1_FLOAT) {
        const float* v = vf + r * dim;
        const float* q = reinterpret_cast<const float*>(qs) + b * dim;
        key = f32_key(s1_dot_f32(v, q, dim));  // (the row is re-read from L1 per query)
      } else {
        int32_t acc = 0;
        const int64_t pos = inv ? inv[r] : r;
        const int4* qq = reinterpret_cast<const int4*>(qs + b * dim);
        for (int k = 0; k < dim / 16; ++k) {
          int4 x = *reinterpret_cast<const int4*>(codes + s1_chunk_offset(pos, k, dim)), y = qq[k];
          acc = __dp4a(x.x, y.x, acc);
          acc = __dp4a(x.y, y.y, acc);
          acc = __dp4a(x.z, y.z, acc);
          acc = __dp4a(x.w, y.w, acc);
        }
        key = MODE == MOLR_S1_INT8_RAW ? i32_key(acc) : f32_key(__fmul_rn((float)acc, scales[pos]));
      }
      bool pass = strict ? key > tk[b] : key >= tk[b];
      if (pass) {
        int64_t pos = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(counts + b), 1ull);
        if (pos < cap) cand[int64_t(b) * cap + pos] = (int32_t)r;
      }
    }
  }
}

// flag |= 1 if any query's passer count overflowed its capacity
__global__ void max_count_kernel(int B, const int64_t* __restrict__ counts, int64_t cap, int* __restrict__ flag) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (__syncthreads_or(b < B && counts[b] > cap) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void cap_segs_kernel(int B, int64_t cap, const int64_t* __restrict__ counts, int64_t* __restrict__ beg,
                                int64_t* __restrict__ end) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
    beg[b] = int64_t(b) * cap;
    end[b] = int64_t(b) * cap + min(counts[b], cap);
  }
}

// gather sampled stage-1 rows (codes interleaved + scales) into a contiguous operand padded to
// n_pad rows (the padding rows are zeroed here): one thread per row, its four 16-B chunks loaded
// together (the idx -> inv -> row chain is paid once per row, not once per chunk)
__global__ void gather_sample_kernel(const int8_t* __restrict__ codes, const float* __restrict__ scales,
                                     const int32_t* __restrict__ inv, const int64_t* __restrict__ idx, int64_t n,
                                     int64_t n_pad, int8_t* __restrict__ dcodes, float* __restrict__ dscales) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_pad; r += (int64_t)gridDim.x * blockDim.x) {
    int4 v[4] = {make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0), make_int4(0, 0, 0, 0)};
    float sc = 0.f;
    if (r < n) {
      const int64_t src = inv ? inv[idx[r]] : idx[r];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __ldg(reinterpret_cast<const int4*>(codes + s1_chunk_offset(src, c, 64)));
      sc = __ldg(scales + src);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) *reinterpret_cast<int4*>(dcodes + s1_chunk_offset(r, c, 64)) = v[c];
    dscales[r] = sc;
  }
}

// gather interleaved stage-1 code rows (index_select)
__global__ void gather_codes_kernel(const int8_t* __restrict__ src, const float* __restrict__ ssc,
                                    const int32_t* __restrict__ inv, const int64_t* __restrict__ idx, int64_t n,
                                    int8_t* __restrict__ dst, float* __restrict__ dsc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> 2;
    const int c = int(i & 3);
    const int64_t pos = inv ? inv[idx[r]] : idx[r];
    *reinterpret_cast<int4*>(dst + s1_chunk_offset(r, c, 64)) = *reinterpret_cast<const int4*>(src + s1_chunk_offset(pos, c, 64));
    if (c == 0) dsc[r] = ssc[pos];
  }
}

// Threshold of the lam-row sample (the n_rank-th largest sampled score per query,
// hindexer.py:115-132) without materialising the B x lam score matrix:
//   1. pilot: score the first lam0 sample rows (a uniform subsample: the Feistel prefix is a
//      uniform random order) and take their n0-th largest t0, with n0 set ~6 sigma above the
//      expected count of rows above the true threshold, so t0 <= t with overwhelming probability
//   2. scan the whole sample with the fused filter (>= t0), appending only the passers' score keys
//   3. the n_rank-th largest passer key IS the n_rank-th largest sampled score whenever at least
//      n_rank rows passed (every row >= t passes); otherwise (or on capacity overflow) fall back to
//      scoring the full sample.  Exact in every case.
//
// With `fail` (device int) the pilot's outcome is not read back: the pilot threshold is used and a
// failed pilot (fewer than n_rank passers, or key-buffer / segment overflow) only sets *fail, which
// the caller checks after its end-of-call synchronisation and reruns with force_full.
int sample_threshold_tc(molr_ctx* ctx, int mode, const int8_t* scodes, const float* sscales, int64_t lam, int B,
                        const int8_t* qc, int64_t n_rank, Scratch& ss, uint32_t* tkey, cudaStream_t s,
                        bool force_full = false, int* fail = nullptr, const S1Deferred* defer = nullptr) {
  const bool raw = mode == MOLR_S1_INT8_RAW;
  const double p = double(n_rank) / double(lam);
  int64_t lam0 = (int64_t)std::ceil(16.0 / p);
  lam0 = (lam0 + 255) / 256 * 256;
  if (!force_full && !dev_knob("MOLR_NO_PILOT") && lam0 * 4 <= lam) {
    const double mu = double(lam0) * p;
    int64_t n0 = std::min<int64_t>(lam0, (int64_t)std::ceil(mu + 6.0 * std::sqrt(mu) + 16.0));
    if (const char* e = dev_knob("MOLR_PILOT_N0")) n0 = std::max<int64_t>(1, std::min<int64_t>(lam0, atoll(e)));  // tests
    const double expect = double(lam) * double(n0) / double(lam0);
    const int64_t cap = (int64_t)(2.0 * expect) + 2048;
    Scratch pilot, t0, keys, counts, flag;
    MOLR_TRY(pilot.alloc(size_t(B) * lam0 * 4, s));
    MOLR_TRY(t0.alloc(size_t(B) * 4, s));
    MOLR_TRY(keys.alloc(size_t(B) * cap * 4, s));
    MOLR_TRY(counts.alloc(size_t(B) * 8, s));
    MOLR_TRY(flag.alloc(sizeof(int) * 2, s));
    Scratch mm;
    const int64_t lp = (lam + 255) / 256 * 256;
    MOLR_TRY(mm.alloc(size_t(lp / 32) * sizeof(float2), s));
    {
      KTimer t(ctx, "stage1_sample_scan_tc", s, double(B) * lam);
      MOLR_TRY(s1_tc_scan(ctx, mode, scodes, sscales, nullptr, nullptr, lam0, B, qc, nullptr, 0, 0, nullptr, nullptr,
                          pilot.p, lam0, s));
      MOLR_TRY(nth_largest_rows(ctx, B, lam0, pilot.p, raw, lam0, nullptr, 0, n0, t0.as<uint32_t>(), s));
      MOLR_TRY(chunk_minmax(ctx, sscales, 0, lp / 32, mm.as<float2>(), s));
      MOLR_CUDA(cudaMemsetAsync(counts.p, 0, size_t(B) * 8, s));
      MOLR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int) * 2, s));
      MOLR_TRY(s1_tc_scan(ctx, mode, scodes, sscales, mm.as<float2>(), nullptr, lam, B, qc, t0.as<uint32_t>(), 0, cap,
                          keys.as<int32_t>(), counts.as<int64_t>(), nullptr, 0, s, /*emit_keys=*/true, defer));
    }
    int* fl = fail ? fail : flag.as<int>();
    {
      KTimer t(ctx, "select_nth", s, double(B) * expect);
      MOLR_TRY(nth_largest_keys(ctx, B, cap, keys.as<uint32_t>(), counts.as<int64_t>(), n_rank, tkey, fl, s));
      max_count_kernel<<<div_up(B, 256), 256, 0, s>>>(B, counts.as<int64_t>(), cap, fl);
      MOLR_LAUNCHED(ctx);
    }
    if (fail) return MOLR_OK;  // checked after the caller's end-of-call synchronisation
    int hf = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (!hf) return MOLR_OK;
  }
  // full sample: write every score, then select
  MOLR_TRY(ss.alloc(size_t(B) * lam * 4, s));
  {
    KTimer t(ctx, "stage1_sample_scan_tc", s, double(B) * lam);
    MOLR_TRY(s1_tc_scan(ctx, mode, scodes, sscales, nullptr, nullptr, lam, B, qc, nullptr, 0, 0, nullptr, nullptr,
                        ss.p, lam, s));
  }
  KTimer t(ctx, "select_nth", s, double(B) * lam);
  return nth_largest_rows(ctx, B, lam, ss.p, raw, lam, nullptr, 0, n_rank, tkey, s);
}


// Float view: score the sampled rows (v row in registers, the s1_dot64 order of
// scan_scores_kernel) and append the ascending keys of the scores >= t0[b] (pilot threshold).
__global__ void __launch_bounds__(256) sample_keys_f32_kernel(int64_t n, const float* __restrict__ vf,
                                                              const int64_t* __restrict__ rows_idx, int B,
                                                              const float* __restrict__ qf, const uint32_t* __restrict__ t0,
                                                              int64_t cap, uint32_t* __restrict__ keys,
                                                              int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char sq[];
  float* q = reinterpret_cast<float*>(sq);
  uint32_t* tk = reinterpret_cast<uint32_t*>(sq + size_t(B) * 256);
  for (int i = threadIdx.x; i < B * 64; i += blockDim.x) q[i] = qf[i];
  for (int i = threadIdx.x; i < B; i += blockDim.x) tk[i] = t0[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows_idx[i];
    float v[64];
    const float4* v4 = reinterpret_cast<const float4*>(vf + r * 64);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 x = __ldg(v4 + k);
      v[4 * k] = x.x, v[4 * k + 1] = x.y, v[4 * k + 2] = x.z, v[4 * k + 3] = x.w;
    }
    for (int b = 0; b < B; ++b) {
      const uint32_t key = f32_key(s1_dot64(v, q + b * 64));
      if (key >= tk[b]) {
        const int64_t pos = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(counts + b), 1ull);
        if (pos < cap) keys[int64_t(b) * cap + pos] = key;
      }
    }
  }
}

// The float view's sampled threshold with the pilot filter of sample_threshold_tc (exact: the
// n-th largest passer key is the n-th largest sample score whenever >= n rows pass t0).
int sample_threshold_f32(molr_ctx* ctx, const molr_cache* c, const int64_t* samp, int64_t lam, int B, const float* q,
                         int64_t n_rank, Scratch& ss, uint32_t* tkey, cudaStream_t s) {
  const double p = double(n_rank) / double(lam);
  int64_t lam0 = (int64_t)std::ceil(16.0 / p);
  lam0 = (lam0 + 255) / 256 * 256;
  if (c->d1 == 64 && !dev_knob("MOLR_NO_PILOT") && lam0 * 4 <= lam) {
    const double mu = double(lam0) * p;
    int64_t n0 = std::min<int64_t>(lam0, (int64_t)std::ceil(mu + 6.0 * std::sqrt(mu) + 16.0));
    if (const char* e = dev_knob("MOLR_PILOT_N0")) n0 = std::max<int64_t>(1, std::min<int64_t>(lam0, atoll(e)));
    const double expect = double(lam) * double(n0) / double(lam0);
    const int64_t cap = (int64_t)(2.0 * expect) + 2048;
    Scratch pilot, t0, keys, counts, flag;
    MOLR_TRY(pilot.alloc(size_t(B) * lam0 * 4, s));
    MOLR_TRY(t0.alloc(size_t(B) * 4, s));
    MOLR_TRY(keys.alloc(size_t(B) * cap * 4, s));
    MOLR_TRY(counts.alloc(size_t(B) * 8, s));
    MOLR_TRY(flag.alloc(sizeof(int) * 2, s));
    {
      KTimer t(ctx, "stage1_sample_pilot", s, double(B) * lam0);
      MOLR_TRY(scan_scores(ctx, MOLR_S1_FLOAT, lam0, 64, c->s1_f32, nullptr, false, nullptr, nullptr, samp, B, q, nullptr,
                           pilot.p, lam0, s));
      MOLR_TRY(nth_largest_rows(ctx, B, lam0, pilot.p, false, lam0, nullptr, 0, n0, t0.as<uint32_t>(), s));
      MOLR_CUDA(cudaMemsetAsync(counts.p, 0, size_t(B) * 8, s));
      MOLR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int) * 2, s));
    }
    if (s1_bf_supported(c, MOLR_S1_FLOAT)) {
      // the sampled rows' fp16 image through the tensor-core filter (>= t0, exact fp32 re-check),
      // then the exact fp32 keys of the passers
      Scratch f32r, himg, hn, hc, pids;
      F16View V;
      MOLR_TRY(s1_f16_image(ctx, c, samp, lam, f32r, himg, hn, hc, &V, s));
      MOLR_TRY(pids.alloc(size_t(B) * cap * 4, s));
      MOLR_TRY(s1_f16_filter(ctx, V, B, q, t0.as<uint32_t>(), 0, cap, pids.as<int32_t>(), counts.as<int64_t>(), s,
                             "stage1_sample_scan_f16"));
      MOLR_TRY(s1_passer_keys(ctx, B, cap, pids.as<int32_t>(), counts.as<int64_t>(), V.f32, q, keys.as<uint32_t>(), s));
    } else {
      KTimer t(ctx, "stage1_sample_scan", s, double(B) * lam);
      const int bchunk = 128;  // 32 KB of queries per launch
      for (int b0 = 0; b0 < B; b0 += bchunk) {
        const int bb = std::min(bchunk, B - b0);
        const size_t smem = size_t(bb) * 260;
        const int blocks = (int)imin64(div_up(lam, 256), int64_t(ctx->num_sms) * 8);
        sample_keys_f32_kernel<<<blocks, 256, smem, s>>>(lam, c->s1_f32, samp, bb, q + size_t(b0) * 64,
                                                         t0.as<uint32_t>() + b0, cap, keys.as<uint32_t>() + size_t(b0) * cap,
                                                         counts.as<int64_t>() + b0);
        MOLR_LAUNCHED(ctx);
      }
    }
    {
      KTimer t(ctx, "select_nth", s, double(B) * expect);
      MOLR_TRY(nth_largest_keys(ctx, B, cap, keys.as<uint32_t>(), counts.as<int64_t>(), n_rank, tkey, flag.as<int>(), s));
      max_count_kernel<<<div_up(B, 256), 256, 0, s>>>(B, counts.as<int64_t>(), cap, flag.as<int>());
      MOLR_LAUNCHED(ctx);
    }
    int hf = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (!hf) return MOLR_OK;
  }
  MOLR_TRY(ss.alloc(size_t(B) * lam * 4, s));
  {
    KTimer t(ctx, "stage1_sample_scan", s, double(B) * lam);
    MOLR_TRY(scan_scores(ctx, MOLR_S1_FLOAT, lam, c->d1, c->s1_f32, nullptr, false, nullptr, nullptr, samp, B, q, nullptr,
                         ss.p, lam, s));
  }
  KTimer t(ctx, "select_nth", s, double(B) * lam);
  return nth_largest_rows(ctx, B, lam, ss.p, false, lam, nullptr, 0, n_rank, tkey, s);
}


// global sample rows inside [lo, hi) -> local row ids (order irrelevant: only the top keys matter)
__global__ void shard_rows_kernel(int64_t lam, const int64_t* __restrict__ samp, int64_t lo, int64_t hi,
                                  int64_t* __restrict__ loc, unsigned long long* __restrict__ cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < lam; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = samp[j];
    if (r >= lo && r < hi) loc[atomicAdd(cnt, 1ull)] = r - lo;
  }
}

// per query: the nk largest score keys (the nk-th largest is t[b]: every key > t plus copies of t),
// padded with 0 (below every real key) up to n_keep
__global__ void __launch_bounds__(256) top_keys_kernel(int64_t m, const void* __restrict__ sc, int is_int,
                                                      const uint32_t* __restrict__ t, int64_t nk, int64_t n_keep,
                                                      uint32_t* __restrict__ out) {
  __shared__ unsigned long long n_gt;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) n_gt = 0;
  __syncthreads();
  uint32_t* o = out + int64_t(b) * n_keep;
  const uint32_t tb = nk > 0 ? t[b] : 0u;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t idx = int64_t(b) * m + i;
    const uint32_t key = is_int ? i32_key(reinterpret_cast<const int32_t*>(sc)[idx])
                                : f32_key(reinterpret_cast<const float*>(sc)[idx]);
    if (key > tb) {
      const unsigned long long p = atomicAdd(&n_gt, 1ull);
      if ((int64_t)p < nk) o[p] = key;
    }
  }
  __syncthreads();
  const int64_t filled = (int64_t)n_gt < nk ? (int64_t)n_gt : nk;
  for (int64_t i = filled + threadIdx.x; i < n_keep; i += blockDim.x)
    o[i] = i < nk ? tb : 0u;
}

// the same from a list of ascending keys per query (row b: keys[b*cap, b*cap + min(counts[b], cap)))
__global__ void __launch_bounds__(256) top_keys_list_kernel(int64_t cap, const uint32_t* __restrict__ keys,
                                                           const int64_t* __restrict__ counts,
                                                           const uint32_t* __restrict__ t, int64_t nk, int64_t n_keep,
                                                           uint32_t* __restrict__ out) {
  __shared__ unsigned long long n_gt;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) n_gt = 0;
  __syncthreads();
  uint32_t* o = out + int64_t(b) * n_keep;
  const uint32_t tb = t[b];
  const int64_t m = counts[b] < cap ? counts[b] : cap;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t key = keys[int64_t(b) * cap + i];
    if (key > tb) {
      const unsigned long long p = atomicAdd(&n_gt, 1ull);
      if ((int64_t)p < nk) o[p] = key;
    }
  }
  __syncthreads();
  const int64_t filled = (int64_t)n_gt < nk ? (int64_t)n_gt : nk;
  for (int64_t i = filled + threadIdx.x; i < n_keep; i += blockDim.x) o[i] = i < nk ? tb : 0u;
}

__global__ void fill_i64_kernel(int n, int64_t v, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

}  // namespace molr

using namespace molr;

extern "C" {

static int mol_common_checks(const molr_cache* c, const molr_gating* g, int k_u) {
  if (!c || !g) MOLR_FAIL(MOLR_ERR_INVALID, "null cache/gating");
  if (g->G != k_u * c->k_x || c->G != g->G)
    MOLR_FAIL(MOLR_ERR_DIMENSION, "logit grid mismatch: k_u*k_x=%d, cache G=%d, gating G=%d", k_u * c->k_x, c->G,
              g->G);
  return MOLR_OK;
}

int molr_score(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
               const float* uw, float tau, const int64_t* off, const int64_t* ids, float* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_TRY(mol_common_checks(c, g, k_u));
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  int64_t total = int64_t(B) * c->X;
  std::vector<int64_t> hoff;
  if (off) {
    hoff.resize(B + 1);
    MOLR_CUDA(cudaMemcpyAsync(hoff.data(), off, size_t(B + 1) * 8, cudaMemcpyDefault, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    total = hoff[B];
    for (int b = 0; b < B; ++b)
      if (hoff[b + 1] - hoff[b] <= 0) MOLR_FAIL(MOLR_ERR_EMPTY_CANDIDATES, "no candidates to score");
  }
  In iue, iuw, ioff, iids;
  MOLR_TRY(iue.stage(ue, size_t(B) * k_u * c->d * 4, s));
  MOLR_TRY(iuw.stage(uw, size_t(B) * g->G * 4, s));
  Scratch sb, se, bad;
  Segs<int64_t> segs;
  segs.X = c->X;
  if (off) {
    MOLR_TRY(ioff.stage(off, size_t(B + 1) * 8, s));
    MOLR_TRY(iids.stage(ids, size_t(total) * 8, s));
    MOLR_TRY(sb.alloc(size_t(B) * 8, s));
    MOLR_TRY(se.alloc(size_t(B) * 8, s));
    csr_to_segs_kernel<<<div_up(B, 256), 256, 0, s>>>(B, ioff.as<int64_t>(), sb.as<int64_t>(), se.as<int64_t>());
    MOLR_LAUNCHED(ctx);
    // ids must lie inside the corpus (mol.py:339-340)
    MOLR_TRY(bad.alloc(4, s));
    MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
    validate_ids_kernel<<<std::min(div_up(total, 256), ctx->num_sms * 8), 256, 0, s>>>(total, iids.as<int64_t>(),
                                                                                       c->X, bad.as<int>());
    MOLR_LAUNCHED(ctx);
    int hb = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (hb) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "candidate id outside the corpus");
    segs.begin = sb.as<int64_t>();
    segs.end = se.as<int64_t>();
    segs.ids = iids.as<int64_t>();
  }
  Out o;
  MOLR_TRY(o.stage(out, size_t(total) * 4, s));
  {
    KTimer t(ctx, "mol_score", s, double(total));
    MOLR_TRY(mol_score_any<int64_t>(ctx, c, g, B, k_u, iue.as<float>(), iuw.as<float>(), tau, segs, o.as<float>(),
                                    c->X, s));
  }
  return finish_outputs(s, {&o});
}

int molr_mol_top_k(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
                   const float* uw, float tau, const int64_t* off, const int64_t* ids, int k, int64_t* out_ids,
                   float* out_scores, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_TRY(mol_common_checks(c, g, k_u));
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  int64_t total = int64_t(B) * c->X;
  if (off) {
    std::vector<int64_t> hoff(B + 1);
    MOLR_CUDA(cudaMemcpyAsync(hoff.data(), off, size_t(B + 1) * 8, cudaMemcpyDefault, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    total = hoff[B];
    for (int b = 0; b < B; ++b) {
      int64_t n = hoff[b + 1] - hoff[b];
      if (n <= 0) MOLR_FAIL(MOLR_ERR_EMPTY_CANDIDATES, "no candidates to rank");
      if (k < 1 || k > n) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "k=%d outside [1, %lld]", k, (long long)n);
    }
  } else if (k < 1 || k > c->X) {
    MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "k=%d outside [1, %lld]", k, (long long)c->X);
  } else {
    // whole-corpus ranking materialises a (users x X) f32 score block: bound it (4 GB) by running
    // the users in chunks (100M items x 1024 users would otherwise need 400 GB)
    const int64_t per = std::max<int64_t>(1, (int64_t(1) << 30) / std::max<int64_t>(c->X, 1));
    if (B > per) {
      for (int64_t b0 = 0; b0 < B; b0 += per) {
        const int nb = int(std::min<int64_t>(per, B - b0));
        MOLR_TRY(molr_mol_top_k(ctx, c, g, nb, k_u, ue + b0 * k_u * c->d, uw + b0 * c->G, tau, nullptr, nullptr, k,
                                out_ids + b0 * k, out_scores + b0 * k, stream));
      }
      return MOLR_OK;
    }
  }
  Scratch sc;
  MOLR_TRY(sc.alloc(size_t(total) * 4, s));
  MOLR_TRY(molr_score(ctx, c, g, B, k_u, ue, uw, tau, off, ids, sc.as<float>(), s));
  In ioff, iids;
  Scratch sb, se;
  Segs<int64_t> segs;
  segs.X = c->X;
  if (off) {
    MOLR_TRY(ioff.stage(off, size_t(B + 1) * 8, s));
    MOLR_TRY(iids.stage(ids, size_t(total) * 8, s));
    MOLR_TRY(sb.alloc(size_t(B) * 8, s));
    MOLR_TRY(se.alloc(size_t(B) * 8, s));
    csr_to_segs_kernel<<<div_up(B, 256), 256, 0, s>>>(B, ioff.as<int64_t>(), sb.as<int64_t>(), se.as<int64_t>());
    MOLR_LAUNCHED(ctx);
    segs.begin = sb.as<int64_t>();
    segs.end = se.as<int64_t>();
    segs.ids = iids.as<int64_t>();
  }
  Out oi, os;
  MOLR_TRY(oi.stage(out_ids, size_t(B) * k * 8, s));
  MOLR_TRY(os.stage(out_scores, size_t(B) * k * 4, s));
  {
    KTimer t(ctx, "topk_segmented", s, double(total));
    MOLR_TRY(segmented_top_k<int64_t>(ctx, B, segs, sc.as<float>(), c->X, k, 0, oi.as<int64_t>(), os.as<float>(), s));
  }
  return finish_outputs(s, {&oi, &os});
}

int molr_index_select(molr_ctx* ctx, const molr_cache* c, int64_t n, const int64_t* ids, molr_cache** out) {
  if (!ctx || !c || !out) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, nullptr);
  if (c->s1_codes) MOLR_TRY(s1_seal(const_cast<molr_cache*>(c), s));
  molr_cache* r = nullptr;
  MOLR_TRY(molr_cache_alloc(ctx, n, c->k_x, c->d, c->G, c->d1, c->storage, &r));
  if (n > 0) {
    In ii;
    int st = ii.stage(ids, size_t(n) * 8, s);
    auto g = [&](const void* src, void* dst, int64_t row_bytes) {
      if (st == MOLR_OK && src) st = gather_rows(ctx, n, row_bytes, src, ii.as<int64_t>(), dst, s);
    };
    g(c->embs_bf16, r->embs_bf16, int64_t(c->k_x) * c->d * 2);
    g(c->embs_f32, r->embs_f32, int64_t(c->k_x) * c->d * 4);
    if (st == MOLR_OK && r->embs_hl) st = build_embs_hilo(r, 0, n, s);
    g(c->gp_bf16, r->gp_bf16, int64_t(c->G) * 2);
    g(c->gp_f32, r->gp_f32, int64_t(c->G) * 4);
    g(c->s1_f32, r->s1_f32, int64_t(c->d1) * 4);
    if (st == MOLR_OK && c->s1_codes) {
      if (s1_interleaved(c->d1)) {
        gather_codes_kernel<<<std::min(div_up(n * 4, 256), ctx->num_sms * 8), 256, 0, s>>>(
            c->s1_codes, c->s1_scales, c->s1_inv, ii.as<int64_t>(), n, r->s1_codes, r->s1_scales);
        if (cudaGetLastError() != cudaSuccess) st = MOLR_ERR_CUDA;
        ctx->launches++;
      } else {
        g(c->s1_codes, r->s1_codes, int64_t(c->d1));
        g(c->s1_scales, r->s1_scales, 4);
      }
    }
    if (st == MOLR_OK && r->s1_chunk_mm) st = s1_update_chunk_mm(r, 0, n, s);
    if (st == MOLR_OK && cudaStreamSynchronize(s) != cudaSuccess) st = MOLR_ERR_CUDA;
    if (st) {
      molr_cache_destroy(r);
      return st;
    }
  }
  *out = r;
  return MOLR_OK;
}

// Fused batched two-stage retrieval.  See header.  Steps:
//  1. stage-1 query = mean of user components; quantize (int8 views)          engine.py:131
//  2. lam distinct rows from a seeded Feistel permutation prefix (batch-shared) hindexer.py:125
//  3. sample scores with the same arithmetic as the scan; n-th largest         hindexer.py:156-158
//  4. scan + threshold filter, passers appended per query                      hindexer.py:155,159-163
//  5. MoL scoring of each query's passers; fallback to the corpus if < k      engine.py:134-137
//  6. top-k by (score desc, id asc)                                            mol.py:407
// tkeys_in != null: the per-query thresholds are given (molr_two_stage_top_k_at) and steps 2-3
// are skipped; no_fallback: queries with < k passers keep their short lists (the caller decides
// the fallback from the global counts).
static int two_stage_impl(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
                          const float* uw, float tau, int mode, int64_t k_prime, int64_t lam, uint64_t seed,
                          int comparator, int k, int64_t id_offset, int64_t* out_ids, float* out_scores,
                          int64_t* out_cand, void* stream, const uint32_t* tkeys_in, bool no_fallback) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_TRY(mol_common_checks(c, g, k_u));
  MOLR_TRY(check_view(c, mode));
  if (c->d1 != c->d) MOLR_FAIL(MOLR_ERR_DIMENSION, "stage-1 dim %d != d %d", c->d1, c->d);
  if (k_prime < 1) MOLR_FAIL(MOLR_ERR_INVALID, "k_prime must be >= 1");
  if (!tkeys_in) {
    if (k_prime > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "k_prime %lld exceeds corpus %lld", (long long)k_prime,
                                  (long long)c->X);
    if (lam < 1 || lam > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "lambda %lld outside [1, %lld]", (long long)lam,
                                         (long long)c->X);
  }
  if (k < 1) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "k=%d", k);
  if (mode != MOLR_S1_FLOAT && (c->d1 % 16) != 0) MOLR_FAIL(MOLR_ERR_DIMENSION, "int8 batched scan needs d1%%16==0");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  WorkspaceScope ws(ctx, s);  // this call synchronises its stream before returning
  const int64_t X = c->X;
  const int kk = (int)imin64(k, X);
  In iue, iuw;
  MOLR_TRY(iue.stage(ue, size_t(B) * k_u * c->d * 4, s));
  MOLR_TRY(iuw.stage(uw, size_t(B) * g->G * 4, s));
  Out oi, os, oc;
  MOLR_TRY(oi.stage(out_ids, size_t(B) * k * 8, s));
  MOLR_TRY(os.stage(out_scores, size_t(B) * k * 4, s));
  MOLR_TRY(oc.stage(out_cand, out_cand ? size_t(B) * 8 : 0, s));
  if (kk < k) {  // short corpus: pad the tail
    MOLR_CUDA(cudaMemsetAsync(oi.dptr, 0xff, size_t(B) * k * 8, s));
  }

  Segs<int32_t> segs;
  segs.X = X;
  Scratch cand, counts, sb, se;
  std::vector<int64_t> hcnt(B, X);
  if (k_prime < X || tkeys_in) {
    // 1. queries
    Scratch q, qc, qs;
    MOLR_TRY(q.alloc(size_t(B) * c->d * 4, s));
    s1_query_kernel<<<div_up(int64_t(B) * c->d, 256), 256, 0, s>>>(B, k_u, c->d, iue.as<float>(), q.as<float>());
    MOLR_LAUNCHED(ctx);
    if (mode != MOLR_S1_FLOAT) {
      MOLR_TRY(qc.alloc(size_t(B) * c->d1, s));
      MOLR_TRY(qs.alloc(size_t(B) * 4, s));
      MOLR_TRY(prepare_queries(ctx, mode, B, c->d1, q.as<float>(), qc.as<int8_t>(), qs.as<float>(), s));
    }
    // 2-6 run as one stream of launches with no host round trip: the pilot's outcome, the
    // filter's per-CTA segment and per-query capacity overflows are recorded on the device and
    // checked once after the call's single synchronisation; the (rare) overflow reruns 2-6 with
    // the exact sizes.
    const bool use_tc = s1_tc_supported(c, mode);
    int64_t cap = imin64(X, k_prime + k_prime / 4 + 1024);
    bool full_sample = false;
    int64_t seg_min_pilot = 0, seg_min_main = 0;
    MOLR_TRY(counts.alloc(size_t(B) * 8, s));
    Scratch dflags;  // [0] pilot failed  [1] pilot key-scan segment need  [2] filter segment need
    MOLR_TRY(dflags.alloc(16, s));
    int hfl[4] = {0, 0, 0, 0};
    for (int attempt = 0; attempt < 4; ++attempt) {
      MOLR_CUDA(cudaMemsetAsync(dflags.p, 0, 16, s));
      int64_t seg_used_pilot = 0, seg_used_main = 0;
      const S1Deferred dpilot{dflags.as<int>() + 1, seg_min_pilot, &seg_used_pilot};
      const S1Deferred dmain{dflags.as<int>() + 2, seg_min_main, &seg_used_main};
      Scratch ss, tkey;
      MOLR_TRY(tkey.alloc(size_t(B) * 4, s));
      if (tkeys_in) {
        MOLR_CUDA(cudaMemcpyAsync(tkey.p, tkeys_in, size_t(B) * 4, cudaMemcpyDefault, s));
      } else {
        // 2. sample
        int bits = 2;
        while ((int64_t(1) << bits) < X) bits += 2;
        Scratch samp;
        MOLR_TRY(samp.alloc(size_t(lam) * 8, s));
        feistel_sample_kernel<<<div_up(lam, 256), 256, 0, s>>>(X, lam, seed, bits / 2, samp.as<int64_t>());
        MOLR_LAUNCHED(ctx);
        // 3. n-th largest sampled score per query
        const double nr = std::nearbyint(double(k_prime * lam) / double(X));  // Python round(): half-even
        const int64_t n_rank = std::max<int64_t>(1, (int64_t)nr);
        if (use_tc) {
          // gather the sample rows into a contiguous operand, then the tensor-core scans
          const int64_t lp = (lam + 255) / 256 * 256;
          Scratch scodes, sscales;
          MOLR_TRY(scodes.alloc(size_t(lp) * 64, s));
          MOLR_TRY(sscales.alloc(size_t(lp) * 4, s));
          gather_sample_kernel<<<div_up(lp, 256), 256, 0, s>>>(c->s1_codes, c->s1_scales, c->s1_inv, samp.as<int64_t>(), lam,
                                                              lp, scodes.as<int8_t>(), sscales.as<float>());
          MOLR_LAUNCHED(ctx);
          MOLR_TRY(sample_threshold_tc(ctx, mode, scodes.as<int8_t>(), sscales.as<float>(), lam, B, qc.as<int8_t>(),
                                       n_rank, ss, tkey.as<uint32_t>(), s, full_sample, dflags.as<int>(), &dpilot));
        } else if (mode == MOLR_S1_FLOAT) {
          MOLR_TRY(sample_threshold_f32(ctx, c, samp.as<int64_t>(), lam, B, q.as<float>(), n_rank, ss,
                                        tkey.as<uint32_t>(), s));
        } else {
          MOLR_TRY(ss.alloc(size_t(B) * lam * 4, s));
          {
            KTimer t(ctx, "stage1_sample_scan", s, double(B) * lam);
            MOLR_TRY(scan_scores(ctx, mode, lam, c->d1, c->s1_f32, c->s1_codes, s1_interleaved(c->d1), c->s1_inv,
                                 c->s1_scales, samp.as<int64_t>(), B, q.as<float>(), qc.as<int8_t>(), ss.p, lam, s));
          }
          KTimer t(ctx, "select_nth", s, double(B) * lam);
          MOLR_TRY(nth_largest_rows(ctx, B, lam, ss.p, mode == MOLR_S1_INT8_RAW, lam, nullptr, 0, n_rank,
                                    tkey.as<uint32_t>(), s));
        }
      }
      // 4. filter scan with capacity (overflow: rerun with the exact maximum)
      MOLR_TRY(cand.alloc(size_t(B) * cap * 4, s));
      MOLR_CUDA(cudaMemsetAsync(counts.p, 0, size_t(B) * 8, s));
      const int per_q = mode == MOLR_S1_FLOAT ? c->d1 * 4 : c->d1;
      const int bchunk = std::max(1, std::min(B, (128 * 1024) / (per_q + 4)));  // queries per launch
      auto launch = [&](auto kern) -> int {
        for (int b0 = 0; b0 < B; b0 += bchunk) {
          const int bb = std::min(bchunk, B - b0);
          const size_t smem = size_t((bb * 4 + 15) / 16) * 16 + size_t(bb) * per_q;
          MOLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          int blocks = std::min(div_up(X, 256), ctx->num_sms * std::max(1, int((220 * 1024) / (smem + 1024))));
          kern<<<blocks, 256, smem, s>>>(X, c->d1, c->s1_f32, c->s1_codes, c->s1_inv, c->s1_scales, bb,
                                         q.as<float>() + size_t(b0) * c->d1, qc.p ? qc.as<int8_t>() + size_t(b0) * c->d1 : nullptr,
                                         tkey.as<uint32_t>() + b0, comparator == MOLR_STRICT, cap,
                                         cand.as<int32_t>() + size_t(b0) * cap, counts.as<int64_t>() + b0);
          MOLR_LAUNCHED(ctx);
        }
        return MOLR_OK;
      };
      if (s1_bf_supported(c, mode)) {
        MOLR_TRY(s1_bf_scan(ctx, c, B, q.as<float>(), tkey.as<uint32_t>(), comparator == MOLR_STRICT, cap,
                            cand.as<int32_t>(), counts.as<int64_t>(), s));
      } else if (use_tc) {
        KTimer t(ctx, "stage1_filter_tc", s, double(B) * X);
        MOLR_TRY(s1_tc_scan(ctx, mode, c->s1_codes, c->s1_scales, c->s1_chunk_mm, c->s1_perm, X, B, qc.as<int8_t>(),
                            tkey.as<uint32_t>(), comparator == MOLR_STRICT, cap, cand.as<int32_t>(), counts.as<int64_t>(),
                            nullptr, 0, s, false, &dmain));
      } else {
        KTimer t(ctx, "stage1_filter_scan", s, double(B) * X);
        if (mode == MOLR_S1_FLOAT) MOLR_TRY(launch(filter_scan_kernel<MOLR_S1_FLOAT>));
        else if (mode == MOLR_S1_INT8) MOLR_TRY(launch(filter_scan_kernel<MOLR_S1_INT8>));
        else MOLR_TRY(launch(filter_scan_kernel<MOLR_S1_INT8_RAW>));
      }
      MOLR_TRY(sb.alloc(size_t(B) * 8, s));
      MOLR_TRY(se.alloc(size_t(B) * 8, s));
      cap_segs_kernel<<<div_up(B, 256), 256, 0, s>>>(B, cap, counts.as<int64_t>(), sb.as<int64_t>(), se.as<int64_t>());
      MOLR_LAUNCHED(ctx);
      segs.begin = sb.as<int64_t>();
      segs.end = se.as<int64_t>();
      segs.ids = cand.as<int32_t>();
      // 5. MoL over the passers (queries with < k passers are redone on the whole corpus below,
      //    engine.py:134-135)
      Scratch sc;
      MOLR_TRY(sc.alloc(size_t(B) * cap * 4, s));
      KTimer tm(ctx, "mol_score", s, 0.0);
      MOLR_TRY(mol_score_any<int32_t>(ctx, c, g, B, k_u, iue.as<float>(), iuw.as<float>(), tau, segs, sc.as<float>(), 0,
                                      s));
      tm.stop();
      // 6. top-k per query
      KTimer tk(ctx, "topk_segmented", s, 0.0);
      MOLR_TRY(segmented_top_k<int32_t>(ctx, B, segs, sc.as<float>(), 0, k, id_offset, oi.as<int64_t>(),
                                        os.as<float>(), s));
      tk.stop();
      // the call's one synchronisation: passer counts and the deferred overflow flags
      MOLR_CUDA(cudaMemcpyAsync(hcnt.data(), counts.p, size_t(B) * 8, cudaMemcpyDeviceToHost, s));
      MOLR_CUDA(cudaMemcpyAsync(hfl, dflags.p, 16, cudaMemcpyDeviceToHost, s));
      MOLR_CUDA(cudaStreamSynchronize(s));
      double pairs = 0;
      for (int b = 0; b < B; ++b) pairs += double(std::min<int64_t>(hcnt[b], cap));
      tm.work = pairs;
      tk.work = pairs;
      bool redo = false;
      if (hfl[0]) {  // the pilot threshold was not provably the sample's n-th largest
        full_sample = true;
        redo = true;
      }
      if (hfl[1] > seg_used_pilot) {
        seg_min_pilot = hfl[1];
        redo = true;
      }
      if (hfl[2] > seg_used_main) {
        seg_min_main = hfl[2];
        redo = true;
      }
      const int64_t mx = *std::max_element(hcnt.begin(), hcnt.end());
      if (mx > cap) {
        cap = mx;
        redo = true;
      }
      if (!redo) break;
      if (attempt == 3) MOLR_FAIL(MOLR_ERR_CAPACITY, "candidate buffers still overflowing after 3 retries");
      cand.reset();
    }
    std::vector<int> fallback;
    for (int b = 0; b < B && !no_fallback; ++b)
      if (hcnt[b] < kk) fallback.push_back(b);
    if (!fallback.empty()) {
      // dense MoL for the few queries whose candidate set came back smaller than k
      const int F = (int)fallback.size();
      Scratch fue, fuw, fsc, fid, fso;
      MOLR_TRY(fue.alloc(size_t(F) * k_u * c->d * 4, s));
      MOLR_TRY(fuw.alloc(size_t(F) * g->G * 4, s));
      for (int i = 0; i < F; ++i) {
        int b = fallback[i];
        MOLR_CUDA(cudaMemcpyAsync(fue.as<float>() + size_t(i) * k_u * c->d, iue.as<float>() + size_t(b) * k_u * c->d,
                                  size_t(k_u) * c->d * 4, cudaMemcpyDeviceToDevice, s));
        MOLR_CUDA(cudaMemcpyAsync(fuw.as<float>() + size_t(i) * g->G, iuw.as<float>() + size_t(b) * g->G,
                                  size_t(g->G) * 4, cudaMemcpyDeviceToDevice, s));
      }
      MOLR_TRY(fsc.alloc(size_t(F) * X * 4, s));
      Segs<int32_t> dense;
      dense.X = X;
      MOLR_TRY(mol_score_any<int32_t>(ctx, c, g, F, k_u, fue.as<float>(), fuw.as<float>(), tau, dense,
                                      fsc.as<float>(), X, s));
      MOLR_TRY(fid.alloc(size_t(F) * k * 8, s));
      MOLR_TRY(fso.alloc(size_t(F) * k * 4, s));
      MOLR_TRY(segmented_top_k<int32_t>(ctx, F, dense, fsc.as<float>(), X, k, id_offset, fid.as<int64_t>(),
                                        fso.as<float>(), s));
      for (int i = 0; i < F; ++i) {
        int b = fallback[i];
        MOLR_CUDA(cudaMemcpyAsync(oi.as<int64_t>() + size_t(b) * k, fid.as<int64_t>() + size_t(i) * k, size_t(k) * 8,
                                  cudaMemcpyDeviceToDevice, s));
        MOLR_CUDA(cudaMemcpyAsync(os.as<float>() + size_t(b) * k, fso.as<float>() + size_t(i) * k, size_t(k) * 4,
                                  cudaMemcpyDeviceToDevice, s));
        hcnt[b] = X;
      }
    }
  } else {
    // k' >= X: every item is a candidate (engine.py:127-128)
    Scratch sc;
    MOLR_TRY(sc.alloc(size_t(B) * X * 4, s));
    MOLR_TRY(mol_score_any<int32_t>(ctx, c, g, B, k_u, iue.as<float>(), iuw.as<float>(), tau, segs, sc.as<float>(),
                                    X, s));
    MOLR_TRY(segmented_top_k<int32_t>(ctx, B, segs, sc.as<float>(), X, k, id_offset, oi.as<int64_t>(),
                                      os.as<float>(), s));
  }
  if (out_cand) MOLR_CUDA(cudaMemcpyAsync(oc.dptr, hcnt.data(), size_t(B) * 8, cudaMemcpyDefault, s));
  MOLR_CUDA(cudaStreamSynchronize(s));  // hcnt lives on this stack frame
  return finish_outputs(s, {&oi, &os, &oc});
}

int molr_two_stage_top_k(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
                         const float* uw, float tau, int mode, int64_t k_prime, int64_t lam, uint64_t seed,
                         int comparator, int k, int64_t id_offset, int64_t* out_ids, float* out_scores,
                         int64_t* out_cand, void* stream) {
  return two_stage_impl(ctx, c, g, B, k_u, ue, uw, tau, mode, k_prime, lam, seed, comparator, k, id_offset, out_ids,
                        out_scores, out_cand, stream, nullptr, false);
}

int molr_two_stage_top_k_at(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u, const float* ue,
                            const float* uw, float tau, int mode, int64_t cap_hint, const uint32_t* tkeys,
                            int comparator, int k, int64_t id_offset, int64_t* out_ids, float* out_scores,
                            int64_t* out_cand, void* stream) {
  if (!tkeys) MOLR_FAIL(MOLR_ERR_INVALID, "null thresholds");
  return two_stage_impl(ctx, c, g, B, k_u, ue, uw, tau, mode, std::max<int64_t>(1, std::min<int64_t>(cap_hint, c ? c->X : 1)),
                        1, 0, comparator, k, id_offset, out_ids, out_scores, out_cand, stream, tkeys, true);
}

int molr_sample_top_keys(molr_ctx* ctx, const molr_cache* c, int B, int k_u, const float* ue, int mode,
                         int64_t X_global, int64_t row_lo, int64_t lam, uint64_t seed, int64_t n_keep,
                         uint32_t* out_keys, void* stream) {
  if (!ctx || !c) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx/cache");
  MOLR_TRY(check_view(c, mode));
  if (c->d1 != c->d) MOLR_FAIL(MOLR_ERR_DIMENSION, "stage-1 dim %d != d %d", c->d1, c->d);
  if (X_global < c->X || row_lo < 0 || row_lo + c->X > X_global)
    MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "shard [%lld, %lld) outside the corpus [0, %lld)", (long long)row_lo,
              (long long)(row_lo + c->X), (long long)X_global);
  if (lam < 1 || lam > X_global) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "lambda %lld outside [1, %lld]", (long long)lam,
                                           (long long)X_global);
  if (n_keep < 1) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n_keep=%lld", (long long)n_keep);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  WorkspaceScope ws(ctx, s);
  In iue;
  MOLR_TRY(iue.stage(ue, size_t(B) * k_u * c->d * 4, s));
  Out ok;
  MOLR_TRY(ok.stage(out_keys, size_t(B) * n_keep * 4, s));
  Scratch q, qc, qs;
  MOLR_TRY(q.alloc(size_t(B) * c->d * 4, s));
  s1_query_kernel<<<div_up(int64_t(B) * c->d, 256), 256, 0, s>>>(B, k_u, c->d, iue.as<float>(), q.as<float>());
  MOLR_LAUNCHED(ctx);
  if (mode != MOLR_S1_FLOAT) {
    MOLR_TRY(qc.alloc(size_t(B) * c->d1, s));
    MOLR_TRY(qs.alloc(size_t(B) * 4, s));
    MOLR_TRY(prepare_queries(ctx, mode, B, c->d1, q.as<float>(), qc.as<int8_t>(), qs.as<float>(), s));
  }
  // the global sample (same Feistel permutation prefix as a single device), restricted to this shard
  int bits = 2;
  while ((int64_t(1) << bits) < X_global) bits += 2;
  Scratch samp, loc, cnt;
  MOLR_TRY(samp.alloc(size_t(lam) * 8, s));
  MOLR_TRY(loc.alloc(size_t(lam) * 8, s));
  MOLR_TRY(cnt.alloc(8, s));
  feistel_sample_kernel<<<div_up(lam, 256), 256, 0, s>>>(X_global, lam, seed, bits / 2, samp.as<int64_t>());
  MOLR_LAUNCHED(ctx);
  MOLR_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
  shard_rows_kernel<<<std::min(div_up(lam, 256), ctx->num_sms * 8), 256, 0, s>>>(lam, samp.as<int64_t>(), row_lo,
                                                                                 row_lo + c->X, loc.as<int64_t>(),
                                                                                 cnt.as<unsigned long long>());
  MOLR_LAUNCHED(ctx);
  unsigned long long hm = 0;
  MOLR_CUDA(cudaMemcpyAsync(&hm, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  const int64_t m = (int64_t)hm;
  const int64_t nk = std::min<int64_t>(n_keep, m);
  Scratch ss, tk;
  MOLR_TRY(tk.alloc(size_t(B) * 4, s));
  if (m > 0) {
    if (s1_tc_supported(c, mode)) {
      const int64_t lp = (m + 255) / 256 * 256;
      Scratch scodes, sscales;
      MOLR_TRY(scodes.alloc(size_t(lp) * 64, s));
      MOLR_TRY(sscales.alloc(size_t(lp) * 4, s));
      MOLR_TRY(s1_seal(const_cast<molr_cache*>(c), s));
      gather_sample_kernel<<<div_up(lp, 256), 256, 0, s>>>(c->s1_codes, c->s1_scales, c->s1_inv, loc.as<int64_t>(), m, lp,
                                                          scodes.as<int8_t>(), sscales.as<float>());
      MOLR_LAUNCHED(ctx);
      // pilot (as sample_threshold_tc): a low threshold t0 from the first lam0 local sample rows, the
      // fused filter keeps the keys >= t0, and the nk-th largest of those is the shard's nk-th
      // largest whenever >= nk rows passed; otherwise the full score matrix below
      const double p = double(nk) / double(m);
      int64_t lam0 = ((int64_t)std::ceil(16.0 / p) + 255) / 256 * 256;
      if (!dev_knob("MOLR_NO_PILOT") && lam0 * 4 <= m) {
        const double mu = double(lam0) * p;
        const int64_t n0 = std::min<int64_t>(lam0, (int64_t)std::ceil(mu + 6.0 * std::sqrt(mu) + 16.0));
        const int64_t cap = (int64_t)(2.0 * double(m) * double(n0) / double(lam0)) + 2048;
        const int64_t lp = (m + 255) / 256 * 256;
        Scratch pilot, t0, keys, counts, flag, mm;
        MOLR_TRY(pilot.alloc(size_t(B) * lam0 * 4, s));
        MOLR_TRY(t0.alloc(size_t(B) * 4, s));
        MOLR_TRY(keys.alloc(size_t(B) * cap * 4, s));
        MOLR_TRY(counts.alloc(size_t(B) * 8, s));
        MOLR_TRY(flag.alloc(sizeof(int) * 2, s));
        MOLR_TRY(mm.alloc(size_t(lp / 32) * sizeof(float2), s));
        MOLR_TRY(s1_tc_scan(ctx, mode, scodes.as<int8_t>(), sscales.as<float>(), nullptr, nullptr, lam0, B,
                            qc.as<int8_t>(), nullptr, 0, 0, nullptr, nullptr, pilot.p, lam0, s));
        MOLR_TRY(nth_largest_rows(ctx, B, lam0, pilot.p, mode == MOLR_S1_INT8_RAW, lam0, nullptr, 0, n0,
                                  t0.as<uint32_t>(), s));
        MOLR_TRY(chunk_minmax(ctx, sscales.as<float>(), 0, lp / 32, mm.as<float2>(), s));
        MOLR_CUDA(cudaMemsetAsync(counts.p, 0, size_t(B) * 8, s));
        MOLR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int) * 2, s));
        MOLR_TRY(s1_tc_scan(ctx, mode, scodes.as<int8_t>(), sscales.as<float>(), mm.as<float2>(), nullptr, m, B,
                            qc.as<int8_t>(), t0.as<uint32_t>(), 0, cap, keys.as<int32_t>(), counts.as<int64_t>(), nullptr,
                            0, s, /*emit_keys=*/true));
        MOLR_TRY(nth_largest_keys(ctx, B, cap, keys.as<uint32_t>(), counts.as<int64_t>(), nk, tk.as<uint32_t>(),
                                  flag.as<int>(), s));
        max_count_kernel<<<div_up(B, 256), 256, 0, s>>>(B, counts.as<int64_t>(), cap, flag.as<int>());
        MOLR_LAUNCHED(ctx);
        int hf = 0;
        MOLR_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        MOLR_CUDA(cudaStreamSynchronize(s));
        if (!hf) {
          top_keys_list_kernel<<<B, 256, 0, s>>>(cap, keys.as<uint32_t>(), counts.as<int64_t>(), tk.as<uint32_t>(), nk,
                                                 n_keep, ok.as<uint32_t>());
          MOLR_LAUNCHED(ctx);
          MOLR_CUDA(cudaStreamSynchronize(s));
          return finish_outputs(s, {&ok});
        }
      }
      MOLR_TRY(ss.alloc(size_t(B) * m * 4, s));
      MOLR_TRY(s1_tc_scan(ctx, mode, scodes.as<int8_t>(), sscales.as<float>(), nullptr, nullptr, m, B, qc.as<int8_t>(),
                          nullptr, 0, 0, nullptr, nullptr, ss.p, m, s));
    } else {
      MOLR_TRY(ss.alloc(size_t(B) * m * 4, s));
      if (mode != MOLR_S1_FLOAT && c->s1_codes) MOLR_TRY(s1_seal(const_cast<molr_cache*>(c), s));
      MOLR_TRY(scan_scores(ctx, mode, m, c->d1, c->s1_f32, c->s1_codes, s1_interleaved(c->d1), c->s1_inv, c->s1_scales,
                           loc.as<int64_t>(), B, q.as<float>(), qc.as<int8_t>(), ss.p, m, s));
    }
    MOLR_TRY(nth_largest_rows(ctx, B, m, ss.p, mode == MOLR_S1_INT8_RAW, m, nullptr, 0, nk, tk.as<uint32_t>(), s));
  }
  top_keys_kernel<<<B, 256, 0, s>>>(m, ss.p, mode == MOLR_S1_INT8_RAW, tk.as<uint32_t>(), nk, n_keep, ok.as<uint32_t>());
  MOLR_LAUNCHED(ctx);
  MOLR_CUDA(cudaStreamSynchronize(s));
  return finish_outputs(s, {&ok});
}

int molr_select_nth_keys(molr_ctx* ctx, int B, int64_t m, const uint32_t* keys, int64_t n, uint32_t* out_keys,
                         void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (n < 1 || n > m) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n=%lld outside [1, %lld]", (long long)n, (long long)m);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  WorkspaceScope ws(ctx, s);
  In ik;
  MOLR_TRY(ik.stage(keys, size_t(B) * m * 4, s));
  Out ok;
  MOLR_TRY(ok.stage(out_keys, size_t(B) * 4, s));
  Scratch counts;
  MOLR_TRY(counts.alloc(size_t(B) * 8, s));
  fill_i64_kernel<<<div_up(B, 256), 256, 0, s>>>(B, m, counts.as<int64_t>());
  MOLR_LAUNCHED(ctx);
  MOLR_TRY(nth_largest_keys(ctx, B, m, ik.as<uint32_t>(), counts.as<int64_t>(), n, ok.as<uint32_t>(), nullptr, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  return finish_outputs(s, {&ok});
}

}  // extern "C"
