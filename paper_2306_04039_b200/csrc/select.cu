// Selection kernels: radix select (nth_largest, hindexer.py:77-82), segmented exact top-k by
// (score desc, id asc) (mol_top_k's lexsort, mol.py:401-408; exact_top_k, hindexer.py:166-178)
// and the rank-merge of per-shard top-k lists (multi-GPU C1).
#include <algorithm>

#include "kernels.cuh"

namespace molr {

constexpr int kSelThreads = 1024;
constexpr int kSortCap = 4096;  // composite keys sorted in shared memory

// Warp-aggregated shared-memory histogram increment.
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin, bool active) {
  unsigned mask = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  unsigned peers = __match_any_sync(mask, bin);
  int leader = __ffs(peers) - 1;
  if ((threadIdx.x & 31) == leader) atomicAdd(&hist[bin], __popc(peers));
}

// Block-wide radix select over n unsigned keys (uint32 or uint64, ascending).  Returns the
// rank-th smallest key (rank 1-indexed) and the number of keys strictly smaller.  All threads
// must call.  key_of(i, &k) returns false for elements that do not take part.
template <class K, class KeyFn>
__device__ void block_radix_select(KeyFn key_of, int64_t n, int64_t rank, uint32_t* hist, K* out_key,
                                   int64_t* out_less) {
  __shared__ unsigned long long s_prefix;
  __shared__ int64_t s_rank, s_less;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_rank = rank;
    s_less = 0;
  }
  constexpr int kTop = int(sizeof(K)) * 8 - 8;
  for (int shift = kTop; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const K prefix = (K)s_prefix;
    const K hmask = shift == kTop ? K(0) : (~K(0) << (shift + 8));
    // strided loop padded so every lane of a warp takes part in the ballot
    const int64_t n_pad = (n + 31) / 32 * 32;
    for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x) {
      K k = 0;
      bool act = false;
      if (i < n && key_of(i, &k)) act = (k & hmask) == prefix;
      hist_add(hist, uint32_t(k >> shift) & 255u, act);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp scan over 256 bins: lane owns bins [8*lane, 8*lane+8)
      uint32_t c[8];
      uint32_t tot = 0;
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[threadIdx.x * 8 + j];
        tot += c[j];
      }
      uint32_t incl = tot;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)threadIdx.x >= o) incl += v;
      }
      uint32_t excl = incl - tot;
      int64_t r = s_rank;
      __syncwarp();  // every lane has read s_rank before the owning lane rewrites it
      if ((int64_t)excl < r && r <= (int64_t)incl) {  // the lane whose range contains rank
        uint32_t run = excl;
        for (int j = 0; j < 8; ++j) {
          if ((int64_t)(run + c[j]) >= r) {
            s_prefix = (unsigned long long)(prefix | (K(threadIdx.x * 8 + j) << shift));
            s_rank = r - run;
            s_less += run;
            break;
          }
          run += c[j];
        }
      }
    }
    __syncthreads();
  }
  *out_key = (K)s_prefix;
  *out_less = s_less;
  __syncthreads();
}

// In-place ascending bitonic sort of n (power of two) uint64 in shared or global memory.
__device__ void block_bitonic_sort(uint64_t* a, int64_t n) {
  for (int64_t size = 2; size <= n; size <<= 1) {
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int64_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
        int64_t lo = 2 * i - (i & (stride - 1));
        int64_t hi = lo + stride;
        bool up = ((lo & size) == 0);
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == up) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncthreads();
    }
  }
}

__host__ __device__ inline int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// desc-key: ascending order of desc_key(score) == descending score.
__device__ __forceinline__ uint32_t desc_key(float s) { return ~f32_key(s); }

// Segmented top-k: one CTA per query.  Two radix selects make the selected set exact:
// K* = k-th smallest desc-key, then among keys == K* the (k - less)-th smallest id I*.
// Selected = {key < K*} U {key == K*, id <= I*}, sorted by (key, id) — np.lexsort((ids, -s)).
template <class Id>
__global__ void __launch_bounds__(kSelThreads)
segmented_topk_kernel(int B, const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                      const Id* __restrict__ ids, int64_t X, const float* __restrict__ scores, int64_t dense_ld,
                      int k, int64_t id_offset, uint64_t* __restrict__ spill, int64_t spill_ld,
                      int64_t* __restrict__ out_ids, float* __restrict__ out_scores, int P) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t buf[kSortCap];
  __shared__ int s_count;
  // P > 1 (small batches): P CTAs per query, CTA p takes slice p of the segment and writes its
  // top-k as list p of a rank-major (P, B, k) array for merge_topk_kernel
  const int b = blockIdx.x / P, part = blockIdx.x % P;
  int64_t seg0 = begin ? begin[b] : 0;
  int64_t n = begin ? end[b] - begin[b] : X;
  const int64_t sub0 = n * part / P, sub1 = n * (part + 1) / P;
  const float* sc = begin ? scores + seg0 + sub0 : scores + int64_t(b) * dense_ld + sub0;
  const Id* id = ids ? ids + seg0 + sub0 : nullptr;
  const uint32_t id_base = ids ? 0u : uint32_t(sub0);
  n = sub1 - sub0;
  if (P > 1) {
    out_ids += int64_t(part) * B * k;
    out_scores += int64_t(part) * B * k;
  }
  const int kk = (int)imin64(k, n);
  // a segment shorter than k: the tail is "no entry" (id -1, score -inf; merge_topk drops it)
  for (int i = max(kk, 0) + threadIdx.x; i < k; i += blockDim.x) {
    out_ids[int64_t(b) * k + i] = -1;
    out_scores[int64_t(b) * k + i] = -INFINITY;
  }
  if (kk <= 0) return;
  auto idof = [&](int64_t i) -> uint32_t { return id ? (uint32_t)id[i] : id_base + (uint32_t)i; };
  // ---- fast path: sampled bound + one filtering pass ----------------------------------------
  // bound = the r-th largest of every 16th score, r ~ 4 sigma above the expected number of
  // samples beating the k-th largest, so bound <= k-th largest with overwhelming probability.
  // Every score >= bound is gathered (with its id) and sorted; when at least kk passed, the
  // k-th largest is >= bound, so the passers contain the exact top-k including its ties.
  // Otherwise (or on overflow of the smem buffer) the two-radix-select path below runs.
  if (n >= int64_t(32) * kk && kk <= 512) {
    constexpr int kStride = 16;
    const int64_t ns = n / kStride;
    const double mu = double(kk) / kStride;
    const int64_t r = imin64(ns, int64_t(mu + 4.0 * sqrt(mu) + 3.0));
    uint32_t bkey;
    int64_t bless;
    block_radix_select<uint32_t>([&](int64_t i, uint32_t* kk2) { *kk2 = desc_key(sc[i * kStride]); return true; }, ns, r,
                                 hist, &bkey, &bless);
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const int64_t n_pad = (n + 31) / 32 * 32;
    for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x) {
      uint32_t key = 0;
      bool take = false;
      if (i < n) {
        key = desc_key(sc[i]);
        take = key <= bkey;  // score >= bound
      }
      unsigned bal = __ballot_sync(0xffffffffu, take);
      int base = 0;
      if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&s_count, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int pos = base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1));
      if (take && pos < kSortCap) buf[pos] = (uint64_t(key) << 32) | idof(i);
    }
    __syncthreads();
    const int cnt = s_count;
    if (cnt >= kk && cnt <= kSortCap) {
      const int64_t m2 = next_pow2(cnt);
      for (int64_t i = cnt + threadIdx.x; i < m2; i += blockDim.x) buf[i] = ~0ull;
      __syncthreads();
      block_bitonic_sort(buf, m2);
      for (int i = threadIdx.x; i < kk; i += blockDim.x) {
        const uint64_t v = buf[i];
        out_ids[int64_t(b) * k + i] = int64_t(uint32_t(v)) + id_offset;
        out_scores[int64_t(b) * k + i] = key_f32(~uint32_t(v >> 32));
      }
      return;  // uniform: every thread read the same s_count
    }
    __syncthreads();
  }
  uint32_t kstar, istar;
  int64_t less, less2;
  block_radix_select<uint32_t>([&](int64_t i, uint32_t* kk2) { *kk2 = desc_key(sc[i]); return true; }, n, kk,
                               hist, &kstar, &less);
  block_radix_select<uint32_t>(
      [&](int64_t i, uint32_t* kk2) {
        if (desc_key(sc[i]) != kstar) return false;
        *kk2 = idof(i);
        return true;
      },
      n, kk - less, hist, &istar, &less2);
  const int64_t m2 = next_pow2(kk);
  uint64_t* arr = (m2 <= kSortCap) ? buf : spill + int64_t(b) * spill_ld;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  const int64_t n_pad = (n + 31) / 32 * 32;
  for (int64_t i = threadIdx.x; i < n_pad; i += blockDim.x) {
    uint32_t key = 0, iid = 0;
    bool take = false;
    if (i < n) {
      key = desc_key(sc[i]);
      iid = idof(i);
      take = key < kstar || (key == kstar && iid <= istar);
    }
    unsigned bal = __ballot_sync(0xffffffffu, take);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && bal) base = atomicAdd(&s_count, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    int pos = base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1));
    if (take && pos < m2) arr[pos] = (uint64_t(key) << 32) | iid;  // duplicate ids may exceed kk
  }
  __syncthreads();
  const int64_t m = imin64(s_count, m2);
  for (int64_t i = m + threadIdx.x; i < m2; i += blockDim.x) arr[i] = ~0ull;
  __syncthreads();
  block_bitonic_sort(arr, m2);
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    uint64_t v = arr[i];
    out_ids[int64_t(b) * k + i] = int64_t(uint32_t(v)) + id_offset;
    out_scores[int64_t(b) * k + i] = key_f32(~uint32_t(v >> 32));
  }
}

__global__ void merge_topk_kernel(int P, int B, int k_in, const int64_t* __restrict__ ids, const float* __restrict__ sc,
                                  int k, int64_t* __restrict__ out_ids, float* __restrict__ out_sc);

template <class Id>
int segmented_top_k(molr_ctx* ctx, int B, Segs<Id> segs, const float* scores, int64_t dense_ld, int k,
                    int64_t id_offset, int64_t* out_ids, float* out_scores, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  Scratch spill;
  int64_t spill_ld = 0;
  if (next_pow2(k) > kSortCap) {  // large k: sort in global scratch
    spill_ld = next_pow2(k);
    MOLR_TRY(spill.alloc(size_t(B) * spill_ld * 8, s));
  }
  // small batches: one CTA per query leaves the GPU idle while it walks ~K' scores; split each
  // query over P CTAs (slices), then merge the P top-k lists (exact: the top-k of a union of the
  // slices' top-k lists under the same (score desc, id asc) order is the top-k of the whole).
  // At most 8 slices: each stays long enough for the sampled-bound fast path (n >= 32 k)
  const int P = (spill_ld == 0 && 4 * B <= ctx->num_sms)
                    ? std::max(1, std::min(std::min(ctx->num_sms / B, 8), int(kSortCap / std::max(k, 1))))
                    : 1;
  if (P > 1) {
    Scratch pi, ps;
    MOLR_TRY(pi.alloc(size_t(P) * B * k * 8, s));
    MOLR_TRY(ps.alloc(size_t(P) * B * k * 4, s));
    segmented_topk_kernel<Id><<<B * P, kSelThreads, 0, s>>>(B, segs.begin, segs.end, segs.ids, segs.X, scores,
                                                            dense_ld, k, id_offset, nullptr, 0, pi.as<int64_t>(),
                                                            ps.as<float>(), P);
    MOLR_LAUNCHED(ctx);
    merge_topk_kernel<<<B, 256, 0, s>>>(P, B, k, pi.as<int64_t>(), ps.as<float>(), k, out_ids, out_scores);
    MOLR_LAUNCHED(ctx);
    return MOLR_OK;
  }
  segmented_topk_kernel<Id><<<B, kSelThreads, 0, s>>>(B, segs.begin, segs.end, segs.ids, segs.X, scores,
                                                      dense_ld, k, id_offset, spill.as<uint64_t>(), spill_ld,
                                                      out_ids, out_scores, 1);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

template int segmented_top_k<int64_t>(molr_ctx*, int, Segs<int64_t>, const float*, int64_t, int, int64_t,
                                      int64_t*, float*, cudaStream_t);
template int segmented_top_k<int32_t>(molr_ctx*, int, Segs<int32_t>, const float*, int64_t, int, int64_t,
                                      int64_t*, float*, cudaStream_t);

__device__ __forceinline__ uint64_t f64_key(double f) {
  uint64_t u = __double_as_longlong(f);
  if (u == 0x8000000000000000ull) u = 0ull;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(uint64_t k) {
  uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(u);
}

// nth_largest over B rows: value keys (f32 / i32 / f64 / i64), optional gather through sample
// indices.  Writes the ascending-order key of the n-th largest value.
// DT: 0 f32, 1 i32, 2 f64, 3 i64, 4 pre-computed ascending uint32 keys (f32_key / i32_key).
// row_n (optional): row b holds only min(row_n[b], n) values; a row with fewer than rank_n values
// sets *short_rows and writes no key.
template <class K, int DT>
__global__ void __launch_bounds__(kSelThreads)
nth_largest_kernel(int64_t n, const void* __restrict__ values, int64_t ld, const int64_t* __restrict__ gather,
                   int64_t gather_ld, int64_t rank_n, K* __restrict__ out_keys, const int64_t* __restrict__ row_n,
                   int* __restrict__ short_rows) {
  __shared__ uint32_t hist[256];
  const int b = blockIdx.x;
  const int64_t nb = row_n ? imin64(row_n[b], n) : n;
  if (nb < rank_n) {
    if (threadIdx.x == 0 && short_rows) atomicOr(short_rows, 1);
    return;
  }
  const int64_t* gi = gather ? gather + int64_t(b) * gather_ld : nullptr;
  auto key_of = [&](int64_t i, K* k) -> bool {
    int64_t j = int64_t(b) * ld + (gi ? gi[i] : i);
    K v;
    if (DT == 0) v = (K)f32_key(reinterpret_cast<const float*>(values)[j]);
    else if (DT == 1) v = (K)i32_key(reinterpret_cast<const int32_t*>(values)[j]);
    else if (DT == 2) v = (K)f64_key(reinterpret_cast<const double*>(values)[j]);
    else if (DT == 4) v = (K)reinterpret_cast<const uint32_t*>(values)[j];
    else v = (K)(uint64_t(reinterpret_cast<const int64_t*>(values)[j]) ^ 0x8000000000000000ull);
    *k = ~v;
    return true;
  };
  K kstar;
  int64_t less;
  block_radix_select<K>(key_of, nb, rank_n, hist, &kstar, &less);
  if (threadIdx.x == 0) out_keys[b] = ~kstar;
}

int nth_largest_rows(molr_ctx* ctx, int B, int64_t n_values, const void* values, int is_int, int64_t ld,
                     const int64_t* gather, int64_t gather_ld, int64_t n, uint32_t* out_keys, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  if (is_int) nth_largest_kernel<uint32_t, 1><<<B, kSelThreads, 0, s>>>(n_values, values, ld, gather, gather_ld, n, out_keys, nullptr, nullptr);
  else nth_largest_kernel<uint32_t, 0><<<B, kSelThreads, 0, s>>>(n_values, values, ld, gather, gather_ld, n, out_keys, nullptr, nullptr);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

int nth_largest_keys(molr_ctx* ctx, int B, int64_t cap, const uint32_t* keys, const int64_t* counts, int64_t n,
                     uint32_t* out_keys, int* short_rows, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  nth_largest_kernel<uint32_t, 4><<<B, kSelThreads, 0, s>>>(cap, keys, cap, nullptr, 0, n, out_keys, counts, short_rows);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

// Merge P rank-major lists (P, B, k_in) into the top-k per query (multi-GPU C1).
__global__ void __launch_bounds__(256)
merge_topk_kernel(int P, int B, int k_in, const int64_t* __restrict__ ids, const float* __restrict__ sc, int k,
                  int64_t* __restrict__ out_ids, float* __restrict__ out_sc) {
  __shared__ uint64_t buf[kSortCap];
  const int b = blockIdx.x;
  const int m = P * k_in;
  const int m2 = (int)next_pow2(m);
  for (int i = threadIdx.x; i < m2; i += blockDim.x) {
    uint64_t v = ~0ull;
    if (i < m) {
      int p = i / k_in, j = i % k_in;
      int64_t src = (int64_t(p) * B + b) * k_in + j;
      int64_t id = ids[src];
      if (id >= 0) v = (uint64_t(desc_key(sc[src])) << 32) | uint64_t(uint32_t(id));
    }
    buf[i] = v;
  }
  __syncthreads();
  block_bitonic_sort(buf, m2);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    uint64_t v = buf[i];
    out_ids[int64_t(b) * k + i] = v == ~0ull ? -1 : int64_t(uint32_t(v));
    out_sc[int64_t(b) * k + i] = v == ~0ull ? -INFINITY : key_f32(~uint32_t(v >> 32));
  }
}

}  // namespace molr

using namespace molr;

extern "C" {

int molr_nth_largest(molr_ctx* ctx, int B, int64_t n_values, const void* values, int dtype, int64_t n,
                     double* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (n < 1 || n > n_values) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n=%lld outside [1, %lld]", (long long)n,
                                       (long long)n_values);
  if (dtype < 0 || dtype > 3) MOLR_FAIL(MOLR_ERR_INVALID, "dtype code %d", dtype);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  const size_t esz = dtype < 2 ? 4 : 8;
  In v;
  MOLR_TRY(v.stage(values, size_t(B) * n_values * esz, s));
  Scratch keys;
  MOLR_TRY(keys.alloc(size_t(B) * 8, s));
  uint64_t* k64 = keys.as<uint64_t>();
  uint32_t* k32 = keys.as<uint32_t>();
  switch (dtype) {
    case 0: nth_largest_kernel<uint32_t, 0><<<B, kSelThreads, 0, s>>>(n_values, v.dptr, n_values, nullptr, 0, n, k32, nullptr, nullptr); break;
    case 1: nth_largest_kernel<uint32_t, 1><<<B, kSelThreads, 0, s>>>(n_values, v.dptr, n_values, nullptr, 0, n, k32, nullptr, nullptr); break;
    case 2: nth_largest_kernel<uint64_t, 2><<<B, kSelThreads, 0, s>>>(n_values, v.dptr, n_values, nullptr, 0, n, k64, nullptr, nullptr); break;
    default: nth_largest_kernel<uint64_t, 3><<<B, kSelThreads, 0, s>>>(n_values, v.dptr, n_values, nullptr, 0, n, k64, nullptr, nullptr); break;
  }
  MOLR_LAUNCHED(ctx);
  std::vector<uint64_t> hk(B);
  MOLR_CUDA(cudaMemcpyAsync(hk.data(), keys.p, size_t(B) * esz, cudaMemcpyDeviceToHost, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) {
    if (dtype == 0) out[b] = double(key_f32(reinterpret_cast<uint32_t*>(hk.data())[b]));
    else if (dtype == 1) out[b] = double(key_i32(reinterpret_cast<uint32_t*>(hk.data())[b]));
    else if (dtype == 2) {
      uint64_t k = hk[b];
      uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
      double d;
      memcpy(&d, &u, 8);
      out[b] = d;
    } else out[b] = double(int64_t(hk[b] ^ 0x8000000000000000ull));
  }
  return MOLR_OK;
}

int molr_merge_top_k(molr_ctx* ctx, int P, int B, int k_in, const int64_t* ids, const float* scores, int k,
                     int64_t* out_ids, float* out_scores, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (P < 1 || B < 0 || k_in < 1 || k < 1 || k > P * k_in) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "bad merge sizes");
  if (int64_t(P) * k_in > kSortCap) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "P*k_in exceeds %d", kSortCap);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B == 0) return MOLR_OK;
  In a, b;
  Out oi, os;
  MOLR_TRY(a.stage(ids, size_t(P) * B * k_in * 8, s));
  MOLR_TRY(b.stage(scores, size_t(P) * B * k_in * 4, s));
  MOLR_TRY(oi.stage(out_ids, size_t(B) * k * 8, s));
  MOLR_TRY(os.stage(out_scores, size_t(B) * k * 4, s));
  merge_topk_kernel<<<B, 256, 0, s>>>(P, B, k_in, a.as<int64_t>(), b.as<float>(), k, oi.as<int64_t>(),
                                      os.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&oi, &os});
}

}  // extern "C"
