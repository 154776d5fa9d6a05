// C-ABI plumbing: contexts, the immutable device ItemCache (mol.py:216-291) and gating weights.
#include <mutex>
#include <vector>

#include "common.cuh"
#include "stage1.cuh"

namespace molr {
thread_local molr_arena* tl_arena = nullptr;

namespace {
struct ThreadStreams {
  std::vector<std::pair<const molr_ctx*, cudaStream_t>> v;
  ~ThreadStreams() {
    for (auto& e : v) cudaStreamDestroy(e.second);  // (errors at process teardown are moot)
  }
};
thread_local ThreadStreams tl_streams;
}  // namespace

cudaStream_t thread_stream(molr_ctx* ctx) {
  for (auto& e : tl_streams.v)
    if (e.first == ctx) return e.second;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return ctx->stream;
  }
  tl_streams.v.emplace_back(ctx, st);
  return st;
}

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int finish_outputs(cudaStream_t s, std::initializer_list<Out*> outs) {
  bool any_host = false;
  for (Out* o : outs) {
    if (!o) continue;
    MOLR_TRY(o->finish(s));
    any_host |= o->host();
  }
  if (any_host) MOLR_CUDA(cudaStreamSynchronize(s));
  return MOLR_OK;
}

// ---- storage conversion kernels ---------------------------------------------------------------
// bf16 storage of f32 values that must be exactly representable; bad |= any rounding.
__global__ void to_bf16_kernel(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ hi,
                               int* __restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int local_bad = 0;
  for (; i < n; i += stride) {
    float v = x[i];
    __nv_bfloat16 h = __float2bfloat16_rn(v);
    local_bad |= (__bfloat162float(h) != v);
    hi[i] = h;
  }
  if (local_bad) atomicOr(bad, 1);
}

// item components -> bf16 in the cache layout (swizzled when emb_swizzled); bad |= rounding.
__global__ void embs_to_bf16_kernel(const float* __restrict__ x, int64_t rows, int k_x, int d,
                                    __nv_bfloat16* __restrict__ out, int* __restrict__ bad) {
  const int64_t ne = int64_t(k_x) * d;
  const bool swz = emb_swizzled(k_x, d);
  int local_bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ne; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / ne;
    int e = int(i % ne), b = e / d, k = e % d;
    float v = x[i];
    __nv_bfloat16 h = __float2bfloat16_rn(v);
    local_bad |= (__bfloat162float(h) != v);
    out[r * ne + emb_offset(b, k, d, swz)] = h;
  }
  if (local_bad) atomicOr(bad, 1);
}

// f32 item components -> bf16 hi + lo images in the cache's pre-swizzled layout (hi at row r,
// lo at row X + r): x = hi + lo to ~2^-17 relative
__global__ void embs_to_hilo_kernel(const float* __restrict__ x, int64_t rows, int64_t row0, int64_t X, int k_x, int d,
                                    __nv_bfloat16* __restrict__ hl) {
  const int64_t ne = int64_t(k_x) * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ne; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ne;
    const int e = int(i % ne), b = e / d, k = e % d;
    const float v = x[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const int64_t o = (row0 + r) * ne + emb_offset(b, k, d, true);
    hl[o] = h;
    hl[X * ne + o] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

int build_embs_hilo(molr_cache* c, int64_t row0, int64_t n, cudaStream_t s) {
  if (!c->embs_hl || n <= 0) return MOLR_OK;
  const int64_t ne = int64_t(c->k_x) * c->d;
  embs_to_hilo_kernel<<<c->ctx->num_sms * 8, 256, 0, s>>>(c->embs_f32 + row0 * ne, n, row0, c->X, c->k_x, c->d, c->embs_hl);
  MOLR_LAUNCHED(c->ctx);
  return MOLR_OK;
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = int32_t(i);
}

// Sort the stored rows by scale (ascending; padding rows, scale 0, last) inside windows of
// S1_SORT_WINDOW rows: the filter's per-32-row integer bound (from the chunk's scale range) is then
// nearly exact, so far fewer (query, 8-row group) blocks need the exact test (measured on the
// synthetic corpus: 12% -> 7% of warp groups vs 256-row windows).  The candidate ids of a window
// stay within its 4,096 items, so stage 2 keeps its locality.
constexpr int S1_SORT_WINDOW = 4096;

// keys of one window -> the window-local source row of every destination row
__global__ void __launch_bounds__(1024) window_sort_kernel(const float* __restrict__ scales, int64_t n_rows,
                                                           int32_t* __restrict__ src_local) {
  __shared__ uint64_t key[S1_SORT_WINDOW];
  const int64_t w0 = int64_t(blockIdx.x) * S1_SORT_WINDOW;
  const int n = int(imin64(S1_SORT_WINDOW, n_rows - w0));
  for (int i = threadIdx.x; i < S1_SORT_WINDOW; i += blockDim.x) {
    uint32_t k = 0xffffffffu;  // past the end: after everything
    if (i < n) {
      const float sc = scales[w0 + i];
      k = sc > 0.f ? __float_as_uint(sc) : 0xfffffffeu;  // positive floats order as uints; padding last
    }
    key[i] = (uint64_t(k) << 32) | uint32_t(i);
  }
  __syncthreads();
  for (int size = 2; size <= S1_SORT_WINDOW; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < S1_SORT_WINDOW / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t x = key[lo], y = key[hi];
        if ((x > y) == up) {
          key[lo] = y;
          key[hi] = x;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) src_local[w0 + i] = int32_t(key[i] & 0xffffffffu);
}

// rows [r0, r1) := old rows (w0 + src_local) of a copy of the slab starting at row s0
__global__ void window_gather_kernel(int64_t s0, int64_t r0, int64_t r1, const int32_t* __restrict__ src_local,
                                     const int8_t* __restrict__ old_codes, const float* __restrict__ old_scales,
                                     const int32_t* __restrict__ old_perm, int8_t* __restrict__ codes,
                                     float* __restrict__ scales, int32_t* __restrict__ perm) {
  for (int64_t i = r0 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1 * 4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> 2;
    const int c = int(i & 3);
    const int64_t src = r / S1_SORT_WINDOW * S1_SORT_WINDOW + src_local[r];
    *reinterpret_cast<int4*>(codes + s1_chunk_offset(r, c, 64)) =
        *reinterpret_cast<const int4*>(old_codes + s1_chunk_offset(src - s0, c, 64));
    if (c == 0) {
      scales[r] = old_scales[src - s0];
      perm[r] = old_perm[src - s0];
    }
  }
}

static int s1_window_sort(molr_cache* c, int64_t xr, cudaStream_t s) {
  const int64_t nwin = (xr + S1_SORT_WINDOW - 1) / S1_SORT_WINDOW;
  Scratch src;
  MOLR_TRY(src.alloc(size_t(xr) * 4, s));
  window_sort_kernel<<<(unsigned)nwin, 1024, 0, s>>>(c->s1_scales, xr, src.as<int32_t>());
  MOLR_LAUNCHED(c->ctx);
  // permute slab by slab through a bounded copy (whole windows; 2^24 rows = 1 GB of codes)
  const int64_t slab = std::min<int64_t>(xr, int64_t(1) << 24);
  Scratch oc, os_, op;
  MOLR_TRY(oc.alloc(size_t(slab) * 64, s));
  MOLR_TRY(os_.alloc(size_t(slab) * 4, s));
  MOLR_TRY(op.alloc(size_t(slab) * 4, s));
  for (int64_t s0 = 0; s0 < xr; s0 += slab) {
    const int64_t n = std::min<int64_t>(slab, xr - s0);
    // the interleaved layout is row-block linear, so a slab starting at a multiple of 8 rows is contiguous
    MOLR_CUDA(cudaMemcpyAsync(oc.p, c->s1_codes + s1_chunk_offset(s0, 0, 64), size_t(n) * 64, cudaMemcpyDeviceToDevice, s));
    MOLR_CUDA(cudaMemcpyAsync(os_.p, c->s1_scales + s0, size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
    MOLR_CUDA(cudaMemcpyAsync(op.p, c->s1_perm + s0, size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
    window_gather_kernel<<<div_up(n * 4, 256), 256, 0, s>>>(s0, s0, s0 + n, src.as<int32_t>(), oc.as<int8_t>(),
                                                             os_.as<float>(), op.as<int32_t>(), c->s1_codes,
                                                             c->s1_scales, c->s1_perm);
    MOLR_LAUNCHED(c->ctx);
  }
  return MOLR_OK;
}

__global__ void inv_perm_kernel(const int32_t* __restrict__ perm, int64_t n_rows, int64_t X, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = perm[i];
    if (r < X) inv[r] = int32_t(i);
  }
}

// Seal the int8 view of a cache: sort rows by scale within windows, rebuild inv and the chunk min/max.
// Idempotent and thread-safe; called by every stage-1 entry point before reading the view.
int s1_seal(molr_cache* c, cudaStream_t s) {
  if (!c->s1_perm || c->s1_sealed.load(std::memory_order_acquire)) return MOLR_OK;
  std::lock_guard<std::mutex> g(c->seal_mu);
  if (c->s1_sealed.load()) return MOLR_OK;
  const int64_t xr = s1_rows_alloc(c->X, c->d1);
  if (xr > 0) {
    MOLR_TRY(s1_window_sort(c, xr, s));
    inv_perm_kernel<<<div_up(xr, 256), 256, 0, s>>>(c->s1_perm, xr, c->X, c->s1_inv);
    MOLR_LAUNCHED(c->ctx);
    MOLR_TRY(s1_update_chunk_mm(c, 0, xr, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
  }
  c->s1_sealed.store(1, std::memory_order_release);
  return MOLR_OK;
}

// linear (m, 64) int8 rows -> interleaved cache layout starting at row r0
__global__ void codes_to_ilv_kernel(const int8_t* __restrict__ src, int64_t m, int64_t r0, int8_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * 4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> 2;
    const int c = int(i & 3);
    *reinterpret_cast<int4*>(dst + s1_chunk_offset(r0 + r, c, 64)) = *reinterpret_cast<const int4*>(src + r * 64 + c * 16);
  }
}

__global__ void chunk_mm_kernel(const float* __restrict__ scales, int64_t c0, int64_t c1, float2* __restrict__ mm) {
  for (int64_t c = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < c1; c += (int64_t)gridDim.x * blockDim.x) {
    float lo = INFINITY, hi = 0.f;
    for (int j = 0; j < 32; ++j) {
      const float v = scales[c * 32 + j];
      if (v > 0.f) {  // padding rows have scale 0 and are never scored
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
      }
    }
    // stored as reciprocals (1/min, 1/max) for the filter's integer bound; (0, -1) marks a chunk
    // of padding rows only
    mm[c] = hi > 0.f ? make_float2(float(1.0 / double(lo)), float(1.0 / double(hi))) : make_float2(0.f, -1.f);
  }
}

// 2-D tensor map viewing `rows` x 1 KB as uint32 [rows][256], box = one row (for tile::gather4)
int encode_rows_tmap(CUtensorMap* tm, const void* base, int64_t rows) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn enc = [] {
    EncodeFn f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return f;
  }();
  if (!enc) return 0;
  cuuint64_t dims[2] = {256, (cuuint64_t)rows};
  cuuint64_t strides[1] = {1024};
  cuuint32_t box[2] = {256, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int chunk_minmax(molr_ctx* ctx, const float* scales, int64_t c0, int64_t c1, float2* mm, cudaStream_t s) {
  if (c1 <= c0) return MOLR_OK;
  chunk_mm_kernel<<<div_up(c1 - c0, 256), 256, 0, s>>>(scales, c0, c1, mm);
  MOLR_LAUNCHED(ctx);
  return MOLR_OK;
}

int s1_update_chunk_mm(molr_cache* c, int64_t row0, int64_t n, cudaStream_t s) {
  const int64_t c0 = row0 / 32, c1 = (row0 + n + 31) / 32;
  if (c1 <= c0) return MOLR_OK;
  chunk_mm_kernel<<<div_up(c1 - c0, 256), 256, 0, s>>>(c->s1_scales, c0, c1, c->s1_chunk_mm);
  MOLR_LAUNCHED(c->ctx);
  return MOLR_OK;
}

}  // namespace molr

using namespace molr;

extern "C" {

const char* molr_last_error(void) { return g_last_error.c_str(); }
const char* molr_version(void) { return "molr_b200 0.1 (sm_100a)"; }

int molr_ctx_create(int device, molr_ctx** out) {
  if (!out) MOLR_FAIL(MOLR_ERR_INVALID, "out is null");
  MOLR_CUDA(cudaSetDevice(device));
  auto* c = new molr_ctx();
  c->device = device;
  cudaDeviceProp prop;
  MOLR_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    delete c;
    MOLR_FAIL(MOLR_ERR_CUDA, "device %d is sm_%d%d; libmolr_b200 is built for sm_100a only", device,
              prop.major, prop.minor);
  }
  c->num_sms = prop.multiProcessorCount;
  MOLR_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  // keep freed scratch cached in the pool (stream-ordered allocator)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return MOLR_OK;
}

int molr_ctx_destroy(molr_ctx* ctx) {
  if (!ctx) return MOLR_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (molr_arena* a : ctx->ws_all) {
    if (a->base) cudaFree(a->base);
    delete a;
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return MOLR_OK;
}

int molr_ctx_sync(molr_ctx* ctx, void* stream) {
  MOLR_CUDA(cudaStreamSynchronize(pick_stream(ctx, stream)));
  return MOLR_OK;
}

int64_t molr_ctx_launch_count(molr_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

// ---- cache ----------------------------------------------------------------------------------
int molr_cache_alloc(molr_ctx* ctx, int64_t X, int k_x, int d, int G, int d1, int storage,
                     molr_cache** out) {
  if (!ctx || !out) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  if (X < 0 || X >= (int64_t(1) << 31)) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n_items %lld", (long long)X);
  if (k_x < 1 || d < 1 || G < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad cache dims");
  if ((storage & (MOLR_STORE_S1_F32 | MOLR_STORE_S1_INT8)) && d1 < 1)
    MOLR_FAIL(MOLR_ERR_DIMENSION, "stage-1 dim");
  if ((storage & MOLR_STORE_S1_INT8) && d1 > 131070)
    MOLR_FAIL(MOLR_ERR_LENGTH_OVERFLOW, "row length %d exceeds int32-safe bound 131070", d1);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  auto* c = new molr_cache();
  c->ctx = ctx;
  c->X = X;
  c->k_x = k_x;
  c->d = d;
  c->G = G;
  c->d1 = d1;
  c->storage = storage;
  auto grab = [&](void** p, size_t bytes) -> int {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
      set_error(std::string("cudaMalloc cache: ") + cudaGetErrorString(e));
      return MOLR_ERR_CUDA;
    }
    c->bytes += bytes;
    return MOLR_OK;
  };
  size_t ne = size_t(X) * k_x * d;
  int st = (storage & MOLR_STORE_EMBS_F32) ? grab((void**)&c->embs_f32, ne * 4) : grab((void**)&c->embs_bf16, ne * 2);
  if (!st && c->embs_bf16 && k_x * d == 512 && X > 0) c->embs_tmap_ok = encode_rows_tmap(&c->embs_tmap, c->embs_bf16, X);
  if (!st && c->embs_f32 && k_x == 8 && d == 64 && X > 0) {  // hi + lo image for the tensor-core scorer
    st = grab((void**)&c->embs_hl, ne * 4);
    if (!st)
      c->embs_hl_tmap_ok = encode_rows_tmap(&c->embs_hi_tmap, c->embs_hl, X) &&
                           encode_rows_tmap(&c->embs_lo_tmap, c->embs_hl + ne, X);
  }
  if (!st && (storage & MOLR_STORE_GP_F32)) st = grab((void**)&c->gp_f32, size_t(X) * G * 4);
  if (!st && !(storage & MOLR_STORE_GP_F32)) st = grab((void**)&c->gp_bf16, size_t(X) * G * 2);
  if (!st && (storage & MOLR_STORE_S1_F32)) st = grab((void**)&c->s1_f32, size_t(X) * d1 * 4);
  const int64_t xr = s1_rows_alloc(X, d1);
  if (!st && (storage & MOLR_STORE_S1_INT8)) st = grab((void**)&c->s1_codes, size_t(xr) * d1);
  if (!st && (storage & MOLR_STORE_S1_INT8)) st = grab((void**)&c->s1_scales, size_t(xr) * 4);
  if (!st && (storage & MOLR_STORE_S1_INT8) && s1_interleaved(d1)) {
    st = grab((void**)&c->s1_chunk_mm, size_t(xr / 32) * sizeof(float2));
    if (!st) st = grab((void**)&c->s1_perm, size_t(xr) * 4);
    if (!st) st = grab((void**)&c->s1_inv, size_t(xr) * 4);
    if (!st && xr > 0) {
      iota_kernel<<<div_up(xr, 256), 256>>>(c->s1_perm, xr);
      iota_kernel<<<div_up(xr, 256), 256>>>(c->s1_inv, xr);
      if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = MOLR_ERR_CUDA;
    }
  }
  if (!st && (storage & MOLR_STORE_S1_INT8)) {  // zero the padding rows
    if (cudaMemset(c->s1_codes, 0, size_t(xr) * d1) != cudaSuccess || cudaMemset(c->s1_scales, 0, size_t(xr) * 4) != cudaSuccess)
      st = MOLR_ERR_CUDA;
  }
  if (st) {
    molr_cache_destroy(c);
    return st;
  }
  *out = c;
  return MOLR_OK;
}

int molr_cache_fill(molr_cache* c, int64_t row0, int64_t n, const float* embs, const float* gp,
                    const float* s1, const int8_t* codes, const float* scales, void* stream) {
  if (!c) MOLR_FAIL(MOLR_ERR_INVALID, "null cache");
  if (row0 < 0 || n < 0 || row0 + n > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "fill rows out of range");
  if (n == 0) return MOLR_OK;
  if (c->s1_sealed.load() && (codes || scales))
    MOLR_FAIL(MOLR_ERR_INVALID, "stage-1 view is sealed (the cache is immutable once queried)");
  molr_ctx* ctx = c->ctx;
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  Scratch bad;
  MOLR_TRY(bad.alloc(4, s));
  MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  const int64_t per_row = int64_t(c->k_x) * c->d;
  // chunk so staging of host f32 stays bounded (<= 256 MB per chunk)
  int64_t chunk = std::max<int64_t>(1, (int64_t(64) << 20) / std::max<int64_t>(per_row, c->G));
  for (int64_t r = 0; r < n; r += chunk) {
    int64_t m = std::min(chunk, n - r);
    if (embs) {
      size_t off = size_t(row0 + r) * per_row;
      if (c->embs_f32) {
        MOLR_CUDA(cudaMemcpyAsync(c->embs_f32 + off, embs + r * per_row, size_t(m * per_row) * 4, cudaMemcpyDefault, s));
        MOLR_TRY(build_embs_hilo(c, row0 + r, m, s));
      } else {
        In e;
        MOLR_TRY(e.stage(embs + r * per_row, size_t(m * per_row) * 4, s));
        embs_to_bf16_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(e.as<float>(), m, c->k_x, c->d, c->embs_bf16 + off,
                                                             bad.as<int>());
        MOLR_LAUNCHED(ctx);
      }
    }
    if (gp) {
      size_t off = size_t(row0 + r) * c->G;
      if (c->gp_f32) {
        MOLR_CUDA(cudaMemcpyAsync(c->gp_f32 + off, gp + r * c->G, size_t(m) * c->G * 4, cudaMemcpyDefault, s));
      } else {
        In e;
        MOLR_TRY(e.stage(gp + r * c->G, size_t(m) * c->G * 4, s));
        to_bf16_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(e.as<float>(), m * c->G, c->gp_bf16 + off, bad.as<int>());
        MOLR_LAUNCHED(ctx);
      }
    }
    if (s1 && c->s1_f32) {
      MOLR_CUDA(cudaMemcpyAsync(c->s1_f32 + size_t(row0 + r) * c->d1, s1 + r * c->d1,
                                size_t(m) * c->d1 * 4, cudaMemcpyDefault, s));
      c->s1_bf_ready.store(0, std::memory_order_release);  // the bf16 image is rebuilt on next use
    }
    if (codes && c->s1_codes) {
      if (s1_interleaved(c->d1)) {
        In e;
        MOLR_TRY(e.stage(codes + r * c->d1, size_t(m) * c->d1, s));
        codes_to_ilv_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(e.as<int8_t>(), m, row0 + r, c->s1_codes);
        MOLR_LAUNCHED(ctx);
      } else {
        MOLR_CUDA(cudaMemcpyAsync(c->s1_codes + size_t(row0 + r) * c->d1, codes + r * c->d1, size_t(m) * c->d1,
                                  cudaMemcpyDefault, s));
      }
    }
    if (scales && c->s1_scales)
      MOLR_CUDA(cudaMemcpyAsync(c->s1_scales + row0 + r, scales + r, size_t(m) * 4, cudaMemcpyDefault, s));
  }
  if (scales && c->s1_chunk_mm) MOLR_TRY(s1_update_chunk_mm(c, row0, n, s));
  int hbad = 0;
  MOLR_CUDA(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  if (hbad) MOLR_FAIL(MOLR_ERR_INVALID, "values not representable in the cache's bf16 storage");
  return MOLR_OK;
}

// Storage probe: which fields are exactly bf16-representable.
namespace molr {
__global__ void bf16_exact_kernel(const float* __restrict__ x, int64_t n, int* __restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int b = 0;
  for (; i < n; i += stride) b |= (__float_as_uint(x[i]) & 0xffffu) != 0u;
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
static int probe_bf16(molr_ctx* ctx, const float* x, int64_t n, cudaStream_t s, bool* exact) {
  Scratch bad;
  MOLR_TRY(bad.alloc(4, s));
  MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  int64_t chunk = int64_t(64) << 20;
  for (int64_t r = 0; r < n; r += chunk) {
    int64_t m = std::min(chunk, n - r);
    In e;
    MOLR_TRY(e.stage(x + r, size_t(m) * 4, s));
    bf16_exact_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(e.as<float>(), m, bad.as<int>());
    MOLR_LAUNCHED(ctx);
  }
  int h = 0;
  MOLR_CUDA(cudaMemcpyAsync(&h, bad.p, 4, cudaMemcpyDeviceToHost, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  *exact = (h == 0);
  return MOLR_OK;
}
}  // namespace molr

int molr_cache_create(molr_ctx* ctx, int64_t X, int k_x, int d, int G, const float* embs,
                      const float* gp, int d1, const float* s1, const int8_t* codes,
                      const float* scales, molr_cache** out) {
  if (!ctx || !out || !embs || !gp) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, nullptr);
  bool e_exact = false, g_exact = false;
  MOLR_TRY(probe_bf16(ctx, embs, X * k_x * d, s, &e_exact));
  MOLR_TRY(probe_bf16(ctx, gp, X * G, s, &g_exact));
  int storage = (e_exact ? 0 : MOLR_STORE_EMBS_F32) | (g_exact ? 0 : MOLR_STORE_GP_F32) |
                (s1 ? MOLR_STORE_S1_F32 : 0) | ((codes && scales) ? MOLR_STORE_S1_INT8 : 0);
  molr_cache* c = nullptr;
  MOLR_TRY(molr_cache_alloc(ctx, X, k_x, d, G, d1, storage, &c));
  int st = molr_cache_fill(c, 0, X, embs, gp, s1, codes, scales, nullptr);
  if (st) {
    molr_cache_destroy(c);
    return st;
  }
  *out = c;
  return MOLR_OK;
}

int molr_cache_destroy(molr_cache* c) {
  if (!c) return MOLR_OK;
  cudaSetDevice(c->ctx->device);
  cudaFree(c->embs_bf16);
  cudaFree(c->embs_f32);
  cudaFree(c->embs_hl);
  cudaFree(c->gp_bf16);
  cudaFree(c->gp_f32);
  cudaFree(c->s1_f32);
  cudaFree(c->s1_codes);
  cudaFree(c->s1_scales);
  cudaFree(c->s1_chunk_mm);
  cudaFree(c->s1_perm);
  cudaFree(c->s1_inv);
  cudaFree(c->s1_bf);
  cudaFree(c->s1_bnorm);
  cudaFree(c->s1_bnmax);
  delete c;
  return MOLR_OK;
}

int molr_cache_info(const molr_cache* c, int64_t* X, int* storage, int64_t* bytes) {
  if (!c) MOLR_FAIL(MOLR_ERR_INVALID, "null cache");
  if (X) *X = c->X;
  if (storage) *storage = c->storage;
  if (bytes) *bytes = c->bytes;
  return MOLR_OK;
}

// ---- gating ---------------------------------------------------------------------------------
int molr_gating_tc_prepare(molr_gating* g);  // mol_tc.cu

int molr_gating_create(molr_ctx* ctx, int G, int H, const float* w1, const float* b1, const float* w2,
                       int d_u, int H_u, const float* uw1, const float* ub1, const float* uw2,
                       molr_gating** out) {
  if (!ctx || !out || !w1 || !b1 || !w2) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  if (G < 1 || H < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad gating dims");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  auto* g = new molr_gating();
  g->ctx = ctx;
  g->G = G;
  g->H = H;
  g->d_u = d_u;
  g->H_u = H_u;
  auto up = [&](float** dst, const float* src, size_t n) -> int {
    if (!src) return MOLR_OK;
    MOLR_CUDA(cudaMalloc(dst, n * 4));
    MOLR_CUDA(cudaMemcpy(*dst, src, n * 4, cudaMemcpyDefault));
    return MOLR_OK;
  };
  int st = up(&g->w1, w1, size_t(G) * H);
  if (!st) st = up(&g->b1, b1, H);
  if (!st) st = up(&g->w2, w2, size_t(H) * G);
  if (!st && uw1 && d_u > 0 && H_u > 0) {
    st = up(&g->uw1, uw1, size_t(d_u) * H_u);
    if (!st) st = up(&g->ub1, ub1, H_u);
    if (!st) st = up(&g->uw2, uw2, size_t(H_u) * G);
  }
  if (!st) st = molr_gating_tc_prepare(g);
  if (st) {
    molr_gating_destroy(g);
    return st;
  }
  *out = g;
  return MOLR_OK;
}

int molr_gating_destroy(molr_gating* g) {
  if (!g) return MOLR_OK;
  cudaSetDevice(g->ctx->device);
  cudaFree(g->w1);
  cudaFree(g->b1);
  cudaFree(g->w2);
  cudaFree(g->uw1);
  cudaFree(g->ub1);
  cudaFree(g->uw2);
  cudaFree(g->w1t_bf16);  // w2t_bf16 points into the same allocation
  delete g;
  return MOLR_OK;
}

}  // extern "C"

// ---- per-kernel timing registry -------------------------------------------------------------
extern "C" {

int molr_ctx_set_profiling(molr_ctx* ctx, int on) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  ctx->prof.store(on ? 1 : 0);
  return MOLR_OK;
}

static int prof_drain(molr_ctx* ctx) {
  std::lock_guard<std::mutex> g(ctx->prof_mu);
  for (auto& r : ctx->prof_pending) {
    MOLR_CUDA(cudaEventSynchronize(r.end));
    float ms = 0;
    MOLR_CUDA(cudaEventElapsedTime(&ms, r.start, r.end));
    bool found = false;
    for (auto& kv : ctx->prof_sums)
      if (kv.first == r.name) {
        kv.second.count++;
        kv.second.ms += ms;
        kv.second.work += r.work;
        found = true;
        break;
      }
    if (!found) {
      molr_prof_sum s;
      s.count = 1;
      s.ms = ms;
      s.work = r.work;
      ctx->prof_sums.emplace_back(r.name, s);
    }
    ctx->prof_free.push_back(r.start);
    ctx->prof_free.push_back(r.end);
  }
  ctx->prof_pending.clear();
  return MOLR_OK;
}

int molr_ctx_prof_read(molr_ctx* ctx, int idx, char* name, int name_len, int64_t* count, double* total_ms,
                       double* work) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_TRY(prof_drain(ctx));
  std::lock_guard<std::mutex> g(ctx->prof_mu);
  if (idx < 0 || idx >= (int)ctx->prof_sums.size()) return MOLR_ERR_OUT_OF_RANGE;
  const auto& kv = ctx->prof_sums[idx];
  if (name && name_len > 0) {
    strncpy(name, kv.first.c_str(), name_len - 1);
    name[name_len - 1] = 0;
  }
  if (count) *count = kv.second.count;
  if (total_ms) *total_ms = kv.second.ms;
  if (work) *work = kv.second.work;
  return MOLR_OK;
}

int molr_ctx_prof_reset(molr_ctx* ctx) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_TRY(prof_drain(ctx));
  std::lock_guard<std::mutex> g(ctx->prof_mu);
  ctx->prof_sums.clear();
  return MOLR_OK;
}

}  // extern "C"
