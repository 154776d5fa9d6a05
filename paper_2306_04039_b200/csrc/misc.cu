// Small exact elementwise/reduction kernels behind the cache build and the drop-in API:
// l2_normalize_rows (numerics.py:41-50), stage-1 mean (mol.py:318), dequantize (quant.py:45-46),
// cache read-back, estimate_threshold (hindexer.py:115-132).
#include <algorithm>

#include "kernels.cuh"
#include "stage1.cuh"

namespace molr {

// NumPy's pairwise summation for a contiguous row (numpy/_core/src/umath/loops_utils.h.src):
// n < 8: sequential; n <= 128: eight strided partial sums combined ((0+1)+(2+3))+((4+5)+(6+7))
// plus a sequential tail; larger n: split at n/2 rounded down to a multiple of 8 and recurse.
__device__ float np_pairwise_sumsq(const float* a, int n) {
  if (n < 8) {
    float r = 0.f;
    for (int i = 0; i < n; ++i) r += a[i] * a[i];
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j] * a[j];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j] * a[i + j];
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i] * a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sumsq(a, n2) + np_pairwise_sumsq(a + n2, n - n2);
}

__global__ void l2norm_kernel(int64_t rows, int dim, const float* __restrict__ x, float eps, float* __restrict__ out,
                              int* __restrict__ bad) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const float* xr = x + r * dim;
    float nrm = __fsqrt_rn(np_pairwise_sumsq(xr, dim));
    if (!(nrm > eps)) atomicOr(bad, 1);
    for (int k = 0; k < dim; ++k) out[r * dim + k] = __fdiv_rn(xr[k], nrm);
  }
}

// in-place round-to-nearest-even to bf16 precision (value stays f32)
__global__ void round_bf16_kernel(float* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __bfloat162float(__float2bfloat16_rn(x[i]));
}

__global__ void mean_mid_kernel(int64_t n, int k, int d, const float* __restrict__ x, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * d; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / d, c = i % d;
    float acc = x[(r * k) * d + c];
    for (int a = 1; a < k; ++a) acc = __fadd_rn(acc, x[(r * k + a) * d + c]);
    out[i] = __fdiv_rn(acc, (float)k);
  }
}

__global__ void dequant_kernel(int64_t rows, int dim, const int8_t* __restrict__ c, const float* __restrict__ s,
                               float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * dim; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn((float)c[i], s[i / dim]);
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ a, int64_t n, float* __restrict__ o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __bfloat162float(a[i]);
}

// cache item components (bf16, possibly swizzled) -> plain (rows, k_x, d) f32
__global__ void embs_to_f32_kernel(const __nv_bfloat16* __restrict__ a, int64_t rows, int k_x, int d,
                                   float* __restrict__ o) {
  const int64_t ne = int64_t(k_x) * d;
  const bool swz = emb_swizzled(k_x, d);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ne; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / ne;
    int e = int(i % ne);
    o[i] = __bfloat162float(a[r * ne + emb_offset(e / d, e % d, d, swz)]);
  }
}

// interleaved cache codes rows [r0, r0+n) -> linear (n, 64)
__global__ void codes_from_ilv_kernel(const int8_t* __restrict__ src, const int32_t* __restrict__ inv,
                                      const float* __restrict__ scales, int64_t r0, int64_t n, int8_t* __restrict__ dst,
                                      float* __restrict__ dsc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i >> 2;
    const int c = int(i & 3);
    const int64_t pos = inv ? inv[r0 + r] : r0 + r;
    if (dst) *reinterpret_cast<int4*>(dst + r * 64 + c * 16) = *reinterpret_cast<const int4*>(src + s1_chunk_offset(pos, c, 64));
    if (dsc && c == 0) dsc[r] = scales[pos];
  }
}

static int grid_for(molr_ctx* ctx, int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ctx->num_sms * 16)); }

// Elementwise primitives of numerics.py:52-81 (sigmoid = scipy expit, silu, silu_grad) and the
// row softmax (numerics.py:61-66), f32 or f64 like the NumPy inputs.  The hot kernels inline
// their own forms; these serve the drop-in module surface.
template <class T>
__device__ __forceinline__ T expit_(T x) {
  return T(1) / (T(1) + exp(-x));
}
template <class T>
__global__ void eltwise_kernel(int op, int64_t n, const T* __restrict__ x, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[i], sg = expit_(v);
    out[i] = op == 0 ? sg : (op == 1 ? v * sg : sg * (T(1) + v * (T(1) - sg)));
  }
}
// one warp per row: max, exp(x - max), sum, divide
template <class T>
__global__ void softmax_rows_kernel(int64_t rows, int dim, const T* __restrict__ x, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const T* xr = x + r * dim;
    T mx = -INFINITY;
    for (int j = lane; j < dim; j += 32) mx = max(mx, xr[j]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    T sum = 0;
    for (int j = lane; j < dim; j += 32) sum += exp(xr[j] - mx);
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    for (int j = lane; j < dim; j += 32) out[r * dim + j] = exp(xr[j] - mx) / sum;
  }
}

}  // namespace molr

using namespace molr;

extern "C" {

int molr_l2_normalize_rows(molr_ctx* ctx, int64_t rows, int dim, const float* x, float eps, float* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (rows < 0 || dim < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad shape");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (rows == 0) return MOLR_OK;
  In xi;
  Out o;
  Scratch bad;
  MOLR_TRY(xi.stage(x, size_t(rows) * dim * 4, s));
  MOLR_TRY(o.stage(out, size_t(rows) * dim * 4, s));
  MOLR_TRY(bad.alloc(4, s));
  MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  l2norm_kernel<<<grid_for(ctx, rows), 256, 0, s>>>(rows, dim, xi.as<float>(), eps, o.as<float>(), bad.as<int>());
  MOLR_LAUNCHED(ctx);
  int hb = 0;
  MOLR_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
  MOLR_TRY(finish_outputs(s, {&o}));
  MOLR_CUDA(cudaStreamSynchronize(s));
  if (hb) MOLR_FAIL(MOLR_ERR_ZERO_NORM, "at least one row has norm <= eps");
  return MOLR_OK;
}

int molr_mean_rows(molr_ctx* ctx, int64_t n, int k, int d, const float* x, float* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n <= 0) return MOLR_OK;
  In xi;
  Out o;
  MOLR_TRY(xi.stage(x, size_t(n) * k * d * 4, s));
  MOLR_TRY(o.stage(out, size_t(n) * d * 4, s));
  mean_mid_kernel<<<grid_for(ctx, n * d), 256, 0, s>>>(n, k, d, xi.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

// Device-side build_item_cache for rows [row0, row0 + n) of a cache (mol.py:294-326), fused and
// chunked: item_proj MLP -> (k_x, d) -> L2-normalise -> item_net MLP -> [bf16 rounding of the
// stored fields] -> stage-1 = mean over k_x -> rowwise int8 quantisation -> cache rows.  Only
// the item table chunk crosses PCIe; every intermediate stays on the device.
int molr_cache_build_rows(molr_cache* c, int64_t row0, int64_t n, int d_x, const float* item_table, int proj_hidden,
                          const float* pw1, const float* pb1, const float* pw2, int net_hidden, const float* nw1,
                          const float* nb1, const float* nw2, int flags, float eps, void* stream) {
  if (!c) MOLR_FAIL(MOLR_ERR_INVALID, "null cache");
  if (row0 < 0 || n < 0 || row0 + n > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "build rows out of range");
  if (d_x < 1 || proj_hidden < 1 || net_hidden < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad tower dims");
  if (c->d1 && c->d1 != c->d) MOLR_FAIL(MOLR_ERR_DIMENSION, "stage-1 dim %d != d %d", c->d1, c->d);
  if (n == 0) return MOLR_OK;
  molr_ctx* ctx = c->ctx;
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  const int kd = c->k_x * c->d, G = c->G;
  if (size_t(d_x + std::max(proj_hidden, net_hidden)) * 4 > 200 * 1024) MOLR_FAIL(MOLR_ERR_DIMENSION, "mlp too wide");
  In a1, a2, a3, b1, b2, b3;
  MOLR_TRY(a1.stage(pw1, size_t(d_x) * proj_hidden * 4, s));
  MOLR_TRY(a2.stage(pb1, size_t(proj_hidden) * 4, s));
  MOLR_TRY(a3.stage(pw2, size_t(proj_hidden) * kd * 4, s));
  MOLR_TRY(b1.stage(nw1, size_t(d_x) * net_hidden * 4, s));
  MOLR_TRY(b2.stage(nb1, size_t(net_hidden) * 4, s));
  MOLR_TRY(b3.stage(nw2, size_t(net_hidden) * G * 4, s));
  const int64_t chunk = std::max<int64_t>(1, (int64_t(256) << 20) / (int64_t(kd + G + c->d + d_x) * 4));
  Scratch bad;
  MOLR_TRY(bad.alloc(4, s));
  MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  for (int64_t r = 0; r < n; r += chunk) {
    const int m = (int)std::min(chunk, n - r);
    In xt;
    MOLR_TRY(xt.stage(item_table + r * d_x, size_t(m) * d_x * 4, s));
    Scratch e, g, s1, codes, scales;
    MOLR_TRY(e.alloc(size_t(m) * kd * 4, s));
    MOLR_TRY(g.alloc(size_t(m) * G * 4, s));
    MOLR_TRY(s1.alloc(size_t(m) * c->d * 4, s));
    auto mlp = [&](int hidden, const In& w1, const In& bb, const In& w2, int out_dim, float* out) -> int {
      const size_t smem = size_t(d_x + hidden) * 4;
      MOLR_CUDA(cudaFuncSetAttribute(mlp_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      mlp_forward_kernel<<<std::min(m, ctx->num_sms * 8), 128, smem, s>>>(m, d_x, hidden, out_dim, w1.as<float>(),
                                                                        bb.as<float>(), w2.as<float>(), xt.as<float>(), out);
      MOLR_LAUNCHED(ctx);
      return MOLR_OK;
    };
    MOLR_TRY(mlp(proj_hidden, a1, a2, a3, kd, e.as<float>()));
    if (flags & MOLR_BUILD_L2_NORMALIZE) {
      l2norm_kernel<<<grid_for(ctx, int64_t(m) * c->k_x), 256, 0, s>>>(int64_t(m) * c->k_x, c->d, e.as<float>(), eps,
                                                                      e.as<float>(), bad.as<int>());
      MOLR_LAUNCHED(ctx);
    }
    MOLR_TRY(mlp(net_hidden, b1, b2, b3, G, g.as<float>()));
    if (flags & MOLR_BUILD_ROUND_BF16) {  // production storage: the cache IS these bf16 values
      round_bf16_kernel<<<grid_for(ctx, int64_t(m) * kd), 256, 0, s>>>(e.as<float>(), int64_t(m) * kd);
      round_bf16_kernel<<<grid_for(ctx, int64_t(m) * G), 256, 0, s>>>(g.as<float>(), int64_t(m) * G);
      ctx->launches += 2;
    }
    mean_mid_kernel<<<grid_for(ctx, int64_t(m) * c->d), 256, 0, s>>>(m, c->k_x, c->d, e.as<float>(), s1.as<float>());
    MOLR_LAUNCHED(ctx);
    if (c->s1_codes) {
      MOLR_TRY(codes.alloc(size_t(m) * c->d, s));
      MOLR_TRY(scales.alloc(size_t(m) * 4, s));
      MOLR_TRY(quantize_rows(ctx, m, c->d, s1.as<float>(), codes.as<int8_t>(), scales.as<float>(), s));
    }
    int hb = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (hb) MOLR_FAIL(MOLR_ERR_ZERO_NORM, "at least one item component has norm <= eps");
    MOLR_TRY(molr_cache_fill(c, row0 + r, m, e.as<float>(), g.as<float>(), c->s1_f32 ? s1.as<float>() : nullptr,
                             codes.as<int8_t>(), scales.as<float>(), s));
  }
  return MOLR_OK;
}

// Batched user-side query prep (RetrievalEngine.query_state -> model.user_forward,
// engine.py:113-115, model.py:179-208; and decomposed_gating's user_net, mol.py:186):
// user_embs = L2-normalise(user_proj(feats).reshape(k_u, d)) and uw = user_net(feats), on device.
int molr_query_prep(molr_ctx* ctx, int B, int d_u, const float* feats, int proj_hidden, const float* pw1,
                    const float* pb1, const float* pw2, int k_u, int d, int l2_normalized, int net_hidden,
                    const float* nw1, const float* nb1, const float* nw2, int G, float eps, float* user_embs, float* uw,
                    void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (B < 0 || d_u < 1 || proj_hidden < 1 || net_hidden < 1 || k_u < 1 || d < 1 || G < 1)
    MOLR_FAIL(MOLR_ERR_DIMENSION, "bad query-prep dims");
  if (size_t(d_u + std::max(proj_hidden, net_hidden)) * 4 > 200 * 1024) MOLR_FAIL(MOLR_ERR_DIMENSION, "mlp too wide");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B == 0) return MOLR_OK;
  In x, a1, a2, a3, b1, b2, b3;
  MOLR_TRY(x.stage(feats, size_t(B) * d_u * 4, s));
  MOLR_TRY(a1.stage(pw1, size_t(d_u) * proj_hidden * 4, s));
  MOLR_TRY(a2.stage(pb1, size_t(proj_hidden) * 4, s));
  MOLR_TRY(a3.stage(pw2, size_t(proj_hidden) * k_u * d * 4, s));
  MOLR_TRY(b1.stage(nw1, size_t(d_u) * net_hidden * 4, s));
  MOLR_TRY(b2.stage(nb1, size_t(net_hidden) * 4, s));
  MOLR_TRY(b3.stage(nw2, size_t(net_hidden) * G * 4, s));
  Out oe, ow;
  MOLR_TRY(oe.stage(user_embs, size_t(B) * k_u * d * 4, s));
  MOLR_TRY(ow.stage(uw, size_t(B) * G * 4, s));
  auto mlp = [&](int hidden, const In& w1, const In& bb, const In& w2, int out_dim, float* out) -> int {
    const size_t smem = size_t(d_u + hidden) * 4;
    MOLR_CUDA(cudaFuncSetAttribute(mlp_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 grid(std::min(B, ctx->num_sms * 8), std::min(div_up(out_dim, 128), std::max(1, ctx->num_sms / std::max(B, 1))));
    mlp_forward_kernel<<<grid, 128, smem, s>>>(B, d_u, hidden, out_dim, w1.as<float>(), bb.as<float>(), w2.as<float>(),
                                               x.as<float>(), out);
    MOLR_LAUNCHED(ctx);
    return MOLR_OK;
  };
  MOLR_TRY(mlp(proj_hidden, a1, a2, a3, k_u * d, oe.as<float>()));
  MOLR_TRY(mlp(net_hidden, b1, b2, b3, G, ow.as<float>()));
  Scratch bad;
  if (l2_normalized) {
    MOLR_TRY(bad.alloc(4, s));
    MOLR_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
    l2norm_kernel<<<grid_for(ctx, int64_t(B) * k_u), 256, 0, s>>>(int64_t(B) * k_u, d, oe.as<float>(), eps, oe.as<float>(),
                                                                bad.as<int>());
    MOLR_LAUNCHED(ctx);
    int hb = 0;
    MOLR_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (hb) MOLR_FAIL(MOLR_ERR_ZERO_NORM, "a user component has norm <= eps");
  }
  return finish_outputs(s, {&oe, &ow});
}

int molr_eltwise(molr_ctx* ctx, int op, int dtype, int64_t n, const void* x, void* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (op < 0 || op > 2 || (dtype != 0 && dtype != 2)) MOLR_FAIL(MOLR_ERR_INVALID, "op %d dtype %d", op, dtype);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n <= 0) return MOLR_OK;
  const size_t es = dtype == 2 ? 8 : 4;
  In xi;
  Out o;
  MOLR_TRY(xi.stage(x, size_t(n) * es, s));
  MOLR_TRY(o.stage(out, size_t(n) * es, s));
  if (dtype == 2) eltwise_kernel<double><<<grid_for(ctx, n), 256, 0, s>>>(op, n, xi.as<double>(), o.as<double>());
  else eltwise_kernel<float><<<grid_for(ctx, n), 256, 0, s>>>(op, n, xi.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

int molr_softmax_rows(molr_ctx* ctx, int dtype, int64_t rows, int dim, const void* x, void* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (dim < 1 || (dtype != 0 && dtype != 2)) MOLR_FAIL(MOLR_ERR_INVALID, "dim %d dtype %d", dim, dtype);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (rows <= 0) return MOLR_OK;
  const size_t es = dtype == 2 ? 8 : 4;
  In xi;
  Out o;
  MOLR_TRY(xi.stage(x, size_t(rows) * dim * es, s));
  MOLR_TRY(o.stage(out, size_t(rows) * dim * es, s));
  const int blocks = (int)std::min<int64_t>((rows + 7) / 8, int64_t(ctx->num_sms) * 16);
  if (dtype == 2) softmax_rows_kernel<double><<<blocks, 256, 0, s>>>(rows, dim, xi.as<double>(), o.as<double>());
  else softmax_rows_kernel<float><<<blocks, 256, 0, s>>>(rows, dim, xi.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

int molr_dequantize_rows(molr_ctx* ctx, int64_t rows, int dim, const int8_t* codes, const float* scales, float* out,
                         void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (rows <= 0) return MOLR_OK;
  In c, sc;
  Out o;
  MOLR_TRY(c.stage(codes, size_t(rows) * dim, s));
  MOLR_TRY(sc.stage(scales, size_t(rows) * 4, s));
  MOLR_TRY(o.stage(out, size_t(rows) * dim * 4, s));
  dequant_kernel<<<grid_for(ctx, rows * dim), 256, 0, s>>>(rows, dim, c.as<int8_t>(), sc.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

int molr_cache_read(const molr_cache* c, int64_t row0, int64_t n, float* embs, float* gp, float* s1, int8_t* codes,
                    float* scales, void* stream) {
  if (!c) MOLR_FAIL(MOLR_ERR_INVALID, "null cache");
  if (row0 < 0 || n < 0 || row0 + n > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "rows out of range");
  molr_ctx* ctx = c->ctx;
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n == 0) return MOLR_OK;
  const int64_t ne = int64_t(c->k_x) * c->d;
  Out oe, og, os1, oc, osc;
  if (embs) {
    MOLR_TRY(oe.stage(embs, size_t(n) * ne * 4, s));
    if (c->embs_f32)
      MOLR_CUDA(cudaMemcpyAsync(oe.dptr, c->embs_f32 + row0 * ne, size_t(n) * ne * 4, cudaMemcpyDeviceToDevice, s));
    else {
      embs_to_f32_kernel<<<grid_for(ctx, n * ne), 256, 0, s>>>(c->embs_bf16 + row0 * ne, n, c->k_x, c->d, oe.as<float>());
      MOLR_LAUNCHED(ctx);
    }
  }
  if (gp) {
    MOLR_TRY(og.stage(gp, size_t(n) * c->G * 4, s));
    if (c->gp_f32)
      MOLR_CUDA(cudaMemcpyAsync(og.dptr, c->gp_f32 + row0 * c->G, size_t(n) * c->G * 4, cudaMemcpyDeviceToDevice, s));
    else {
      bf16_to_f32_kernel<<<grid_for(ctx, n * c->G), 256, 0, s>>>(c->gp_bf16 + row0 * c->G, n * c->G, og.as<float>());
      MOLR_LAUNCHED(ctx);
    }
  }
  if (s1 && c->s1_f32) MOLR_CUDA(cudaMemcpyAsync(s1, c->s1_f32 + row0 * c->d1, size_t(n) * c->d1 * 4, cudaMemcpyDefault, s));
  Out ocodes, oscales;
  if ((codes || scales) && c->s1_codes) {
    if (s1_interleaved(c->d1)) {
      MOLR_TRY(ocodes.stage(codes, codes ? size_t(n) * c->d1 : 0, s));
      MOLR_TRY(oscales.stage(scales, scales ? size_t(n) * 4 : 0, s));
      codes_from_ilv_kernel<<<grid_for(ctx, n * 4), 256, 0, s>>>(c->s1_codes, c->s1_inv, c->s1_scales, row0, n,
                                                                 ocodes.as<int8_t>(), oscales.as<float>());
      MOLR_LAUNCHED(ctx);
    } else {
      if (codes) MOLR_CUDA(cudaMemcpyAsync(codes, c->s1_codes + row0 * c->d1, size_t(n) * c->d1, cudaMemcpyDefault, s));
      if (scales) MOLR_CUDA(cudaMemcpyAsync(scales, c->s1_scales + row0, size_t(n) * 4, cudaMemcpyDefault, s));
    }
  }
  MOLR_TRY(finish_outputs(s, {&oe, &og, &ocodes, &oscales}));
  MOLR_CUDA(cudaStreamSynchronize(s));
  return MOLR_OK;
}

int molr_estimate_threshold(molr_ctx* ctx, const molr_cache* c, int mode, int B, const float* q, int64_t lam,
                            const int64_t* sample, int64_t n_rank, double* out_t, void* stream) {
  if (!ctx || !c) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_TRY(check_view(c, mode));
  if (lam < 1 || lam > c->X) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "lambda %lld outside [1, %lld]", (long long)lam,
                                       (long long)c->X);
  if (n_rank < 1 || n_rank > lam) MOLR_FAIL(MOLR_ERR_OUT_OF_RANGE, "n=%lld outside [1, %lld]", (long long)n_rank,
                                            (long long)lam);
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (B <= 0) return MOLR_OK;
  In qi, si;
  MOLR_TRY(qi.stage(q, size_t(B) * c->d1 * 4, s));
  MOLR_TRY(si.stage(sample, size_t(B) * lam * 8, s));
  Scratch qc, qs, ss, tk;
  if (mode != MOLR_S1_FLOAT) {
    MOLR_TRY(qc.alloc(size_t(B) * c->d1, s));
    MOLR_TRY(qs.alloc(size_t(B) * 4, s));
    MOLR_TRY(prepare_queries(ctx, mode, B, c->d1, qi.as<float>(), qc.as<int8_t>(), qs.as<float>(), s));
  }
  MOLR_TRY(ss.alloc(size_t(B) * lam * 4, s));
  MOLR_TRY(tk.alloc(size_t(B) * 4, s));
  for (int b = 0; b < B; ++b) {  // each query has its own sample rows
    MOLR_TRY(scan_scores(ctx, mode, lam, c->d1, c->s1_f32, c->s1_codes, s1_interleaved(c->d1), c->s1_inv, c->s1_scales, si.as<int64_t>() + size_t(b) * lam,
                         1, qi.as<float>() + size_t(b) * c->d1, qc.as<int8_t>() ? qc.as<int8_t>() + size_t(b) * c->d1 : nullptr,
                         ss.as<float>() + size_t(b) * lam, lam, s));
  }
  MOLR_TRY(nth_largest_rows(ctx, B, lam, ss.p, mode == MOLR_S1_INT8_RAW, lam, nullptr, 0, n_rank, tk.as<uint32_t>(), s));
  std::vector<uint32_t> hk(B);
  MOLR_CUDA(cudaMemcpyAsync(hk.data(), tk.p, size_t(B) * 4, cudaMemcpyDeviceToHost, s));
  MOLR_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) out_t[b] = mode == MOLR_S1_INT8_RAW ? double(key_i32(hk[b])) : double(key_f32(hk[b]));
  return MOLR_OK;
}

}  // extern "C"
