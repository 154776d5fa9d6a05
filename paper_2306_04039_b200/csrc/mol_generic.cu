// Mixture-of-Logits kernels, generic shapes (SIMT fp32).  These implement the reference's MoL
// primitives for ANY (k_u, k_x, d, G, H) — mol.py:139-205 — and the fused cache scorer used when
// the tcgen05 production kernel (mol_tc.cu, k_u=k_x=8, d=64, H=128) does not apply.
#include <algorithm>

#include "kernels.cuh"

namespace molr {

// ------------------------------------------------------------------------------------------
// primitives
// ------------------------------------------------------------------------------------------
// component_logits — mol.py:139-158: out[i, a*k_x+b] = <u_a, e_{i,b}> / tau  (f32 or f64 inputs,
// computed in the input precision like NumPy)
template <class T>
__global__ void component_logits_kernel(int n, int k_u, int k_x, int d, const T* __restrict__ u,
                                        const T* __restrict__ e, T tau, T* __restrict__ out) {
  int64_t G = int64_t(k_u) * k_x;
  int64_t total = int64_t(n) * G;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = o / G;
    int g = int(o % G), a = g / k_x, b = g % k_x;
    const T* ua = u + int64_t(a) * d;
    const T* eb = e + (i * k_x + b) * d;
    T acc = 0;
    for (int k = 0; k < d; ++k) acc = fma(ua[k], eb[k], acc);
    out[o] = acc / tau;
  }
}

// Mlp.__call__ — mol.py:84-85: silu(x @ w1 + b1) @ w2.  One block per row.
__global__ void mlp_forward_kernel(int rows, int in_dim, int hidden, int out_dim, const float* __restrict__ w1,
                                   const float* __restrict__ b1, const float* __restrict__ w2,
                                   const float* __restrict__ x, float* __restrict__ out) {
  extern __shared__ float sm[];
  float* xs = sm;               // in_dim
  float* hs = sm + in_dim;      // hidden
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    for (int k = threadIdx.x; k < in_dim; k += blockDim.x) xs[k] = x[int64_t(r) * in_dim + k];
    __syncthreads();
    for (int j = threadIdx.x; j < hidden; j += blockDim.x) {
      float acc = 0.f;
      for (int k = 0; k < in_dim; ++k) acc = fmaf(xs[k], w1[int64_t(k) * hidden + j], acc);
      hs[j] = silu_f32(acc + b1[j]);
    }
    __syncthreads();
    // gridDim.y blocks share a row's outputs (small batches: more blocks in flight; every block
    // recomputes the same hidden layer, so results do not depend on the split)
    for (int o = blockIdx.y * blockDim.x + threadIdx.x; o < out_dim; o += gridDim.y * blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < hidden; ++j) acc = fmaf(hs[j], w2[int64_t(j) * out_dim + o], acc);
      out[int64_t(r) * out_dim + o] = acc;
    }
    __syncthreads();
  }
}

// decomposed_gating (inference) — mol.py:161-194: pi = softmax(silu(uw*gp + cross_net(cl))).
// One block per row; G <= 1024.
__global__ void gating_kernel(int n, int G, int H, const float* __restrict__ w1, const float* __restrict__ b1,
                              const float* __restrict__ w2, const float* __restrict__ uw,
                              const float* __restrict__ gp, const float* __restrict__ cl, float* __restrict__ out) {
  extern __shared__ float sm[];
  float* cls = sm;         // G
  float* hs = sm + G;      // H
  float* pre = hs + H;     // G
  __shared__ float red[32];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    for (int g = threadIdx.x; g < G; g += blockDim.x) cls[g] = cl[int64_t(i) * G + g];
    __syncthreads();
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
      float acc = 0.f;
      for (int g = 0; g < G; ++g) acc = fmaf(cls[g], w1[int64_t(g) * H + j], acc);
      hs[j] = silu_f32(acc + b1[j]);
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      float acc = 0.f;
      for (int j = 0; j < H; ++j) acc = fmaf(hs[j], w2[int64_t(j) * G + g], acc);
      float v = silu_f32(uw[g] * gp[int64_t(i) * G + g] + acc);
      pre[g] = v;
      mx = fmaxf(mx, v);
    }
    // block max
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : -INFINITY;
      for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float sum = 0.f;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
      float e = expf(pre[g] - mx);
      pre[g] = e;
      sum += e;
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.f;
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    sum = red[0];
    for (int g = threadIdx.x; g < G; g += blockDim.x) out[int64_t(i) * G + g] = __fdiv_rn(pre[g], sum);
    __syncthreads();
  }
}

// mol_score — mol.py:197-205 (f32 or f64)
template <class T>
__global__ void mol_score_kernel(int n, int G, const T* __restrict__ pi, const T* __restrict__ cl,
                                 T* __restrict__ out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nw) {
    T acc = 0;
    for (int g = lane; g < G; g += 32) acc = fma(pi[int64_t(i) * G + g], cl[int64_t(i) * G + g], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[i] = acc;
  }
}

// ------------------------------------------------------------------------------------------
// fused scorer over a cache: gather -> component logits -> cross net -> combine -> softmax ->
// gated sum, per (query, candidate) pair.  score_candidates / batch_score_all — mol.py:329-386.
// Persistent CTAs walk a tile list; a tile is P candidates of one query.
// ------------------------------------------------------------------------------------------
constexpr int kGenP = 16;
constexpr int kGenThreads = 256;

// tile prefix over segments: pre[b+1] = pre[b] + ceil(len_b / P)
__global__ void tile_prefix_kernel(int B, const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                                   int64_t X, int P, int64_t* __restrict__ pre) {
  // single block scan (B is the query batch, <= a few thousand)
  __shared__ int64_t part[1024];
  int t = threadIdx.x;
  int per = (B + blockDim.x - 1) / blockDim.x;
  int lo = t * per, hi = min(B, lo + per);
  int64_t s = 0;
  for (int b = lo; b < hi; ++b) {
    int64_t len = begin ? (end[b] - begin[b]) : X;
    s += (len + P - 1) / P;
  }
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      int64_t v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  int64_t run = part[t];
  if (t == 0) pre[0] = 0;
  for (int b = lo; b < hi; ++b) {
    int64_t len = begin ? (end[b] - begin[b]) : X;
    run += (len + P - 1) / P;
    pre[b + 1] = run;
  }
}

template <class Id, bool EF32, bool GPF32>
__global__ void __launch_bounds__(kGenThreads)
mol_fused_generic_kernel(int B, int k_u, int k_x, int d, int G, int H, float tau,
                         const void* __restrict__ ev,
                         const void* __restrict__ gpv, const float* __restrict__ w1g,
                         const float* __restrict__ b1g, const float* __restrict__ w2g,
                         const float* __restrict__ user_embs, const float* __restrict__ uwg,
                         const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                         const Id* __restrict__ ids, int64_t X, const int64_t* __restrict__ tile_pre,
                         float* __restrict__ out, int64_t out_ld) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float* W1 = reinterpret_cast<float*>(smraw);          // G*H
  float* W2 = W1 + G * H;                               // H*G
  float* bb1 = W2 + H * G;                              // H
  float* us = bb1 + H;                                  // k_u*d
  float* uws = us + k_u * d;                            // G
  float* cl = uws + G;                                  // P*G
  float* hh = cl + kGenP * G;                           // P*H
  float* cw = hh + kGenP * H;                           // P*G
  float* eh = cw + kGenP * G;                           // P*k_x*d item rows (f32)
  __shared__ int64_t xs[kGenP];
  __shared__ int cur_b;

  const int t = threadIdx.x;
  for (int i = t; i < G * H; i += blockDim.x) {
    W1[i] = w1g[i];
    W2[i] = w2g[i];
  }
  for (int i = t; i < H; i += blockDim.x) bb1[i] = b1g[i];
  if (t == 0) cur_b = -1;
  __syncthreads();

  const int64_t T = tile_pre[B];
  const int ne = k_x * d;
  for (int64_t tile = blockIdx.x; tile < T; tile += gridDim.x) {
    // locate query b: largest b with tile_pre[b] <= tile
    int lo = 0, hi = B - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (tile_pre[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int64_t seg0 = begin ? begin[b] : 0;
    const int64_t len = begin ? (end[b] - begin[b]) : X;
    const int64_t j0 = (tile - tile_pre[b]) * kGenP;
    const int np = (int)imin64(kGenP, len - j0);
    if (b != cur_b) {  // block-uniform
      __syncthreads();
      for (int i = t; i < k_u * d; i += blockDim.x) us[i] = user_embs[int64_t(b) * k_u * d + i];
      for (int i = t; i < G; i += blockDim.x) uws[i] = uwg[int64_t(b) * G + i];
      __syncthreads();
      if (t == 0) cur_b = b;
    }
    if (t < kGenP) xs[t] = t < np ? (ids ? (int64_t)ids[seg0 + j0 + t] : j0 + t) : 0;
    __syncthreads();
    // stage item rows (bf16) into SMEM
    const bool swz = emb_swizzled(k_x, d);
    for (int i = t; i < kGenP * ne; i += blockDim.x) {
      int p = i / ne, r = i % ne;
      int64_t x = xs[p];
      eh[i] = EF32 ? reinterpret_cast<const float*>(ev)[x * ne + r]
                   : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(ev)[x * ne + emb_offset(r / d, r % d, d, swz)]);
    }
    __syncthreads();
    // phase A: component logits
    for (int o = t; o < kGenP * G; o += blockDim.x) {
      int p = o / G, g = o % G, a = g / k_x, bb = g % k_x;
      const float* ua = us + a * d;
      const float* eb = eh + p * ne + bb * d;
      float acc = 0.f;
      for (int k = 0; k < d; ++k) acc = fmaf(ua[k], eb[k], acc);
      cl[o] = __fdiv_rn(acc, tau);
    }
    __syncthreads();
    // phase B: hidden = silu(cl @ W1 + b1)
    for (int o = t; o < kGenP * H; o += blockDim.x) {
      int p = o / H, j = o % H;
      const float* c = cl + p * G;
      float acc = 0.f;
      for (int g = 0; g < G; ++g) acc = fmaf(c[g], W1[g * H + j], acc);
      hh[o] = silu_f32(acc + bb1[j]);
    }
    __syncthreads();
    // phase C: cw = hidden @ W2
    for (int o = t; o < kGenP * G; o += blockDim.x) {
      int p = o / G, g = o % G;
      const float* hp = hh + p * H;
      float acc = 0.f;
      for (int j = 0; j < H; ++j) acc = fmaf(hp[j], W2[j * G + g], acc);
      cw[o] = acc;
    }
    __syncthreads();
    // phase D: combine, softmax, gated sum (one warp per pair)
    const int warp = t >> 5, lane = t & 31;
    for (int p = warp; p < np; p += kGenThreads / 32) {
      int64_t x = xs[p];
      float mx = -INFINITY;
      for (int g = lane; g < G; g += 32) {
        float gpx = GPF32 ? reinterpret_cast<const float*>(gpv)[x * G + g]
                          : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(gpv)[x * G + g]);
        float v = silu_f32(uws[g] * gpx + cw[p * G + g]);
        cw[p * G + g] = v;
        mx = fmaxf(mx, v);
      }
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float sum = 0.f;
      for (int g = lane; g < G; g += 32) {
        float e = expf(cw[p * G + g] - mx);
        cw[p * G + g] = e;
        sum += e;
      }
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      float s = 0.f;
      for (int g = lane; g < G; g += 32) s = fmaf(__fdiv_rn(cw[p * G + g], sum), cl[p * G + g], s);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        if (begin) out[seg0 + j0 + p] = s;
        else out[int64_t(b) * out_ld + j0 + p] = s;
      }
    }
    __syncthreads();
  }
}

size_t generic_smem_bytes(int k_u, int k_x, int d, int G, int H) {
  size_t f = size_t(G) * H * 2 + H + size_t(k_u) * d + G + size_t(kGenP) * (2 * G + H) + size_t(kGenP) * k_x * d;
  return f * 4;
}

template <class Id>
int mol_score_generic(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, int k_u,
                      const float* user_embs, const float* uw, float tau, Segs<Id> segs,
                      float* out, int64_t out_ld, cudaStream_t s) {
  const int G = g->G, H = g->H;
  size_t smem = generic_smem_bytes(k_u, c->k_x, c->d, G, H);
  if (smem > 220 * 1024)
    MOLR_FAIL(MOLR_ERR_DIMENSION, "MoL shape (k_u=%d k_x=%d d=%d G=%d H=%d) exceeds the fused kernel's "
              "shared-memory budget", k_u, c->k_x, c->d, G, H);
  if (B <= 0) return MOLR_OK;
  Scratch pre;
  MOLR_TRY(pre.alloc(size_t(B + 1) * 8, s));
  tile_prefix_kernel<<<1, 1024, 0, s>>>(B, segs.begin, segs.end, segs.X, kGenP, pre.as<int64_t>());
  MOLR_LAUNCHED(ctx);
  auto launch = [&](auto kern) -> int {
    MOLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = std::max(1, int((227 * 1024) / (smem + 1024)));
    kern<<<ctx->num_sms * per_sm, kGenThreads, smem, s>>>(
        B, k_u, c->k_x, c->d, G, H, tau, c->embs_f32 ? (const void*)c->embs_f32 : (const void*)c->embs_bf16,
        c->gp_f32 ? (const void*)c->gp_f32 : (const void*)c->gp_bf16, g->w1, g->b1, g->w2, user_embs, uw,
        segs.begin, segs.end, segs.ids, segs.X, pre.as<int64_t>(), out, out_ld);
    MOLR_LAUNCHED(ctx);
    return MOLR_OK;
  };
  bool lo = c->embs_f32 != nullptr, f32 = c->gp_f32 != nullptr;
  if (lo && f32) return launch(mol_fused_generic_kernel<Id, true, true>);
  if (lo) return launch(mol_fused_generic_kernel<Id, true, false>);
  if (f32) return launch(mol_fused_generic_kernel<Id, false, true>);
  return launch(mol_fused_generic_kernel<Id, false, false>);
}

template int mol_score_generic<int64_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, int,
                                        const float*, const float*, float, Segs<int64_t>, float*, int64_t,
                                        cudaStream_t);
template int mol_score_generic<int32_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, int,
                                        const float*, const float*, float, Segs<int32_t>, float*, int64_t,
                                        cudaStream_t);

// CSR offsets (B+1) -> begin/end views.
struct CsrSegs {
  const int64_t* begin = nullptr;
  const int64_t* end = nullptr;
};

}  // namespace molr

using namespace molr;

// ------------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------------
extern "C" {

int molr_component_logits(molr_ctx* ctx, int n, int k_u, int k_x, int d, const void* u, const void* e,
                          double tau, int is_f64, void* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (n < 0 || k_u < 1 || k_x < 1 || d < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad shapes");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n == 0) return MOLR_OK;
  const size_t es = is_f64 ? 8 : 4;
  In du, de;
  Out dout;
  MOLR_TRY(du.stage(u, size_t(k_u) * d * es, s));
  MOLR_TRY(de.stage(e, size_t(n) * k_x * d * es, s));
  MOLR_TRY(dout.stage(out, size_t(n) * k_u * k_x * es, s));
  if (is_f64)
    component_logits_kernel<double><<<ctx->num_sms * 4, 256, 0, s>>>(n, k_u, k_x, d, du.as<double>(), de.as<double>(),
                                                                     tau, dout.as<double>());
  else
    component_logits_kernel<float><<<ctx->num_sms * 4, 256, 0, s>>>(n, k_u, k_x, d, du.as<float>(), de.as<float>(),
                                                                    (float)tau, dout.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&dout});
}

int molr_mlp_forward(molr_ctx* ctx, int rows, int in_dim, int hidden, int out_dim, const float* w1,
                     const float* b1, const float* w2, const float* x, float* out, void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  if (rows < 0 || in_dim < 1 || hidden < 1 || out_dim < 1) MOLR_FAIL(MOLR_ERR_DIMENSION, "bad mlp shapes");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (rows == 0) return MOLR_OK;
  In a, bb, c, xx;
  Out o;
  MOLR_TRY(a.stage(w1, size_t(in_dim) * hidden * 4, s));
  MOLR_TRY(bb.stage(b1, size_t(hidden) * 4, s));
  MOLR_TRY(c.stage(w2, size_t(hidden) * out_dim * 4, s));
  MOLR_TRY(xx.stage(x, size_t(rows) * in_dim * 4, s));
  MOLR_TRY(o.stage(out, size_t(rows) * out_dim * 4, s));
  size_t smem = size_t(in_dim + hidden) * 4;
  if (smem > 200 * 1024) MOLR_FAIL(MOLR_ERR_DIMENSION, "mlp too wide");
  MOLR_CUDA(cudaFuncSetAttribute(mlp_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  mlp_forward_kernel<<<std::min(rows, ctx->num_sms * 8), 128, smem, s>>>(
      rows, in_dim, hidden, out_dim, a.as<float>(), bb.as<float>(), c.as<float>(), xx.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

int molr_decomposed_gating(molr_ctx* ctx, const molr_gating* g, int n, const float* uw, const float* gp,
                           const float* cl, float* out, void* stream) {
  if (!ctx || !g) MOLR_FAIL(MOLR_ERR_INVALID, "null argument");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n <= 0) return MOLR_OK;
  const int G = g->G, H = g->H;
  In a, b, c;
  Out o;
  MOLR_TRY(a.stage(uw, size_t(G) * 4, s));
  MOLR_TRY(b.stage(gp, size_t(n) * G * 4, s));
  MOLR_TRY(c.stage(cl, size_t(n) * G * 4, s));
  MOLR_TRY(o.stage(out, size_t(n) * G * 4, s));
  size_t smem = size_t(2 * G + H) * 4;
  if (smem > 200 * 1024) MOLR_FAIL(MOLR_ERR_DIMENSION, "gating too wide");
  MOLR_CUDA(cudaFuncSetAttribute(gating_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gating_kernel<<<std::min(n, ctx->num_sms * 8), 128, smem, s>>>(n, G, H, g->w1, g->b1, g->w2, a.as<float>(),
                                                                  b.as<float>(), c.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

int molr_mol_score(molr_ctx* ctx, int n, int G, const void* pi, const void* cl, int is_f64, void* out,
                   void* stream) {
  if (!ctx) MOLR_FAIL(MOLR_ERR_INVALID, "null ctx");
  MOLR_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = pick_stream(ctx, stream);
  if (n <= 0) return MOLR_OK;
  const size_t es = is_f64 ? 8 : 4;
  In a, b;
  Out o;
  MOLR_TRY(a.stage(pi, size_t(n) * G * es, s));
  MOLR_TRY(b.stage(cl, size_t(n) * G * es, s));
  MOLR_TRY(o.stage(out, size_t(n) * es, s));
  if (is_f64) mol_score_kernel<double><<<ctx->num_sms * 4, 256, 0, s>>>(n, G, a.as<double>(), b.as<double>(), o.as<double>());
  else mol_score_kernel<float><<<ctx->num_sms * 4, 256, 0, s>>>(n, G, a.as<float>(), b.as<float>(), o.as<float>());
  MOLR_LAUNCHED(ctx);
  return finish_outputs(s, {&o});
}

}  // extern "C"
