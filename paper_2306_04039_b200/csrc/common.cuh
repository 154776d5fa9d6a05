// Shared host/device plumbing for libmolr_b200: status handling, UVA staging of host buffers,
// stream-ordered scratch, orderable keys, bf16 helpers.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/molr_b200.h"

namespace molr {

// Development / cross-check switches (alternative backends, pilot sizes, the MoL epilogue trace).
// They exist only in the test build, libmolr_b200_dev.so (-DMOLR_DEV_KNOBS), which the cross-check
// tests load in a subprocess; the production library has one backend per shape and reads no
// environment.
#ifdef MOLR_DEV_KNOBS
inline const char* dev_knob(const char* name) { return getenv(name); }
#else
inline const char* dev_knob(const char*) { return nullptr; }
#endif

// ------------------------------------------------------------------------------------------
// status
// ------------------------------------------------------------------------------------------
void set_error(const std::string& msg);

struct Status {
  int code = MOLR_OK;
  bool ok() const { return code == MOLR_OK; }
};

#define MOLR_FAIL(code_, ...)                                   \
  do {                                                         \
    char _b[512];                                              \
    snprintf(_b, sizeof(_b), __VA_ARGS__);                     \
    ::molr::set_error(_b);                                     \
    return (code_);                                            \
  } while (0)

#define MOLR_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      MOLR_FAIL(MOLR_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                cudaGetErrorString(_e));                                                 \
    }                                                                                    \
  } while (0)

#define MOLR_TRY(expr)            \
  do {                            \
    int _s = (expr);              \
    if (_s != MOLR_OK) return _s; \
  } while (0)

#define MOLR_LAUNCHED(ctx)                                                               \
  do {                                                                                   \
    (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                              \
    cudaError_t _e = cudaGetLastError();                                                 \
    if (_e != cudaSuccess)                                                               \
      MOLR_FAIL(MOLR_ERR_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,                    \
                cudaGetErrorString(_e));                                                 \
  } while (0)

}  // namespace molr

// ------------------------------------------------------------------------------------------
// handles
// ------------------------------------------------------------------------------------------
struct molr_prof_rec {
  const char* name;
  cudaEvent_t start, end;
  double work;  // algorithmic units (bytes or flops) of this launch
};
struct molr_prof_sum {
  int64_t count = 0;
  double ms = 0, work = 0;
};

// Grow-only device workspace for one synchronous entry-point call (see WorkspaceScope).
struct molr_arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  size_t need = 0;  // high-water mark of this call (including what did not fit)
};

struct molr_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::atomic<int64_t> launches{0};
  // per-kernel CUDA-event timing registry (molr_ctx_set_profiling)
  std::atomic<int> prof{0};
  std::mutex prof_mu;
  std::vector<molr_prof_rec> prof_pending;
  std::vector<cudaEvent_t> prof_free;
  std::vector<std::pair<std::string, molr_prof_sum>> prof_sums;
  // workspace arenas: one per concurrently running synchronous call
  std::mutex ws_mu;
  std::vector<molr_arena*> ws_free;
  std::vector<molr_arena*> ws_all;
};

namespace molr {
// RAII launch timer: records CUDA events around the kernel(s) launched in its scope on `s`
// when profiling is enabled.  `work` = algorithmic bytes or flops of the launch.
struct KTimer {
  molr_ctx* ctx;
  const char* name;
  cudaStream_t s;
  double work;
  cudaEvent_t a = nullptr, b = nullptr;
  KTimer(molr_ctx* c, const char* n, cudaStream_t st, double w = 0) : ctx(c), name(n), s(st), work(w) {
    if (!ctx->prof.load(std::memory_order_relaxed)) return;
    {
      std::lock_guard<std::mutex> g(ctx->prof_mu);
      if (ctx->prof_free.size() >= 2) {
        a = ctx->prof_free.back();
        ctx->prof_free.pop_back();
        b = ctx->prof_free.back();
        ctx->prof_free.pop_back();
      }
    }
    if (!a) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
    }
    cudaEventRecord(a, s);
  }
  // end of the timed launches; `work` may still be set afterwards (e.g. once counts are known)
  void stop() {
    if (a && !stopped) cudaEventRecord(b, s);
    stopped = true;
  }
  ~KTimer() {
    if (!a) return;
    stop();
    std::lock_guard<std::mutex> g(ctx->prof_mu);
    ctx->prof_pending.push_back({name, a, b, work});
  }
  bool stopped = false;
};
}  // namespace molr

struct molr_cache {
  molr_ctx* ctx = nullptr;
  int64_t X = 0;
  int k_x = 0, d = 0, G = 0, d1 = 0;
  int storage = 0;                     // molr_storage bits
  __nv_bfloat16* embs_bf16 = nullptr;  // (X, k_x, d) when bf16-exact; see emb_offset (pre-swizzled)
  float* embs_f32 = nullptr;           // (X, k_x, d) otherwise
  __nv_bfloat16* gp_bf16 = nullptr;    // (X, G) when bf16-exact
  float* gp_f32 = nullptr;             // (X, G) otherwise
  float* s1_f32 = nullptr;             // (X, d1)
  int8_t* s1_codes = nullptr;          // (X, d1)
  float* s1_scales = nullptr;          // (X,) (padded like the codes)
  float2* s1_chunk_mm = nullptr;       // per 32-row chunk (1/min, 1/max) of s1_scales (d1 = 64)
  // d1 = 64 int8 view: within every 256-row tile the rows are stored sorted by scale (the cache
  // is "sealed" on first stage-1 use), so each 32-row chunk has a narrow scale range and the
  // tensor-core filter's integer pre-test is tight.  perm: stored position -> item id;
  // inv: item id -> stored position.
  // TMA descriptor over item_embs as (X rows x 1 KB) for tile::gather4 loads (bf16, k_x*d = 512)
  alignas(64) CUtensorMap embs_tmap{};
  int embs_tmap_ok = 0;
  // f32-stored item_embs (not bf16-representable, e.g. a reference-built cache, mol.py:322-324)
  // with k_x * d = 512: a bf16 hi + lo image (x = hi + lo to ~2^-17) in the same pre-swizzled
  // layout, hi rows [0, X) then lo rows [X, 2X), so the tensor-core scorer runs two component
  // passes; TMA descriptors over each half
  __nv_bfloat16* embs_hl = nullptr;
  alignas(64) CUtensorMap embs_hi_tmap{};
  alignas(64) CUtensorMap embs_lo_tmap{};
  int embs_hl_tmap_ok = 0;
  int32_t* s1_perm = nullptr;
  int32_t* s1_inv = nullptr;
  std::atomic<int> s1_sealed{0};
  std::mutex seal_mu;
  // float view on the tensor cores (built lazily from s1_f32, d1 = 64): fp16(view / s1_hscale)
  // (s1_hscale a power of two putting max|v| in [2^14, 2^15)) in the interleaved K-major layout
  // (128 B rows, 256-row tiles), per-row ||v||_2 and per-32-row-chunk max of it, for the pre-test
  // bound of the fp16 MMA against the fp32 score
  __half* s1_bf = nullptr;
  float s1_hscale = 1.f;
  float* s1_bnorm = nullptr;
  float* s1_bnmax = nullptr;
  std::atomic<int> s1_bf_ready{0};
  int64_t bytes = 0;
};

struct molr_gating {
  molr_ctx* ctx = nullptr;
  int G = 0, H = 0, d_u = 0, H_u = 0;
  float* w1 = nullptr;  // (G, H)
  float* b1 = nullptr;  // (H,)
  float* w2 = nullptr;  // (H, G)
  float* uw1 = nullptr; // (d_u, H_u)
  float* ub1 = nullptr;
  float* uw2 = nullptr; // (H_u, G)
  // tensor-core operand images (bf16, K-major, built at creation; see mol_tc.cu)
  __nv_bfloat16* w1t_bf16 = nullptr;  // (H, Kpad) : W1^T with b1 hi/lo folded as extra K rows
  __nv_bfloat16* w2t_bf16 = nullptr;  // (G, H)    : W2^T
};

namespace molr {

// The calling thread's own non-blocking stream on ctx's device (created on first use, destroyed
// at thread exit): calls that pass no stream from different threads run concurrently instead of
// serialising on one shared stream (engine.py:6: "any number of threads, no locks").
cudaStream_t thread_stream(molr_ctx* ctx);

// Every entry point resolves its stream first; clearing any stale non-sticky launch error here
// keeps it from being attributed to this call's launches.
inline cudaStream_t pick_stream(molr_ctx* ctx, void* s) {
  cudaGetLastError();
  return s ? reinterpret_cast<cudaStream_t>(s) : thread_stream(ctx);
}

// True if the kernel can dereference p directly (device or managed memory).
bool is_device_ptr(const void* p);

// The calling thread's active workspace arena (set by WorkspaceScope), or null.
extern thread_local molr_arena* tl_arena;

// Stream-ordered scratch that frees itself.  Inside a WorkspaceScope it is bump-allocated from
// the call's arena (no allocator traffic on the hot path); otherwise cudaMallocAsync.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  bool arena = false;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() { reset(); }
  int alloc(size_t bytes, cudaStream_t stream) {
    reset();
    s = stream;
    if (bytes == 0) bytes = 16;
    const size_t rb = (bytes + 255) & ~size_t(255);
    if (molr_arena* a = tl_arena) {
      a->need = std::max(a->need, a->off + rb);
      if (a->off + rb <= a->cap) {
        p = a->base + a->off;
        a->off += rb;
        arena = true;
        return MOLR_OK;
      }
      a->off += rb;  // account for it so the arena grows to the high-water mark
    }
    cudaError_t e = cudaMallocAsync(&p, bytes, stream);
    if (e != cudaSuccess) {
      p = nullptr;
      set_error(std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
      return MOLR_ERR_CUDA;
    }
    return MOLR_OK;
  }
  void reset() {
    if (p && !arena) cudaFreeAsync(p, s);
    p = nullptr;
    arena = false;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

// RAII: gives the calling thread an arena of `ctx` for the duration of a call that synchronises
// its stream before returning (the arena is recycled at scope exit).  An arena that overflowed is
// regrown at exit to the call's high-water mark, so steady-state calls do no allocation at all.
struct WorkspaceScope {
  molr_ctx* ctx;
  cudaStream_t s;
  molr_arena* a = nullptr;
  molr_arena* prev;
  WorkspaceScope(molr_ctx* c, cudaStream_t st) : ctx(c), s(st), prev(tl_arena) {
    {
      std::lock_guard<std::mutex> g(ctx->ws_mu);
      if (!ctx->ws_free.empty()) {
        a = ctx->ws_free.back();
        ctx->ws_free.pop_back();
      } else {
        a = new molr_arena();
        ctx->ws_all.push_back(a);
      }
    }
    a->off = 0;
    a->need = 0;
    tl_arena = a;
  }
  ~WorkspaceScope() {
    tl_arena = prev;
    cudaStreamSynchronize(s);  // no-op on the normal path; covers early error returns
    if (a->need > a->cap) {  // every user of the old block has completed (the call synchronised)
      if (a->base) cudaFree(a->base);
      const size_t cap = a->need + a->need / 8;
      if (cudaMalloc(&a->base, cap) == cudaSuccess) {
        a->cap = cap;
      } else {
        a->base = nullptr;
        a->cap = 0;
        cudaGetLastError();
      }
    }
    std::lock_guard<std::mutex> g(ctx->ws_mu);
    ctx->ws_free.push_back(a);
  }
};

// Input view: device pointer to `bytes` of data from a host-or-device pointer.
struct In {
  const void* dptr = nullptr;
  Scratch buf;
  int stage(const void* src, size_t bytes, cudaStream_t s) {
    if (src == nullptr || bytes == 0 || is_device_ptr(src)) {
      dptr = src;
      return MOLR_OK;
    }
    int st = buf.alloc(bytes, s);
    if (st) return st;
    cudaError_t e = cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      set_error(std::string("H2D: ") + cudaGetErrorString(e));
      return MOLR_ERR_CUDA;
    }
    dptr = buf.p;
    return MOLR_OK;
  }
  template <class T>
  const T* as() const { return reinterpret_cast<const T*>(dptr); }
};

// Output view: device buffer written by kernels; finish() copies back to a host destination.
struct Out {
  void* user = nullptr;
  void* dptr = nullptr;
  size_t bytes = 0;
  Scratch buf;
  int stage(void* dst, size_t nbytes, cudaStream_t s) {
    user = dst;
    bytes = nbytes;
    if (dst == nullptr || nbytes == 0 || is_device_ptr(dst)) {
      dptr = dst;
      return MOLR_OK;
    }
    int st = buf.alloc(nbytes, s);
    if (st) return st;
    dptr = buf.p;
    return MOLR_OK;
  }
  int finish(cudaStream_t s) {
    if (dptr != user && user != nullptr && bytes) {
      cudaError_t e = cudaMemcpyAsync(user, dptr, bytes, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) {
        set_error(std::string("D2H: ") + cudaGetErrorString(e));
        return MOLR_ERR_CUDA;
      }
    }
    return MOLR_OK;
  }
  bool host() const { return dptr != user; }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(dptr); }
};

// Synchronise when any output lives in host memory (the call must return with it filled).
int finish_outputs(cudaStream_t s, std::initializer_list<Out*> outs);

// ------------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------------
// Monotone map float -> uint32: a < b (as floats, no NaN) <=> key(a) < key(b).
__host__ __device__ __forceinline__ uint32_t f32_key(float f) {
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(f);
#else
  memcpy(&u, &f, 4);
#endif
  if (u == 0x80000000u) u = 0u;  // -0 == +0 as floats: same key
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float key_f32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(u);
#else
  memcpy(&f, &u, 4);
#endif
  return f;
}
__host__ __device__ __forceinline__ uint32_t i32_key(int32_t v) { return uint32_t(v) ^ 0x80000000u; }
__host__ __device__ __forceinline__ int32_t key_i32(uint32_t k) { return int32_t(k ^ 0x80000000u); }

__device__ __forceinline__ float silu_f32(float x) {
  // x * sigmoid(x) with full-precision expf (reference: x * scipy.special.expit(x))
  return x / (1.0f + expf(-x));
}

// bf16 item-component blocks with d = 64 (128-byte rows) and k_x % 8 == 0 are stored in the
// UMMA K-major SWIZZLE_128B atom order: the 16-byte chunk c of component row b sits at chunk
// position c ^ (b % 8).  One 1 KB bulk copy of an item (k_x = 8) into a 1024-aligned shared slot
// is then a ready tcgen05 operand (8 rows x 64 K).  Offset (elements) of (b, k) within an item:
__host__ __device__ __forceinline__ int emb_offset(int b, int k, int d, bool swz) {
  return swz ? b * d + ((((k >> 3) ^ (b & 7)) << 3) | (k & 7)) : b * d + k;
}
__host__ __device__ __forceinline__ bool emb_swizzled(int k_x, int d) { return d == 64 && (k_x % 8) == 0; }

// Stage-1 int8 codes with d1 = 64 are stored in the tcgen05 K-major "interleave" (no-swizzle)
// layout: blocks of 8 rows x 64 B = 512 B, each block ordered [16-byte K chunk c][row r%8][16 B],
// so a bulk copy of 256 consecutive rows (16 KB) is directly an MMA operand (LBO 128 B, SBO
// 512 B).  Rows are padded to a multiple of 256 (zero codes, zero scales).  Byte offset of 16-byte
// chunk c of row r:
__host__ __device__ __forceinline__ bool s1_interleaved(int d1) { return d1 == 64; }
__host__ __device__ __forceinline__ int64_t s1_chunk_offset(int64_t r, int c, int d1) {
  return d1 == 64 ? ((r >> 3) << 9) + (int64_t(c) << 7) + ((r & 7) << 4) : r * d1 + int64_t(c) * 16;
}
__host__ __device__ __forceinline__ int64_t s1_rows_alloc(int64_t X, int d1) {
  return d1 == 64 ? (X + 255) / 256 * 256 : X;
}

// The reference's float stage-1 score is NumPy's `view @ q` (hindexer.py:112), i.e. OpenBLAS sgemv.
// Its summation order on the reference host (OpenBLAS 0.3.30 SkylakeX kernels; the GPU box reports
// the same, tools/blas_order_probe.py) for rows inside sgemv's 4-row blocks is reproduced exactly:
//   d % 8 == 0 and d >= 16: four lanes and two accumulators taking alternate 4-element blocks
//     (fused multiply-add), lanes combined (acc0 + acc1), then (l0 + l1) + (l2 + l3);
//   d == 8: rounded products, ((p0 + p1) + (p2 + p3)) + ((p4 + p5) + (p6 + p7));
//   d == 4: (p0 + p1) + (p2 + p3);
//   other d: the sequential fmaf chain (within fp32 summation-order tolerance of the reference).
// (OpenBLAS scores the last X % 4 rows of a matrix with another kernel; those rows agree only to
// within summation-order tolerance.)
__device__ __forceinline__ float s1_dot_f32(const float* __restrict__ v, const float* __restrict__ q, int d) {
  if (d >= 16 && (d & 7) == 0) {
    float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < d; k += 8) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        a0[l] = fmaf(v[k + l], q[k + l], a0[l]);
        a1[l] = fmaf(v[k + 4 + l], q[k + 4 + l], a1[l]);
      }
    }
    const float t0 = a0[0] + a1[0], t1 = a0[1] + a1[1], t2 = a0[2] + a1[2], t3 = a0[3] + a1[3];
    return (t0 + t1) + (t2 + t3);
  }
  if (d == 8) {
    float p[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = __fmul_rn(v[k], q[k]);
    return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
  }
  if (d == 4) return (__fmul_rn(v[0], q[0]) + __fmul_rn(v[1], q[1])) + (__fmul_rn(v[2], q[2]) + __fmul_rn(v[3], q[3]));
  float acc = 0.f;
  for (int k = 0; k < d; ++k) acc = fmaf(v[k], q[k], acc);
  return acc;
}

// d = 64 with the row already in registers (same order as s1_dot_f32)
__device__ __forceinline__ float s1_dot64(const float (&v)[64], const float* __restrict__ q) {
  float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 64; k += 8) {
    const float4 x = *reinterpret_cast<const float4*>(q + k), y = *reinterpret_cast<const float4*>(q + k + 4);
    a0[0] = fmaf(v[k], x.x, a0[0]);
    a0[1] = fmaf(v[k + 1], x.y, a0[1]);
    a0[2] = fmaf(v[k + 2], x.z, a0[2]);
    a0[3] = fmaf(v[k + 3], x.w, a0[3]);
    a1[0] = fmaf(v[k + 4], y.x, a1[0]);
    a1[1] = fmaf(v[k + 5], y.y, a1[1]);
    a1[2] = fmaf(v[k + 6], y.z, a1[2]);
    a1[3] = fmaf(v[k + 7], y.w, a1[3]);
  }
  const float t0 = a0[0] + a1[0], t1 = a0[1] + a1[1], t2 = a0[2] + a1[2], t3 = a0[3] + a1[3];
  return (t0 + t1) + (t2 + t3);
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

inline int div_up(int64_t a, int64_t b) { return int((a + b - 1) / b); }

}  // namespace molr
