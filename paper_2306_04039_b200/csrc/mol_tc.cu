// Fused MoL scorer on the 5th-gen tensor cores (tcgen05 + TMEM), production shape
// k_u = k_x = 8, d = 64, G = k_u * k_x = 64, H = 128 — score_candidates / batch_score_all /
// mol_top_k's scoring (mol.py:139-205, 329-386).
//
// One persistent CTA per SM, warp-specialised:
//   warp 0       producer: per tile, the query's pre-built B0 operand (2 KB) into a small ring, and
//                per candidate one 1 KB cp.async.bulk of the item's component block (the cache
//                stores it pre-swizzled, see emb_offset) into a ring of 16-item stages
//   warp 1       MMA issuer (one thread, non-blocking state machine) + TMEM owner
//   warps 2..9   two epilogue warpgroups; tile k belongs to group k % 2
// TMEM (512 columns): D0 = cols [0,128) is ONE buffer shared by both groups: the component
// GEMM streams through it tile after tile (it only waits for the previous tile's E0 to drain it),
// so the item ring is consumed continuously and the gather never stalls on an epilogue.
// Group g owns cols [128 + 192 g, 320 + 192 g): A1 then A2 (64 cols) and D1 then D2 (128 cols).
// Per tile of 128 (query, candidate) pairs of ONE query:
//   C : 8 x [M=128 rows = 16 items x 8 components] x [N=16 = (hi,lo) x 8 user components] x K=64
//       (SS) -> D0.  Query side split u = hi + lo in bf16 (~2^-17 relative), item side exact
//       bf16, fp32 accumulation.
//   E0: D0 -> (hi+lo)/tau -> fp32 logits, transposed to one row per pair in the group's smem CL
//       (kept there for the final gated sum); D0 released
//   E0.5: row p -> A1 = the logits split in bf16 hi + lo, packed two per column (the A operand
//       of layer 1, from TMEM: hi in group cols [0,32), lo in [32,64))
//   L1: A1_hi . W1_hi + A1_lo . W1_hi + A1_hi . W1_lo (TMEM x smem, three passes: ~2^-16
//       relative) + [1 1 0..] . [b1_hi b1_lo 0..]^T (SS, K=16) -> D1
//   E1: h = silu(D1) (ex2 + rcp) -> A2 = h split in fp16 hi + lo (hi over the dead A1, lo over
//       D1 columns this warp has already read)
//   L2: A2_hi . W2_hi + A2_lo . W2_hi + A2_hi . W2_lo (fp16, three passes: ~2^-21) -> D2
//   E2: pi = softmax(silu(uw * gate_pre + D2)); score = sum pi * CL  -> global
// The cross net runs at ~fp32 accuracy: a single bf16 / fp16 pass and a tanh.approx SiLU gave
// score errors above the 1e-3 |s| + 1e-6 tolerance once the cross net is sharpened x16
// (tests/test_gpu_parity.py::test_tc_kernel_precision_margin, emulated in tools/precision_emu.py).
// The G logits and H hidden units never leave the SM.
#include <algorithm>
#include <vector>
#include <cstdlib>

#include <cuda_fp16.h>

#include "kernels.cuh"
#include "stage1.cuh"

namespace molr {
namespace tc {

constexpr int KX = 8, D = 64, G = 64, H = 128;
constexpr int TILE = 128;           // pairs per tile (MMA M)
constexpr int GROUP = 16;           // items per component MMA (16 items x 8 rows = 128)
constexpr int NGROUPS = TILE / GROUP;
#ifndef MOL_NSTAGE
#define MOL_NSTAGE 5
#endif
// (MOL_FAST / MOL_NSTAGE: timing experiments only — single-pass cross net; not built by the Makefile)
constexpr int NSTAGE = MOL_NSTAGE;  // ring stages (16 KB each): 80 KB of item blocks in flight per SM
constexpr int NE = 2;               // epilogue groups
constexpr int CL_LD = 68;           // fp32 row stride of the logit transpose buffer (conflict-free LDS.128)

// ---- shared memory map (bytes; regions holding MMA operands are 1024-aligned) --------------
constexpr int SZ_STAGE = GROUP * 1024;                  // 16 KB
constexpr int OFF_RING = 0;
constexpr int OFF_W1T = OFF_RING + NSTAGE * SZ_STAGE;   // 128 x 64 bf16, SW128      16 KB
constexpr int OFF_W2T = OFF_W1T + 16384;                // 2 x (64 x 64) fp16, SW128 16 KB
#ifdef MOL_FAST
constexpr int SZ_LO = 0;
#else
constexpr int SZ_LO = 16384;
#endif
constexpr int OFF_W1TL = OFF_W2T + 16384;               // W1 lo parts, as W1T        16 KB
constexpr int OFF_W2TL = OFF_W1TL + SZ_LO;              // W2 lo parts, as W2T        16 KB
constexpr int OFF_W1B = OFF_W2TL + SZ_LO;               // 128 x 16 bf16, interleave  4 KB
constexpr int OFF_BIASA = OFF_W1B + 4096;               // 128 x 16 bf16, interleave  4 KB
constexpr int NB0 = 3;                                  // B0 (query operand) ring slots
constexpr int OFF_B0 = OFF_BIASA + 4096;                // NB0 x 16 x 64 bf16 SW128 (u_hi ; u_lo), 2 KB each
constexpr int OFF_GRP = OFF_B0 + NB0 * 2048;            // per epilogue group:
constexpr int G_CL = 0;                                 //   fp32 logits [128 x 68]        34 KB
constexpr int G_UW = G_CL + TILE * CL_LD * 4;           //   64 f32
constexpr int SZ_GRP = G_UW + 256;
constexpr int OFF_BAR = OFF_GRP + NE * SZ_GRP;
// barriers: full[NSTAGE], empty[NSTAGE], b0full[NB0], b0empty[NB0], d0free,
//           then per group: d0_full, a1_ready, d1_full, a2_ready, d2_full
constexpr int NBAR = 2 * NSTAGE + 2 * NB0 + 1 + 5 * NE;
constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");
constexpr int TM_D0 = 0;                                // shared component-logit accumulator
__host__ __device__ constexpr int tm_grp(int g) { return 128 + 192 * g; }  // A1/A2 at +0, D1 at +64, D2 at +96
// group column of A2_lo's hidden chunk ch (8 packed columns): inside D1 columns its warp has read
// (warp half 0 reads D1 chunks 0..3 in order, half 1 chunks 7..4 in reverse), clear of D2 = D1 [32, 96)
__host__ __device__ constexpr int a2lo_col(int ch) { return 64 + (ch < 4 ? 8 * ch : 64 + 8 * ch); }
constexpr int TM_D2 = 96;

// ---- PTX wrappers ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// tile::gather4: rows r0..r3 (1 KB each) of a [rows][256 x u32] tensor map -> 4 KB of smem
__device__ __forceinline__ void gather4_g2s(uint32_t dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// SW128 K-major descriptor: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// no-swizzle ("interleave") K-major descriptor: core matrices 8 rows x 16 B; LBO = K stride, SBO = M stride
__device__ __forceinline__ uint64_t desc_interleave(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46);
}
// kind::f16 instruction descriptor: A = B = bf16, D = f32, both K-major, M = 128
// kind::f16 instruction descriptor: A = B = fp16, D = f32, both K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
// A operand from TMEM (packed bf16 pairs per 32-bit column, row m = lane m), B from smem
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define TMEM_LD16(taddr, r)                                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
                 "=r"(r[15])                                                                                       \
               : "r"(taddr))
#define TMEM_ST16(taddr, r)                                                                                        \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))
#define TMEM_ST8(taddr, r)                                                                                  \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),   \
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x = lo (low 16 bits), .y = hi
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);  // .x = lo (low 16 bits), .y = hi
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// The cross net and the combine run in "log2 units": layer 1's weights and bias, and uw, carry a
// factor -log2(e) (folded into the weight images / the per-query uw load), so with x' = -log2(e) x
//   sigmoid(x) = 1 / (1 + 2^x'),  -log2(e) silu(x) = x' / (1 + 2^x')
// and the hidden units h' = -log2(e) h make layer 2 return -log2(e) D2 with W2 unchanged.  One
// ex2 + one rcp per SiLU (~1e-7 relative), no scaling multiplies.
__device__ __forceinline__ float silu_l2(float xs) { return xs * rcp(1.0f + ex2(xs)); }

// SW128 K-major byte offset of 16-byte chunk `c` of row `r` within a [rows x 128 B] region.
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4); }
// interleave (no-swizzle) K-major offset of chunk c (0/1) of row r, LBO = 128, SBO = 256.
__device__ __forceinline__ uint32_t ilv(int r, int c) { return (r >> 3) * 256 + c * 128 + (r & 7) * 16; }

// Walks a CTA's strided tile sequence; the query cursor only moves forward (tiles of one query
// are contiguous in the global tile order), so locating a tile costs O(1) amortised loads.
struct TileCursor {
  int b = 0;
  __device__ __forceinline__ void seek(int64_t tile, int B, const int64_t* __restrict__ pre) {
    while (b + 1 < B && __ldg(pre + b + 1) <= tile) ++b;
  }
};

struct TileInfo {
  int b;
  int64_t seg0, j0;
  int np;
};

__device__ __forceinline__ TileInfo tile_info(TileCursor& cur, int64_t tile, int B, const int64_t* __restrict__ pre,
                                              const int64_t* __restrict__ begin, const int64_t* __restrict__ end,
                                              int64_t X) {
  cur.seek(tile, B, pre);
  TileInfo t;
  t.b = cur.b;
  t.seg0 = begin ? __ldg(begin + t.b) : 0;
  const int64_t len = begin ? __ldg(end + t.b) - t.seg0 : X;
  t.j0 = (tile - __ldg(pre + t.b)) * TILE;
  t.np = (int)imin64(TILE, len - t.j0);
  return t;
}

template <class Id>
__device__ __forceinline__ int64_t cand_id(const Id* __restrict__ ids, const TileInfo& t, int q) {
  return ids ? (int64_t)__ldg(ids + t.seg0 + t.j0 + q) : t.j0 + q;
}

struct Params {
  int B;
  float inv_tau;
  const __nv_bfloat16* embs;  // (X, 8, 64) pre-swizzled item blocks (the hi image of an f32 cache)
  const __nv_bfloat16* embs_lo;  // hl: the lo image (x = hi + lo), same layout
  int hl;                     // f32 cache: two component passes (hi, lo) per item group
  const __nv_bfloat16* gp;    // (X, 64) bf16, or null when gpf is set
  const float* gpf;           // (X, 64) f32 gate pre-activations (f32-stored cache)
  const __nv_bfloat16* w1t;   // SW128 image (16 KB)
  const __nv_bfloat16* w2t;   // SW128 image (16 KB), followed by the residual image (16 KB)
  const __nv_bfloat16* w1b;   // interleave image (4 KB)
  const __nv_bfloat16* w1tl;  // SW128 image of the W1 lo parts (16 KB)
  const __nv_bfloat16* w2tl;  // SW128 image of the W2 lo parts (16 KB)
  const float* user_embs;     // (B, 8, 64)
  const float* uw;            // (B, 64)
  const int64_t* begin;
  const int64_t* end;
  int64_t X;
  const int64_t* tile_pre;
  const uint8_t* b0img;       // (B, 2048) per-query B0 operand images (b0_image_kernel)
  float* out;
  int64_t out_ld;
  unsigned long long* trace;  // dev tool (MOLR_TRACE_MOL): CTA 0 epilogue timeline, else null
  int gather4;  // item fetch by TMA tile::gather4 (4 items per request) instead of 1 KB bulk copies
};

template <class Id, bool GPF>
__global__ void __launch_bounds__(64 + NE * 256 + 32 * NE, 1) mol_tc_kernel(Params P, const Id* __restrict__ ids,
                                                                  const __grid_constant__ CUtensorMap tmap,
                                                                  const __grid_constant__ CUtensorMap tmap_lo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t sbase = smem_u32(sm);
  if ((sbase & 1023u) != 0u) __trap();  // SW128 operands need 1024-aligned atoms
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto bar = [&](int i) { return sbase + OFF_BAR + 8 * i; };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(NSTAGE + s); };
  auto b0full = [&](int s) { return bar(2 * NSTAGE + s); };
  auto b0empty = [&](int s) { return bar(2 * NSTAGE + NB0 + s); };
  const uint32_t d0free = bar(2 * NSTAGE + 2 * NB0);
  // k: 0 d0_full 1 a1_ready 2 d1_full 3 a2_ready 4 d2_full
  auto gbar = [&](int g, int k) { return bar(2 * NSTAGE + 2 * NB0 + 1 + 5 * g + k); };

  // ---- one-time setup: weight images + constant bias operand, barriers, TMEM ----
  {
    const uint4* src1 = reinterpret_cast<const uint4*>(P.w1t);
    const uint4* src2 = reinterpret_cast<const uint4*>(P.w2t);
    const uint4* src3 = reinterpret_cast<const uint4*>(P.w1b);
    const uint4* src4 = reinterpret_cast<const uint4*>(P.w1tl);
    const uint4* src5 = reinterpret_cast<const uint4*>(P.w2tl);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
      reinterpret_cast<uint4*>(sm + OFF_W1T)[i] = __ldg(src1 + i);
      reinterpret_cast<uint4*>(sm + OFF_W2T)[i] = __ldg(src2 + i);
      if (SZ_LO) {
        reinterpret_cast<uint4*>(sm + OFF_W1TL)[i] = __ldg(src4 + i);
        reinterpret_cast<uint4*>(sm + OFF_W2TL)[i] = __ldg(src5 + i);
      }
    }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) reinterpret_cast<uint4*>(sm + OFF_W1B)[i] = __ldg(src3 + i);
    // bias A operand: K columns 0 and 1 of every row = 1.0 (pairs with the b1 hi / lo rows of W1B)
    for (int r = threadIdx.x; r < TILE; r += blockDim.x) {
      *reinterpret_cast<uint4*>(sm + OFF_BIASA + ilv(r, 0)) = make_uint4(0x3F803F80u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sm + OFF_BIASA + ilv(r, 1)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (threadIdx.x == 0) {
      for (int s = 0; s < NSTAGE; ++s) {
        mbar_init(full_bar(s), 1);
        mbar_init(empty_bar(s), 1);
      }
      for (int s = 0; s < NB0; ++s) {
        mbar_init(b0full(s), 1);
        mbar_init(b0empty(s), 1);
      }
      mbar_init(d0free, 256);
      for (int g = 0; g < NE; ++g) {
        mbar_init(gbar(g, 0), 1);
        mbar_init(gbar(g, 1), 256);
        mbar_init(gbar(g, 2), 1);
        mbar_init(gbar(g, 3), 256);
        mbar_init(gbar(g, 4), 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem_base = *tmem_slot;
  const int64_t T = P.tile_pre[P.B];

  if (warp == 0) {
    // ================= producer: B0 image + item blocks -> rings =================
    int stage = 0, slot = 0;
    uint32_t phase = 0, bphase = 0;
    TileCursor cur;
    for (int64_t tile = blockIdx.x; tile < T; tile += gridDim.x) {
      const TileInfo t = tile_info(cur, tile, P.B, P.tile_pre, P.begin, P.end, P.X);
      // the tile's 128 candidate ids, 4 per lane (q = lane + 32 i); padding rows reuse row 0
      int64_t xid[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = lane + 32 * i;
        xid[i] = cand_id(ids, t, q < t.np ? q : 0);
      }
      mbar_wait(b0empty(slot), bphase ^ 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(b0full(slot), 2048);
        bulk_g2s(sbase + OFF_B0 + slot * 2048, P.b0img + int64_t(t.b) * 2048, 2048, b0full(slot));
      }
      if (++slot == NB0) {
        slot = 0;
        bphase ^= 1;
      }
#pragma unroll
      for (int g = 0; g < NGROUPS; ++g) {
        const int64_t x = __shfl_sync(0xffffffffu, xid[g >> 1], 16 * (g & 1) + (lane & 15));
        for (int part = 0; part <= P.hl; ++part) {  // f32 cache: the group's hi blocks, then its lo blocks
          mbar_wait(empty_bar(stage), phase ^ 1);
          if (lane == 0) mbar_arrive_expect_tx(full_bar(stage), SZ_STAGE);
          __syncwarp();
          if (P.gather4) {  // 4 items (4 KB) per TMA request: lane l < 4 fetches items 4l .. 4l+3
            const int r0 = __shfl_sync(0xffffffffu, int(x), (4 * lane) & 15), r1 = __shfl_sync(0xffffffffu, int(x), (4 * lane + 1) & 15);
            const int r2 = __shfl_sync(0xffffffffu, int(x), (4 * lane + 2) & 15), r3 = __shfl_sync(0xffffffffu, int(x), (4 * lane + 3) & 15);
            if (lane < 4)
              gather4_g2s(sbase + OFF_RING + stage * SZ_STAGE + lane * 4096, part ? &tmap_lo : &tmap, r0, r1, r2, r3, full_bar(stage));
          } else if (lane < GROUP) {
            bulk_g2s(sbase + OFF_RING + stage * SZ_STAGE + lane * 1024, (part ? P.embs_lo : P.embs) + x * (KX * D), 1024,
                     full_bar(stage));
          }
          __syncwarp();
          if (++stage == NSTAGE) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread, never blocks on a single barrier) =================
    if (lane == 0) {
      constexpr uint32_t ID16 = idesc_bf16(16), ID128 = idesc_bf16(128), ID64 = idesc_bf16(64);
      int stage = 0, slot = 0;
      uint32_t rphase = 0, bphase = 0;
      // component stream: local tile kc (ring order), 8 stage groups each
      int64_t ctile = blockIdx.x;
      int64_t kc = 0;
      int cgrp = -1;  // -1: waiting for D0 free + B0
      int cpart = 0;  // f32 cache: 0 = the group's hi blocks, 1 = its lo blocks (accumulated)
      // per epilogue group chain: state 0 need L1 (a1_ready), 1 need L2 (a2_ready); use count
      int gstate[NE];
      uint32_t guse[NE];
      int64_t gk[NE];  // local tile index the group is on (its m-th tile: k = 2 m + g)
#pragma unroll
      for (int g = 0; g < NE; ++g) {
        gstate[g] = 0;
        guse[g] = 0;
        gk[g] = g;
      }
      const int64_t my_tiles = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      while (kc < my_tiles) {
        // ---- component GEMM stream ----
        if (kc < my_tiles) {
          if (cgrp < 0) {
            // D0 drained by the previous tile's E0, and this tile's query operand landed
            if ((kc == 0 || mbar_test(d0free, uint32_t((kc - 1) & 1))) && mbar_test(b0full(slot), bphase)) {
              tc_fence_after();
              cgrp = 0;
            }
          }
          if (cgrp >= 0) {
            const uint32_t b0 = sbase + OFF_B0 + slot * 2048;
            while (cgrp < NGROUPS && mbar_test(full_bar(stage), rphase)) {
              tc_fence_after();
              const uint32_t a0 = sbase + OFF_RING + stage * SZ_STAGE;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16(tmem_base + TM_D0 + cgrp * 16, desc_sw128(a0 + kk * 32), desc_sw128(b0 + kk * 32), ID16,
                         (kk > 0 || cpart > 0) ? 1u : 0u);
              mma_commit(empty_bar(stage));
              if (++stage == NSTAGE) {
                stage = 0;
                rphase ^= 1;
              }
              if (cpart < P.hl) {
                ++cpart;
              } else {
                cpart = 0;
                ++cgrp;
              }
            }
            if (cgrp == NGROUPS) {
              mma_commit(gbar(int(kc & 1), 0));  // D0 of local tile kc complete -> group kc % 2
              mma_commit(b0empty(slot));
              if (++slot == NB0) {
                slot = 0;
                bphase ^= 1;
              }
              ++kc;
              ctile += gridDim.x;
              cgrp = -1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 2 + 8 * NE) {
    // ================= cross-net issuers: one thread per epilogue group =================
    // blocking waits (the thread sleeps until its group's A operand is ready), so each handoff
    // costs one barrier wake-up rather than a poll of every stream
    const int g = warp - (2 + 8 * NE);
    if (lane == 0) {
      constexpr uint32_t ID128 = idesc_bf16(128), ID64 = idesc_bf16(64);
      const uint32_t tg = tmem_base + tm_grp(g);
      const int64_t my_tiles = T > blockIdx.x ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      uint32_t up = 0;
      for (int64_t k = g; k < my_tiles; k += NE, up ^= 1) {
        mbar_wait(gbar(g, 1), up);  // A1 stored by the group
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // A1_hi . W1_hi + A1_lo . W1_hi + A1_hi . W1_lo
          mma_bf16_ts(tg + 64, tg + kk * 8, desc_sw128(sbase + OFF_W1T + kk * 32), ID128, kk > 0);
          if (SZ_LO) {
            mma_bf16_ts(tg + 64, tg + 32 + kk * 8, desc_sw128(sbase + OFF_W1T + kk * 32), ID128, 1);
            mma_bf16_ts(tg + 64, tg + kk * 8, desc_sw128(sbase + OFF_W1TL + kk * 32), ID128, 1);
          }
        }
        mma_bf16(tg + 64, desc_interleave(sbase + OFF_BIASA, 128, 256), desc_interleave(sbase + OFF_W1B, 128, 256),
                 ID128, 1);
        mma_commit(gbar(g, 2));
        mbar_wait(gbar(g, 3), up);  // A2 (SiLU hidden, fp16) stored by the group
        tc_fence_after();
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {  // hidden K [16ch, 16ch+16): A2_hi cols [8ch, 8ch+8), A2_lo a2lo_col(ch)
          const uint32_t bo = (ch >> 2) * 8192 + (ch & 3) * 32;
          mma_bf16_ts(tg + TM_D2, tg + ch * 8, desc_sw128(sbase + OFF_W2T + bo), idesc_f16(64), ch > 0);
          if (SZ_LO) {
            mma_bf16_ts(tg + TM_D2, tg + a2lo_col(ch), desc_sw128(sbase + OFF_W2T + bo), idesc_f16(64), 1);
            mma_bf16_ts(tg + TM_D2, tg + ch * 8, desc_sw128(sbase + OFF_W2TL + bo), idesc_f16(64), 1);
          }
        }
        mma_commit(gbar(g, 4));
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue groups: 8 warps each =================
    // Group eg = warps 2+8eg .. 9+8eg.  Warp w of a group reads TMEM lane quarter w & 3 (its
    // tile rows p) and column half hf = w >> 2 of every phase, so each SMSP runs four epilogue
    // warps and each phase is half as long; the two halves of a row exchange the softmax max and
    // partial sums through the spare columns 64..67 of the row's CL line.
    const int eg = (warp - 2) >> 3;
    const int hf = ((warp - 2) >> 2) & 1;    // column half
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int p = quarter * 32 + lane;       // tile row = TMEM lane
    uint8_t* gs = sm + OFF_GRP + eg * SZ_GRP;
    float* CL = reinterpret_cast<float*>(gs + G_CL);
    float* UW = reinterpret_cast<float*>(gs + G_UW);
    float* XR = CL + p * CL_LD + 64;         // row p's exchange slots: [max h0, max h1, sum h1, acc h1]
    const uint32_t lq = (uint32_t)(quarter * 32) << 16;
    const uint32_t td0 = tmem_base + TM_D0 + lq;
    const uint32_t tg = tmem_base + tm_grp(eg) + lq;
    const int bar_id = 1 + eg;
    constexpr int NT = 256;                  // threads per group
    uint32_t ph = 0;
#ifndef MOLR_DEV_KNOBS
#define TRACE(tag)
#else
#define TRACE(tag)                                                                                     \
  if (P.trace && blockIdx.x == 0 && p == 0 && hf == 0) {                                               \
    unsigned long long c;                                                                              \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));                                                  \
    const unsigned long long i = atomicAdd(P.trace, 1ull);                                             \
    if (i < 65535) P.trace[1 + i] = (uint64_t(eg * 16 + (tag)) << 56) | (c & ((1ull << 56) - 1));      \
  }
#endif
    TileCursor cur;
    for (int64_t tile = blockIdx.x + (int64_t)eg * gridDim.x; tile < T; tile += (int64_t)NE * gridDim.x) {
      const TileInfo t = tile_info(cur, tile, P.B, P.tile_pre, P.begin, P.end, P.X);
      if (hf == 0 && p < G) UW[p] = -1.4426950408889634f * __ldg(P.uw + (int64_t)t.b * G + p);  // log2 units
      uint4 gpr[4];
      const int64_t xrow = cand_id(ids, t, p < t.np ? p : 0);
      // this row's gate pre-activations into L1 now, read in E2 (holding them in registers through
      // the tile spilled)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(GPF ? (const void*)(P.gpf + xrow * G + hf * 32) : (const void*)(P.gp + xrow * G + hf * 32)));
      // ---- E0: component logits (shared D0) -> CL (transpose to one row per pair); free D0 ----
      TRACE(0);
      mbar_wait(gbar(eg, 0), ph);
      TRACE(1);
      tc_fence_after();
#pragma unroll
      for (int gi = 0; gi < NGROUPS / 2; gi += 2) {
        const int grp = hf * (NGROUPS / 2) + gi;
        uint32_t v[16], w[16];
        TMEM_LD16(td0 + grp * 16, v);
        TMEM_LD16(td0 + grp * 16 + 16, w);
        tmem_wait_ld();
        const int q = grp * GROUP + (p >> 3), bb = p & 7;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          CL[q * CL_LD + a * 8 + bb] = (__uint_as_float(v[a]) + __uint_as_float(v[8 + a])) * P.inv_tau;
          CL[(q + GROUP) * CL_LD + a * 8 + bb] = (__uint_as_float(w[a]) + __uint_as_float(w[8 + a])) * P.inv_tau;
        }
      }
      tc_fence_before();
      mbar_arrive(d0free);  // the next tile's component GEMM may overwrite D0
      TRACE(2);
      named_sync(bar_id, NT);
      // ---- E0.5: row p, logits [32 hf, 32 hf + 32) -> A1 (bf16 pairs, group cols [16 hf, 16 hf + 16)) ----
      {
        const float4* row = reinterpret_cast<const float4*>(CL + p * CL_LD + 32 * hf);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t a1[8], a1l[8];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const float4 x = row[h * 4 + m];
            a1[2 * m] = pack_bf16(x.x, x.y);
            a1[2 * m + 1] = pack_bf16(x.z, x.w);
            a1l[2 * m] = pack_bf16(x.x - bf16_lo(a1[2 * m]), x.y - bf16_hi(a1[2 * m]));
            a1l[2 * m + 1] = pack_bf16(x.z - bf16_lo(a1[2 * m + 1]), x.w - bf16_hi(a1[2 * m + 1]));
          }
          TMEM_ST8(tg + 16 * hf + h * 8, a1);
          TMEM_ST8(tg + 32 + 16 * hf + h * 8, a1l);
        }
        tmem_wait_st();
      }
      tc_fence_before();
      mbar_arrive(gbar(eg, 1));
      TRACE(3);
      {  // while L1 runs: pull the next tile's candidate id and gate row into L1 (the dependent
         // metadata loads otherwise sit on the critical path between this tile's E2 and the next)
        const int64_t nt = tile + (int64_t)NE * gridDim.x;
        if (nt < T) {
          TileCursor c2 = cur;
          const TileInfo u = tile_info(c2, nt, P.B, P.tile_pre, P.begin, P.end, P.X);
          const int64_t xn = cand_id(ids, u, p < u.np ? p : 0);
          if (GPF) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.gpf + xn * G + hf * 32));
          else asm volatile("prefetch.global.L1 [%0];" ::"l"(P.gp + xn * G + hf * 32));
          if (hf == 0 && p < G) asm volatile("prefetch.global.L1 [%0];" ::"l"(P.uw + (int64_t)u.b * G + p));
        }
      }
      // ---- E1: h = silu(D1) -> A2 (fp16 pairs, group cols [32 hf, 32 hf + 32)), hidden chunks [4 hf, 4 hf + 4) ----
      mbar_wait(gbar(eg, 2), ph);
      TRACE(4);
      tc_fence_after();
      {
        // warp half 0 walks hidden chunks 0..3, half 1 chunks 7..4, so the A2_lo columns it writes
        // (a2lo_col) are always D1 columns it has already read
        uint32_t va[16], vb[16];
        const int ch0 = hf ? 7 : 0, dch = hf ? -1 : 1;
        TMEM_LD16(tg + 64 + ch0 * 16, va);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int ch = ch0 + dch * c4;
          uint32_t* v = (c4 & 1) ? vb : va;
          tmem_wait_ld();
          if (c4 < 3) {  // next chunk loads under this chunk's SiLU
            if (c4 & 1) TMEM_LD16(tg + 64 + (ch + dch) * 16, va);
            else TMEM_LD16(tg + 64 + (ch + dch) * 16, vb);
          }
          uint32_t w[8], wl[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            const float x0 = __uint_as_float(v[2 * m]), x1 = __uint_as_float(v[2 * m + 1]);
            const float h0 = silu_l2(x0), h1 = silu_l2(x1);  // -log2(e) silu(D1)
            const __half2 hh = __floats2half2_rn(h0, h1);
            const float2 hb = __half22float2(hh);
            w[m] = *reinterpret_cast<const uint32_t*>(&hh);
            wl[m] = pack_f16(h0 - hb.x, h1 - hb.y);
          }
          TMEM_ST8(tg + ch * 8, w);  // A2_hi, two per column (A1 is dead: L1 has completed)
          TMEM_ST8(tg + a2lo_col(ch), wl);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(gbar(eg, 3));
      TRACE(5);
      // ---- E2: combine + softmax + gated sum over gates [32 hf, 32 hf + 32), halves merged ----
      mbar_wait(gbar(eg, 4), ph);
      TRACE(6);
      tc_fence_after();
      // pre = silu(x), x = uw gate_pre + D2 (mol.py:186-193); t = x' sigmoid(x) = -log2(e) pre, so the
      // softmax is 2^(min t - t) / sum
      float pre[32];
      float mx = INFINITY;
      {
        uint32_t v0[16], v1[16];
        TMEM_LD16(tg + TM_D2 + 32 * hf, v0);
        TMEM_LD16(tg + TM_D2 + 32 * hf + 16, v1);
        tmem_wait_ld();
        // GPF (f32 cache): the row, prefetched into L1 during the previous tile
        const float4* gsrc = GPF ? reinterpret_cast<const float4*>(P.gpf + xrow * G + 32 * hf) : nullptr;
        if (!GPF) {
          const uint4* src = reinterpret_cast<const uint4*>(P.gp + xrow * G) + hf * 4;
#pragma unroll
          for (int m = 0; m < 4; ++m) gpr[m] = __ldg(src + m);
        }
#pragma unroll
        for (int m = 0; m < 32; ++m) {
          const int g = 32 * hf + m;
          float gpv;
          if (GPF) {
            const float4 g4 = __ldg(gsrc + (m >> 2));
            gpv = (m & 3) == 0 ? g4.x : (m & 3) == 1 ? g4.y : (m & 3) == 2 ? g4.z : g4.w;
          } else {
            const uint32_t wv = (&gpr[m >> 3].x)[(m & 7) >> 1];
            gpv = __uint_as_float((m & 1) ? (wv & 0xFFFF0000u) : (wv << 16));
          }
          const float d2 = __uint_as_float(m < 16 ? v0[m] : v1[m - 16]);
          const float x = silu_l2(fmaf(UW[g], gpv, d2));
          pre[m] = x;
          mx = fminf(mx, x);
        }
      }
      XR[hf] = mx;
      named_sync(bar_id, NT);
      mx = fminf(XR[0], XR[1]);
      float sum = 0.f, acc = 0.f;
      const float4* row = reinterpret_cast<const float4*>(CL + p * CL_LD + 32 * hf);
#pragma unroll
      for (int m4 = 0; m4 < 8; ++m4) {
        const float4 c = row[m4];
        const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float e = ex2(mx - pre[m4 * 4 + i]);
          sum += e;
          acc = fmaf(e, cv[i], acc);
        }
      }
      if (hf == 1) {
        XR[2] = sum;
        XR[3] = acc;
      }
      named_sync(bar_id, NT);
      if (hf == 0 && p < t.np) {
        const float s = __fdiv_rn(acc + XR[3], sum + XR[2]);
        if (P.begin) P.out[t.seg0 + t.j0 + p] = s;
        else P.out[(int64_t)t.b * P.out_ld + t.j0 + p] = s;
      }
      tc_fence_before();
      TRACE(7);
      named_sync(bar_id, NT);  // CL / UW / exchange slots are rewritten by this group's next tile
      ph ^= 1;
    }
  }
  // ---- teardown ----
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// B0 operand image per query: 16 rows x 64 bf16, SW128 K-major; rows 0-7 = bf16(u_a),
// rows 8-15 = bf16(u_a - bf16(u_a)) (the fp32 query split hi + lo)
__global__ void b0_image_kernel(int B, const float* __restrict__ ue, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < int64_t(B) * 128; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = int(i >> 7), r = int(i & 127) >> 3, c = int(i & 7), a = r & 7;
    const float* u = ue + (int64_t)b * (KX * D) + a * D + c * 8;
    const float4 v0 = __ldg(reinterpret_cast<const float4*>(u)), v1 = __ldg(reinterpret_cast<const float4*>(u) + 1);
    const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t w[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint32_t hw = pack_bf16(f[2 * m], f[2 * m + 1]);
      w[m] = (r < 8) ? hw : pack_bf16(f[2 * m] - __uint_as_float(hw << 16), f[2 * m + 1] - __uint_as_float(hw & 0xFFFF0000u));
    }
    *reinterpret_cast<uint4*>(out + (int64_t)b * 2048 + sw128(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace tc

bool mol_tc_supported(const molr_cache* c, const molr_gating* g, int k_u) {
  return c && g && k_u == 8 && c->k_x == 8 && c->d == 64 && c->G == 64 && g->G == 64 && g->H == 128 &&
         (c->embs_bf16 != nullptr || (c->embs_hl != nullptr && c->embs_hl_tmap_ok)) &&
         (c->gp_bf16 != nullptr || c->gp_f32 != nullptr) && g->w1t_bf16 != nullptr && !dev_knob("MOLR_DISABLE_TC");
}

__global__ void tile_prefix_kernel(int B, const int64_t* begin, const int64_t* end, int64_t X, int P, int64_t* pre);

template <class Id>
int mol_score_tc(molr_ctx* ctx, const molr_cache* c, const molr_gating* g, int B, const float* ue, const float* uw,
                 float tau, Segs<Id> segs, float* out, int64_t out_ld, cudaStream_t s) {
  if (B <= 0) return MOLR_OK;
  Scratch pre;
  MOLR_TRY(pre.alloc(size_t(B + 1) * 8, s));
  tile_prefix_kernel<<<1, 1024, 0, s>>>(B, segs.begin, segs.end, segs.X, tc::TILE, pre.as<int64_t>());
  MOLR_LAUNCHED(ctx);
  // the persistent kernel reads the tile count from pre[B] itself (no host round trip); the grid
  // is one CTA per SM unless the (dense) tile count is known to be smaller
  const int64_t T = segs.begin ? int64_t(ctx->num_sms) : int64_t(B) * ((segs.X + tc::TILE - 1) / tc::TILE);
  if (T == 0) return MOLR_OK;
  Scratch b0;
  MOLR_TRY(b0.alloc(size_t(B) * 2048, s));
  tc::b0_image_kernel<<<std::min(div_up(int64_t(B) * 128, 256), ctx->num_sms * 8), 256, 0, s>>>(B, ue, b0.as<uint8_t>());
  MOLR_LAUNCHED(ctx);
  tc::Params P;
  P.B = B;
  P.b0img = b0.as<uint8_t>();
  P.inv_tau = 1.0f / tau;
  const bool hl = c->embs_bf16 == nullptr;  // f32-stored components: hi + lo image, two passes
  P.hl = hl ? 1 : 0;
  P.embs = hl ? c->embs_hl : c->embs_bf16;
  P.embs_lo = hl ? c->embs_hl + size_t(c->X) * 512 : nullptr;
  P.gp = c->gp_bf16;
  P.gpf = c->gp_bf16 ? nullptr : c->gp_f32;
  P.w1t = g->w1t_bf16;
  P.w2t = g->w2t_bf16;
  P.w1b = g->w1t_bf16 + 8192;
  P.w1tl = g->w1t_bf16 + 18432;
  P.w2tl = g->w1t_bf16 + 26624;
  P.user_embs = ue;
  P.uw = uw;
  P.begin = segs.begin;
  P.end = segs.end;
  P.X = segs.X;
  P.tile_pre = pre.as<int64_t>();
  P.out = out;
  P.out_ld = out_ld;
  {
    const char* gm = dev_knob("MOLR_GATHER");
    P.gather4 = ((hl ? c->embs_hl_tmap_ok : c->embs_tmap_ok) && !(gm && gm[0] == 'b')) ? 1 : 0;
  }
  Scratch trace;
  P.trace = nullptr;
  const char* trace_path = dev_knob("MOLR_TRACE_MOL");
  if (trace_path) {
    MOLR_TRY(trace.alloc(65536 * 8, s));
    MOLR_CUDA(cudaMemsetAsync(trace.p, 0, 8, s));
    P.trace = trace.as<unsigned long long>();
  }
  auto kern = P.gpf ? tc::mol_tc_kernel<Id, true> : tc::mol_tc_kernel<Id, false>;
  const int smem = tc::SMEM_BYTES;
  MOLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = (int)std::min<int64_t>(T, ctx->num_sms);
  kern<<<grid, 64 + tc::NE * 256 + 32 * tc::NE, smem, s>>>(P, segs.ids, hl ? c->embs_hi_tmap : c->embs_tmap,
                                                            hl ? c->embs_lo_tmap : c->embs_tmap);
  MOLR_LAUNCHED(ctx);
  if (trace_path) {  // dev tool: dump CTA 0's epilogue timeline
    std::vector<unsigned long long> h(65536);
    MOLR_CUDA(cudaMemcpyAsync(h.data(), trace.p, 65536 * 8, cudaMemcpyDeviceToHost, s));
    MOLR_CUDA(cudaStreamSynchronize(s));
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return MOLR_OK;
}

template int mol_score_tc<int64_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, const float*, const float*,
                                   float, Segs<int64_t>, float*, int64_t, cudaStream_t);
template int mol_score_tc<int32_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, const float*, const float*,
                                   float, Segs<int32_t>, float*, int64_t, cudaStream_t);

}  // namespace molr

using namespace molr;

extern "C" int molr_mol_uses_tensor_cores(const molr_cache* c, const molr_gating* g, int k_u) {
  if (!c || !g) return MOLR_ERR_INVALID;
  return mol_tc_supported(c, g, k_u) ? 1 : 0;
}

// Weight operand images for the tensor-core path (built once per gating handle):
//   W1T  [128 hidden rows j][64 K = logit g]      bf16, SW128 K-major   (16 KB)
//   W1B  [128 rows j][16 K]: K0 = bf16(b1[j]), K1 = bf16(b1[j] - K0)   interleave (4 KB)
//   W2T  2 atoms x [64 rows g][64 K = hidden j]  bf16, SW128 K-major   (16 KB)
extern "C" int molr_gating_tc_prepare(molr_gating* g) {
  if (g->G != 64 || g->H != 128) return MOLR_OK;  // the generic kernel serves other shapes
  std::vector<float> w1(size_t(64) * 128), b1(128), w2(size_t(128) * 64);
  MOLR_CUDA(cudaMemcpy(w1.data(), g->w1, w1.size() * 4, cudaMemcpyDefault));
  MOLR_CUDA(cudaMemcpy(b1.data(), g->b1, b1.size() * 4, cudaMemcpyDefault));
  MOLR_CUDA(cudaMemcpy(w2.data(), g->w2, w2.size() * 4, cudaMemcpyDefault));
  // [W1T hi 8192][W1B 2048][W2T hi 8192 (fp16)][W1T lo 8192][W2T lo 8192 (fp16)]
  std::vector<__nv_bfloat16> img(8192 + 2048 + 8192 + 8192 + 8192, __float2bfloat16(0.0f));
  auto sw = [](int r, int k) {  // element offset in an SW128 K-major [rows x 64] region
    return (r >> 3) * 512 + (r & 7) * 64 + ((((k >> 3) ^ (r & 7))) << 3) + (k & 7);
  };
  // layer 1 in log2 units (see silu_l2): W1 and b1 times -log2(e), rounded once to f32, then split
  const double nl2e = -1.4426950408889634;
  for (int j = 0; j < 128; ++j)
    for (int gg = 0; gg < 64; ++gg) {
      const float x = float(nl2e * double(w1[size_t(gg) * 128 + j]));
      const __nv_bfloat16 hi = __float2bfloat16(x);
      img[sw(j, gg)] = hi;
      img[18432 + sw(j, gg)] = __float2bfloat16(x - __bfloat162float(hi));
    }
  for (int j = 0; j < 128; ++j) {
    const float bj = float(nl2e * double(b1[j]));
    __nv_bfloat16 hi = __float2bfloat16(bj);
    __nv_bfloat16 lo = __float2bfloat16(bj - __bfloat162float(hi));
    const int base = 8192 + (j >> 3) * 128 + (j & 7) * 8;  // ilv(j, 0) in elements (chunk 0: K 0..7)
    img[base + 0] = hi;
    img[base + 1] = lo;
  }
  // W2^T as fp16 (the L2 MMA runs fp16 x fp16 -> f32: h and W2 at 2^-11 relative)
  for (int gg = 0; gg < 64; ++gg)
    for (int j = 0; j < 128; ++j) {
      const float x = w2[size_t(j) * 64 + gg];
      const __half hv = __float2half_rn(x);
      reinterpret_cast<__half*>(img.data())[8192 + 2048 + (j >> 6) * 4096 + sw(gg, j & 63)] = hv;
      reinterpret_cast<__half*>(img.data())[26624 + (j >> 6) * 4096 + sw(gg, j & 63)] = __float2half_rn(x - __half2float(hv));
    }
  // w1t_bf16 points at the start of the image, w2t_bf16 at +10240
  MOLR_CUDA(cudaMalloc(&g->w1t_bf16, img.size() * 2));
  MOLR_CUDA(cudaMemcpy(g->w1t_bf16, img.data(), img.size() * 2, cudaMemcpyHostToDevice));
  g->w2t_bf16 = g->w1t_bf16 + 10240;
  return MOLR_OK;
}
